"""Cycle split of the on-chip segment sorter per size class (exp/lib_trace.so built with -DKS_TRACE)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KSORT_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "exp", "lib_trace.so")
from paper_1107_3622_b200 import _lib  # noqa: E402
import torch  # noqa: E402
import paper_1107_3622_b200 as K  # noqa: E402

L = _lib.load()
L.ks_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
p = K.generate_device(10_000_000, 20260816)
k = torch.empty_like(p)
buf = (ctypes.c_ulonglong * 32)()
for rep in range(2):
    k.copy_(p)
    torch.cuda.synchronize()
    L.ks_trace_read(ctypes.addressof(buf), 32, 1)
    K.k_sort(k)
    torch.cuda.synchronize()
    L.ks_trace_read(ctypes.addressof(buf), 32, 0)
    for c in range(3):
        b = 16 + 5 * c
        segs = max(buf[b + 4], 1)
        print("rep %d class %d: %d segs; cycles/seg load %.0f hist %.0f scan+scatter %.0f order+write %.0f" %
              (rep, c, buf[b + 4], buf[b] / segs, buf[b + 1] / segs, buf[b + 2] / segs, buf[b + 3] / segs))
buf2 = (ctypes.c_ulonglong * 64)()
k.copy_(p)
torch.cuda.synchronize()
L.ks_trace_read(ctypes.addressof(buf2), 64, 1)
K.k_sort(k)
torch.cuda.synchronize()
L.ks_trace_read(ctypes.addressof(buf2), 64, 0)
for c in range(3):
    b = 32 + 8 * c
    segs = max(buf2[16 + 5 * c + 4], 1)
    print("class %d: %d segs, %.0f keys/seg; order+write split: pre %.0f | 4a %.0f | sync %.0f | 4b %.0f | 4c %.0f | sync %.0f" %
          (c, segs, buf2[b + 7] / segs, buf2[b] / segs, buf2[b + 1] / segs, buf2[b + 2] / segs, buf2[b + 3] / segs,
           buf2[b + 4] / segs, buf2[b + 5] / segs))
