"""Cycle split of the level-0 pivot build (needs exp/lib_trace.so built with KS_DEFS=-DKS_TRACE)."""
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
buf = (ctypes.c_ulonglong * 16)()
for rep in range(3):
    k.copy_(p)
    torch.cuda.synchronize()
    L.ks_trace_read(ctypes.addressof(buf), 16, 1)
    K.k_sort(k)
    torch.cuda.synchronize()
    L.ks_trace_read(ctypes.addressof(buf), 16, 0)
    print("rep", rep, "L0 pivots cycles: sort+merge %d dedupe %d lut %d | build total %d writes %d" %
          (buf[8], buf[9], buf[10], buf[11], buf[12]))
