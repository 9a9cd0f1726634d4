"""Cycle split of the leaf kernel (exp/lib_trace.so built with -DKS_TRACE)."""
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
    tot = buf[13] + buf[14] + buf[15]
    print("rep %d: leaf CTA-cycles fetch %.1fM local %.1fM sort %.1fM (sum %.1fM = %.0f us/CTA over 148); "
          "local segs %d keys %d; local split pivots %.1fM count %.1fM scatter %.1fM emit %.1fM" %
          (rep, buf[13] / 1e6, buf[14] / 1e6, buf[15] / 1e6, tot / 1e6, tot / 148 / 1965.0, buf[4], buf[5],
           buf[0] / 1e6, buf[1] / 1e6, buf[2] / 1e6, buf[3] / 1e6))
