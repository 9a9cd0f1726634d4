"""Phase cycles of the local partitioner per segment (needs exp/lib_trace.so: scripts/exp_build.sh trace -DKS_TRACE)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1107_3622_b200 import _lib  # noqa: E402

os.environ["KSORT_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "exp", "lib_trace.so")
L = _lib.load(os.environ["KSORT_LIB"])
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
p = K.generate_device(n, 20260816)
k = torch.empty_like(p)
buf = (ctypes.c_ulonglong * 16)()
L.ks_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
for rep in range(3):
    k.copy_(p)
    L.ks_trace_read(ctypes.addressof(buf), 16, 1)
    K.k_sort(k)
    torch.cuda.synchronize()
    L.ks_trace_read(ctypes.addressof(buf), 16, 0)
    segs, keys = buf[4], buf[5]
    print("rep %d: %d local segments, %d keys (%.0f/seg); cycles/seg: pivots %.0f count %.0f scatter %.0f emit %.0f; "
          "cycles/key: count %.2f scatter %.2f" % (
              rep, segs, keys, keys / max(segs, 1), buf[0] / max(segs, 1), buf[1] / max(segs, 1), buf[2] / max(segs, 1),
              buf[3] / max(segs, 1), buf[1] / max(keys, 1), buf[2] / max(keys, 1)))
