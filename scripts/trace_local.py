"""Phase cycles of k_finish per piece (needs scripts/libksort_trace.so built with KS_TRACE=1)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1107_3622_b200 import _lib  # noqa: E402

L = _lib.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libksort_trace.so"))
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
    print("rep %d: %d pieces (> 512 keys), %d keys; cycles/piece: load+pivots %.0f classify %.0f scan+perm %.0f "
          "sort-units %.0f; cycles/key: classify %.2f sort %.2f" % (
              rep, segs, keys, buf[0] / max(segs, 1), buf[1] / max(segs, 1), buf[2] / max(segs, 1),
              buf[3] / max(segs, 1), buf[1] / max(keys, 1), buf[3] / max(keys, 1)))
