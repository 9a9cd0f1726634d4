"""Host-side overhead of one k_sort call (python wrapper vs direct ctypes), C0.
Event span with the GPU busy before the call (pre-call host work hidden) and
idle before the call (pre-call host work exposed), plus host wall time."""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1107_3622_b200 import _lib  # noqa: E402
import paper_1107_3622_b200 as K  # noqa: E402
from paper_1107_3622_b200.sort_core import _sort_device, _workspace, _workspace_bytes  # noqa: E402

n = int(os.environ.get("EXP_N", "10000000"))
L = _lib.load()
pristine = K.generate_device(n, 20260816)
keys = torch.empty_like(pristine)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream()
wsb = _workspace_bytes(L, n, 1, 0)
ws = _workspace(wsb)
st = _lib.KsStatus()
sp = stream.cuda_stream


def direct():
    L.ks_sort_f64(keys.data_ptr(), n, ws.data_ptr(), wsb, sp, 0, ctypes.byref(st))


paths = {"k_sort": lambda: K.k_sort(keys), "_sort_device": lambda: _sort_device(keys, 0), "ctypes": direct}
for busy in (True, False):
    for name, fn in paths.items():
        ev, wall = [], []
        for r in range(33):
            keys.copy_(pristine)
            flush.zero_()
            if not busy:
                torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record(stream)
            fn()
            b.record(stream)
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            if r >= 3:
                ev.append(a.elapsed_time(b))
                wall.append((t1 - t0) * 1e3)
        print("%-13s gpu_busy_before=%-5s event %.4f ms  host call %.4f ms" %
              (name, busy, statistics.median(ev), statistics.median(wall)))
