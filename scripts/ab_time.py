"""Interleaved A/B timing of libksort.so builds in ONE process (resolves a few us).
Usage: python scripts/ab_time.py exp/lib_a.so exp/lib_b.so ...   (env EXP_N, EXP_KIND, EXP_REPS)
Each round sorts the same pristine input once per library (order rotated), L2
flushed before each sort; prints the median / p20 device time per library."""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1107_3622_b200 import _lib  # noqa: E402
import paper_1107_3622_b200 as K  # noqa: E402

n = int(os.environ.get("EXP_N", "10000000"))
kind = os.environ.get("EXP_KIND", "uniform01")
reps = int(os.environ.get("EXP_REPS", "40"))
batch = int(os.environ.get("EXP_BATCH", "0"))   # C4 shape: EXP_BATCH arrays of EXP_N keys, one segmented call
libs = []
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path))
    L.ks_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32]
    L.ks_workspace_bytes.restype = ctypes.c_size_t
    L.ks_sort_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                              ctypes.c_uint32, ctypes.POINTER(_lib.KsStatus)]
    L.ks_sort_f64.restype = ctypes.c_int
    L.ks_sort_f64_segmented.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_size_t, ctypes.c_void_p, ctypes.c_uint32, ctypes.POINTER(_lib.KsStatus)]
    L.ks_sort_f64_segmented.restype = ctypes.c_int
    wsb = L.ks_workspace_bytes(n * max(1, batch), max(1, batch), 0)
    libs.append((os.path.basename(path), L, torch.empty(wsb, dtype=torch.uint8, device="cuda"), wsb))

if batch:
    pristine = torch.cat([K.generate_device(n, 20260816 + r, kind) for r in range(batch)])
    off = torch.arange(batch + 1, dtype=torch.int64, device="cuda") * n
    want = torch.sort(pristine.view(batch, n), dim=1).values.reshape(-1)
else:
    pristine = K.generate_device(n, 20260816, kind)
    want = torch.sort(pristine).values
keys = torch.empty_like(pristine)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream()
st = _lib.KsStatus()
times = {nm: [] for nm, *_ in libs}
ok = {nm: True for nm, *_ in libs}
for r in range(reps + 3):
    order = libs[r % len(libs):] + libs[:r % len(libs)]
    for nm, L, ws, wsb in order:
        keys.copy_(pristine)
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if batch:
            rc = L.ks_sort_f64_segmented(keys.data_ptr(), off.data_ptr(), batch, n * batch, ws.data_ptr(), wsb,
                                         stream.cuda_stream, 0, ctypes.byref(st))
        else:
            rc = L.ks_sort_f64(keys.data_ptr(), n, ws.data_ptr(), wsb, stream.cuda_stream, 0, ctypes.byref(st))
        b.record(stream)
        torch.cuda.synchronize()
        if rc != 0:
            ok[nm] = False
        if r >= 3:
            times[nm].append(a.elapsed_time(b))
            if r == 3:
                ok[nm] = ok[nm] and bool(torch.equal(keys, want))
for nm, *_ in libs:
    t = sorted(times[nm])
    print(json.dumps({"lib": nm, "n": n, "kind": kind, "ms_median": round(statistics.median(t), 4),
                      "ms_p20": round(t[len(t) // 5], 4), "ms_min": round(t[0], 4), "ms_p80": round(t[(4 * len(t)) // 5], 4),
                      "ok": ok[nm]}))
