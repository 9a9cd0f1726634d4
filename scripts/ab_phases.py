"""Per-phase device times (KS_FLAG_PROFILE: CUDA events around every launch)
of several libksort.so builds in one process, interleaved; L2 flushed before
each sort.  Usage: python scripts/ab_phases.py exp/lib_a.so exp/lib_b.so
(env EXP_N, EXP_KIND, EXP_REPS)."""
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
reps = int(os.environ.get("EXP_REPS", "15"))
libs = []
for path in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(path))
    L.ks_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32]
    L.ks_workspace_bytes.restype = ctypes.c_size_t
    L.ks_sort_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                              ctypes.c_uint32, ctypes.POINTER(_lib.KsStatus)]
    wsb = L.ks_workspace_bytes(n, 1, 0)
    libs.append((os.path.basename(path), L, torch.empty(wsb, dtype=torch.uint8, device="cuda"), wsb))
pristine = K.generate_device(n, 20260816, kind)
want = torch.sort(pristine).values
keys = torch.empty_like(pristine)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
stream = torch.cuda.current_stream()
ph = {nm: [] for nm, *_ in libs}
ok = {nm: True for nm, *_ in libs}
for r in range(reps + 2):
    for nm, L, ws, wsb in (libs[r % len(libs):] + libs[:r % len(libs)]):
        keys.copy_(pristine)
        flush.zero_()
        torch.cuda.synchronize()
        st = _lib.KsStatus()
        rc = L.ks_sort_f64(keys.data_ptr(), n, ws.data_ptr(), wsb, stream.cuda_stream, _lib.KS_FLAG_PROFILE,
                           ctypes.byref(st))
        torch.cuda.synchronize()
        ok[nm] = ok[nm] and rc == 0 and bool(torch.equal(keys, want))
        if r >= 2:
            ph[nm].append([float(st.phase_ms[i]) for i in range(8)])
for nm, *_ in libs:
    med = [statistics.median(x[i] for x in ph[nm]) for i in range(8)]
    print(json.dumps({"lib": nm, "n": n, "kind": kind, "ok": ok[nm], "total_ms": round(sum(med), 4),
                      **{p: round(m, 4) for p, m in zip(_lib.PHASES, med)}}))
