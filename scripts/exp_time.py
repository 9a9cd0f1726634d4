"""Time experiment builds of libksort.so against each other on one GPU.
Usage: python scripts/exp_time.py lib1.so lib2.so ...   (each timed in its own process)"""
import json
import os
import subprocess
import sys

CHILD = r'''
import os, sys, json, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_1107_3622_b200 as K
n = int(os.environ.get("EXP_N", "10000000")); kind = os.environ.get("EXP_KIND", "uniform01")
pristine = K.generate_device(n, 20260816, kind)
keys = torch.empty_like(pristine)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
ts = []
for r in range(int(os.environ.get("EXP_REPS", "13"))):
    keys.copy_(pristine); flush.zero_(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); K.k_sort(keys); b.record(); torch.cuda.synchronize()
    if r >= 3: ts.append(a.elapsed_time(b))
ok = bool(K.is_sorted(keys)) and bool(torch.equal(keys, torch.sort(pristine).values))
from paper_1107_3622_b200 import _lib
from paper_1107_3622_b200.sort_core import _sort_device
keys.copy_(pristine); flush.zero_(); torch.cuda.synchronize()
st = _sort_device(keys, _lib.KS_FLAG_PROFILE)
ph = {nm: round(st.phase_ms[i] * 1000, 1) for i, nm in enumerate(_lib.PHASES) if st.phase_launches[i]}
print(json.dumps({"lib": os.path.basename(os.environ.get("KSORT_LIB")), "ms_median": round(statistics.median(ts), 4),
                  "ms_min": round(min(ts), 4), "ok": ok, "phases_us": ph}))
'''

for lib in sys.argv[1:]:
    env = dict(os.environ, KSORT_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    line = (r.stdout.strip().splitlines() or ["{}"])[-1]
    print(line if r.returncode == 0 else json.dumps({"lib": lib, "error": r.stderr[-800:]}), flush=True)
