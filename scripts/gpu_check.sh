#!/bin/bash
# One GPU round trip: smoke, parity tests, bench (no ncu).  Usage under gpurun:
#   gpurun --timeout 1500 -- 'bash scripts/gpu_check.sh [pytest -k expr]'
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"; tail -3 gpurun_out/smoke.log
K=${1:-}
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
fi
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench=$?"
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
    print("value %.3e keys/s  ms/step %.3f  levels %s  bytes/key %.1f  correct %s" % (d["value"], d["ms_per_step"], d["multi_pass"]["levels"], d["multi_pass"]["bytes_per_key"], d["correct"]))
    for k, v in d["phases"].items():
        if v["launches"]:
            print("  %-8s %8.3f ms  %3d launches  %8.1f GB/s" % (k, v["ms"], v["launches"], v["bytes"] / max(v["ms"], 1e-9) / 1e6))
    print("e2e", d.get("e2e"))
except Exception as e:
    print("bench parse failed", e); print(open("gpurun_out/bench.log").read()[-3000:])
PY
