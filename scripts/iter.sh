#!/bin/bash
# One build -> measure iteration on the GPU box (no ncu):
#   gpurun -- 'bash scripts/iter.sh TAG [pytest-k-expr]'
set -u
TAG=${1:-it}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke=$?"; tail -2 gpurun_out/smoke_$TAG.log
if [ -n "${2:-}" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$2" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?"
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?"
fi
tail -3 gpurun_out/pytest_$TAG.log
timeout 300 python scripts/configs_time.py > gpurun_out/configs_$TAG.json 2> gpurun_out/configs_$TAG.err; echo "configs=$?"
cat gpurun_out/configs_$TAG.json
if [ -f exp/lib_tl.so ]; then
  timeout 120 python scripts/timeline.py 10000000 uniform01 gpurun_out/tl_$TAG.json > gpurun_out/tl_$TAG.txt 2>&1; echo "timeline=$?"
  head -12 gpurun_out/tl_$TAG.txt
fi
timeout 300 python scripts/adversarial_time.py > gpurun_out/adv_$TAG.json 2> gpurun_out/adv_$TAG.err; echo "adv=$?"
python - <<PY
import json
try:
    for ln in open("gpurun_out/adv_$TAG.json"):
        r = json.loads(ln); print("  %9d %-12s %.3f ms levels %d %s" % (r["n"], r["kind"], r["ms"], r["levels"], r["correct"]))
except Exception as e: print("adv parse", e)
PY
