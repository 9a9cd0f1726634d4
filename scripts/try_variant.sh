#!/bin/bash
# One GPU round trip for an experiment: GPU tests of the default build (-k EXPR
# optional), interleaved A/B of exp/lib_*.so over the configs, per-phase times,
# and an ncu --set full capture of kernels matching NCU_K on the default build.
#   gpurun -- 'NCU_K="k_scatter2|k_count2" bash scripts/try_variant.sh exp/lib_old.so exp/lib_staged.so'
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -4 gpurun_out/pytest_gpu.log
EXP_REPS=${EXP_REPS:-20} timeout 300 python scripts/ab_phases.py "$@" 2>&1 | grep "^{"
EXP_REPS=${EXP_REPS:-20} timeout 600 bash scripts/ab_suite.sh "$@"
if [ -n "${NCU_K:-}" ]; then
  python scripts/run_one.py > gpurun_out/plain_v.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$NCU_K" -c ${NCU_C:-4} \
      -o gpurun_out/${NCU_O:-var} python scripts/run_one.py > gpurun_out/ncu_v.log 2>&1; echo "ncu=$?"
fi
