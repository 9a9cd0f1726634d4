#!/bin/bash
# A/B device timing of exp/lib_*.so builds over the BASELINE single-array configs.
#   gpurun -- 'bash scripts/ab_suite.sh exp/lib_a.so exp/lib_b.so'
LIBS=("$@")
for cfg in "10000000 uniform01" "7000000 uniform01" "1000000 uniform01" "100000 uniform01" "10000000 dup256"; do
  set -- $cfg; n=$1; k=$2; shift 2
  echo "== n=$n kind=$k"
  EXP_N=$n EXP_KIND=$k EXP_REPS=${EXP_REPS:-30} timeout 300 python scripts/ab_time.py "${LIBS[@]}" 2>&1 | grep "^{"
done
echo "== C4 500 x 100000"
EXP_N=100000 EXP_BATCH=500 EXP_REPS=${EXP_REPS:-15} timeout 300 python scripts/ab_time.py "${LIBS[@]}" 2>&1 | grep "^{"
