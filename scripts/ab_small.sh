#!/bin/bash
# A/B device timing of exp/lib_*.so builds over small single arrays (latency-bound sizes).
#   gpurun -- 'bash scripts/ab_small.sh exp/lib_a.so exp/lib_b.so'
LIBS=("$@")
for n in ${SIZES:-100000 300000 1000000 2000000 4000000}; do
  echo "== n=$n"
  EXP_N=$n EXP_KIND=uniform01 EXP_REPS=${EXP_REPS:-30} timeout 300 python scripts/ab_time.py "${LIBS[@]}" 2>&1 | grep "^{" | cut -c1-140
done
