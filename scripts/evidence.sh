#!/bin/bash
# Round evidence: default bench line, reference arm, ncu launch list of the bench.
# Usage under gpurun:  bash scripts/evidence.sh TAG
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench=$?"
tail -c 600 gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref=$?"
cat gpurun_out/bench_ref_$TAG.json | head -c 400; echo
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu=$?"
