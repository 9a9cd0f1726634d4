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
BARGS="--steps 3 --warmup 3 --no-cpu-baseline --no-configs --no-e2e"
timeout 300 python bench.py $BARGS > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py $BARGS \
    > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu=$?"
# per-kernel DRAM traffic of one warm sort (roofline.traffic)
timeout 300 python scripts/run_one.py > gpurun_out/plain_t_$TAG.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none --csv --log-file gpurun_out/traffic_$TAG.csv python scripts/run_one.py \
    > gpurun_out/ncu_t_$TAG.log 2>&1; echo "ncu_traffic=$?"
