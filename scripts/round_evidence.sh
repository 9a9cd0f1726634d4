#!/bin/bash
# Full round evidence on one B200: smoke, GPU parity tests, bench + reference arm,
# ncu launch list of the bench, one --set full capture of the top kernels.
#   gpurun --timeout 3000 -- 'bash scripts/round_evidence.sh r01e'
set -u
TAG=${1:-r01}
bash scripts/gpu_check.sh
bash scripts/evidence.sh $TAG
python scripts/configs_time.py > gpurun_out/configs_$TAG.json 2> gpurun_out/configs_$TAG.err; echo "configs=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scatter|k_leaf|k_segsort|k_count' \
    -s 0 -c 8 -o gpurun_out/full_$TAG python scripts/run_one.py > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncufull=$?"
python scripts/ncu_summary.py gpurun_out/full_$TAG.ncu-rep > gpurun_out/full_summary_$TAG.txt 2>&1
python scripts/ncu_counters.py gpurun_out/full_$TAG.ncu-rep gpurun_out/counters_$TAG > /dev/null 2>&1; echo "counters=$?"
timeout 300 python scripts/adversarial_time.py --out gpurun_out/adversarial_$TAG.json > gpurun_out/adversarial_$TAG.log 2>&1; echo "adv=$?"
timeout 500 python scripts/exact_time.py > gpurun_out/exact_time_$TAG.json 2> gpurun_out/exact_time_$TAG.err; echo "exact=$?"
if [ -f exp/lib_tl.so ]; then
  timeout 120 python scripts/timeline.py 10000000 uniform01 gpurun_out/tl_$TAG.json > gpurun_out/timeline_$TAG.txt 2>&1; echo "timeline=$?"
fi
