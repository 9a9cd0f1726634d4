#!/bin/bash
# A/B over several fresh processes (buffer placement differs per process):
#   bash scripts/ab_multi.sh PROCS "N KIND [BATCH]" lib_a.so lib_b.so ...
P=$1; CFG=$2; shift 2
set -- "$@"
read -r N KIND BATCH <<< "$CFG"
for p in $(seq 1 $P); do
  EXP_N=$N EXP_KIND=$KIND EXP_BATCH=${BATCH:-0} EXP_REPS=${EXP_REPS:-20} timeout 300 python scripts/ab_time.py "$@" 2>&1 | grep "^{"
done | python -c "
import sys, json, collections, statistics
d = collections.defaultdict(list)
for l in sys.stdin:
    j = json.loads(l); d[j['lib']].append(j['ms_median'])
for k, v in d.items():
    print('  %-14s %s  median-of-medians %.4f' % (k, ' '.join('%.4f' % x for x in v), statistics.median(v)))
"
