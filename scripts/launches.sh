#!/bin/bash
# per-kernel device times of one warm sort (ncu launch list, cold-cache & serialised)
python scripts/run_one.py "$@" > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches.csv \
    python scripts/run_one.py "$@" > gpurun_out/ncu_l.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; I = {x: i for i, x in enumerate(h)}
ks = [r for r in rows[hi+1:] if len(r) == len(h) and r[I["Metric Name"]] == "gpu__time_duration.sum"]
# run_one sorts twice (L2 flushed before each, as in bench.py); report the second sort
starts = [i for i, r in enumerate(ks) if "k_init" in r[I["Kernel Name"]]]
half = starts[-1] if starts else len(ks) // 2
agg = collections.OrderedDict()
for r in ks[half:]:
    nm = r[I["Kernel Name"]].split("(")[0].replace("void ", "")
    t = float(r[I["Metric Value"]].replace(",", ""))
    unit = r[I["Metric Unit"]]
    t = t / 1000.0 if unit in ("nsecond", "ns") else (t if unit in ("usecond", "us") else t * 1000.0)
    a = agg.setdefault(nm, [0, 0.0]); a[0] += 1; a[1] += t
tot = sum(v[1] for v in agg.values())
for k, (c, t) in agg.items():
    print("%-40s %3d launches %9.1f us  %5.1f%%" % (k, c, t, 100 * t / tot))
print("total %.1f us over %d launches" % (tot, sum(v[0] for v in agg.values())))
PY
