"""Per-launch device times (second sort of scripts/run_one.py) from an ncu launch-list CSV."""
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
I = {x: i for i, x in enumerate(h)}
seen = set()
ks = []
for r in rows[hi + 1:]:
    if len(r) != len(h) or r[I["Metric Name"]] != "gpu__time_duration.sum":
        continue
    if r[I["ID"]] in seen:
        continue
    seen.add(r[I["ID"]])
    t = float(r[I["Metric Value"]].replace(",", ""))
    u = r[I["Metric Unit"]]
    t = t / 1000.0 if u in ("ns", "nsecond") else (t * 1000.0 if u in ("ms", "msecond") else t)
    ks.append((r[I["Kernel Name"]].split("(")[0].replace("void ", ""), t, r[I["Grid Size"]]))
# split the two sorts at the second k_init
starts = [i for i, k in enumerate(ks) if k[0].startswith("k_init")]
seq = ks[starts[-1]:] if starts else ks
tot = 0.0
for name, t, grid in seq:
    tot += t
    print("%-28s %9.1f us  grid %s" % (name, t, grid))
print("total %.1f us over %d launches" % (tot, len(seq)))
