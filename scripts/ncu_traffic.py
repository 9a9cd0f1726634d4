"""DRAM traffic and device time of every kernel of one warm C0 sort, from an ncu
launch list taken with
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --cache-control none --csv --log-file L.csv python scripts/run_one.py
(run_one sorts twice, flushing L2 before each sort like bench.py; the second
sort is reported).  Writes profiles/ncu_traffic.json, which bench.py reads for
roofline.traffic (per phase and for the whole sort).

    python scripts/ncu_traffic.py gpurun_out/traffic_r02b.csv [profiles/ncu_traffic.json]
"""
import collections
import csv
import json
import sys

path = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_traffic.json"
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
I = {x: i for i, x in enumerate(h)}
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) != len(h):
        continue
    k = per.setdefault(r[I["ID"]], {"kernel": r[I["Kernel Name"]].split("(")[0].replace("void ", ""),
                                    "grid": r[I["Grid Size"]]})
    v = float(r[I["Metric Value"]].replace(",", ""))
    u = r[I["Metric Unit"]]
    m = r[I["Metric Name"]]
    if m == "gpu__time_duration.sum":
        k["duration_us"] = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[u]
    elif m.startswith("dram__bytes_"):
        b = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        k["dram_read_MB" if "read" in m else "dram_write_MB"] = b / 1e6
ks = list(per.values())
starts = [i for i, k in enumerate(ks) if k["kernel"].startswith("k_init")]
seq = ks[starts[-1]:] if starts else ks


def phase_of(name):
    for pre, ph in (("k_count", "count"), ("k_scatter", "scatter"), ("k_leaf", "leaf"), ("k_segsort", "leaf"),
                    ("k_scan", "scan"), ("k_plan", "plan"), ("k_pivot", "pivots"), ("k_seg_offsets", "pivots")):
        if name.startswith(pre):
            return ph
    return "gate"


phases = collections.OrderedDict()
for k in seq:
    p = phases.setdefault(phase_of(k["kernel"]), {"launches": 0, "dram_bytes": 0.0, "duration_us": 0.0})
    p["launches"] += 1
    p["dram_bytes"] += 1e6 * (k.get("dram_read_MB", 0) + k.get("dram_write_MB", 0))
    p["duration_us"] += k.get("duration_us", 0)
for p in phases.values():
    p["dram_bytes_per_launch"] = p["dram_bytes"] / p["launches"]
tot = sum(p["dram_bytes"] for p in phases.values())
phases["sort"] = {"launches": len(seq), "dram_bytes": tot, "dram_bytes_per_launch": tot,
                  "duration_us": sum(p["duration_us"] for p in phases.values())}
d = {"source": f"ncu launch list ({path.split('/')[-1]}): gpu__time_duration + dram__bytes_read/write per kernel, "
               "--clock-control none --cache-control none, second of two sorts (L2 flushed before each)",
     "workload": "C0: 1 x 10,000,000 float64 uniform01", "kernels": seq, "phases": phases}
json.dump(d, open(out, "w"), indent=1)
for k in seq:
    print("%-26s %8.1f us  DRAM r %7.2f MB  w %7.2f MB" % (k["kernel"], k.get("duration_us", 0),
                                                          k.get("dram_read_MB", 0), k.get("dram_write_MB", 0)))
print("sort: %.1f us serialised, %.1f MB DRAM" % (phases["sort"]["duration_us"], tot / 1e6))
