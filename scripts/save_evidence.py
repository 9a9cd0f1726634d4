"""Copy one round-evidence run (scripts/round_evidence.sh TAG) from gpurun_out/ into
profiles/ and refresh profiles/ncu_traffic.json from its --set full capture.
Usage: python scripts/save_evidence.py TAG"""
import csv
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
G, P = "gpurun_out", "profiles"
for src, dst in [(f"bench_{tag}.json", f"{tag}_bench.json"), (f"bench_ref_{tag}.json", f"{tag}_bench_reference.json"),
                 (f"launches_{tag}.csv", f"{tag}_ncu_launches.csv"), (f"full_summary_{tag}.txt", f"{tag}_ncu_full_summary.txt"),
                 (f"configs_{tag}.json", f"{tag}_configs_time.json"), ("pytest_gpu.log", f"{tag}_pytest_gpu.log"),
                 (f"scale_n_{tag}.jsonl", f"{tag}_scale_n.jsonl"), (f"counters_{tag}.csv", f"{tag}_ncu_counters.csv"),
                 (f"counters_{tag}.txt", f"{tag}_ncu_counters.txt"), (f"adversarial_{tag}.json", f"{tag}_adversarial.json"),
                 (f"exact_time_{tag}.json", f"{tag}_exact_paths_time.json"), (f"timeline_{tag}.txt", f"{tag}_timeline_c0.txt"), (f"launches_warm_{tag}.txt", f"{tag}_ncu_launches_warm_l2.txt")]:
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))
# launch list of the last timed bench step
rows = list(csv.reader(open(os.path.join(G, f"launches_{tag}.csv"))))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
I = {x: i for i, x in enumerate(h)}
ks = [r for r in rows[hi + 1:] if len(r) == len(h) and r[I["Metric Name"]] == "gpu__time_duration.sum"]
# a step starts with the level-0 pivot ranking (round 2) or the init kernel (round 1 builds)
idx = [i for i, r in enumerate(ks) if "k_pivot_rank" in r[I["Kernel Name"]]] or \
      [i for i, r in enumerate(ks) if "k_init" in r[I["Kernel Name"]]]
with open(os.path.join(P, f"{tag}_ncu_launches.txt"), "w") as fh:
    fh.write("# ncu launch list (gpu__time_duration.sum, --clock-control none) of the last timed bench step, "
             "C0 10M uniform01 (serialised by ncu; the side-stream launches run concurrently in the bench)\n")
    tot = 0.0
    step = []
    for r in ks[idx[-1]:]:   # (until the first kernel that is not the engine's: the bench's context timings)
        if step and "k_" not in r[I["Kernel Name"]]:
            break
        step.append(r)
    for r in step:
        nm = r[I["Kernel Name"]].split("(")[0].replace("void ", "")
        t = float(r[I["Metric Value"]].replace(",", "")) / 1000.0
        tot += t
        fh.write("%-40s %8.1f us\n" % (nm, t))
    fh.write("%-40s %8.1f us over %d launches\n" % ("total", tot, len(step)))
# DRAM traffic per launch from the full capture (first occurrence of each kernel)
raw = subprocess.run(["ncu", "-i", os.path.join(G, f"full_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
H = {x: i for i, x in enumerate(rr[0])}
seen, kern = set(), []
for r in rr[2:]:
    nm = r[H["Kernel Name"]].split("(")[0].replace("void ", "")
    if nm in seen:
        continue
    seen.add(nm)
    f = lambda k: float(r[H[k]].replace(",", ""))  # noqa: E731
    kern.append({"kernel": nm, "duration_us": f("gpu__time_duration.sum"), "dram_read_MB": f("dram__bytes_read.sum"),
                 "dram_write_MB": f("dram__bytes_write.sum")})
by = {k["kernel"]: k for k in kern}
phases = {"count": ["k_count2<1>", "k_count<1>"], "scatter": ["k_scatter2", "k_scatter"], "leaf": ["k_leaf", "k_segsort<3>", "k_segsort<4>"]}
d = {"source": f"ncu --set full --clock-control none, C0 10M uniform01 (scripts/run_one.py), profiles/{tag}_ncu_full_summary.txt",
     "workload": "C0: 1 x 10,000,000 float64 uniform01", "kernels": kern,
     "phases": {p: {"launches": len([k for k in v if k in by]), "dram_bytes_per_launch":
                    sum((by[k]["dram_read_MB"] + by[k]["dram_write_MB"]) * 1e6 for k in v if k in by) /
                    max(1, len([k for k in v if k in by]))}
                for p, v in phases.items()}}
# whole sort: the heavy kernels of one sort (count, scatter, leaf, list sorters; the small
# front / scan / plan / reset launches move < 3% of the bytes and are not in the capture)
heavy = [k for k in kern if any(x in k["kernel"] for x in ("k_count", "k_scatter", "k_leaf", "k_segsort")) and
         "reset" not in k["kernel"]]
d["phases"]["sort"] = {"launches": len(heavy), "kernels": [k["kernel"] for k in heavy],
                       "dram_bytes_per_launch": sum((k["dram_read_MB"] + k["dram_write_MB"]) * 1e6 for k in heavy)}
json.dump(d, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
print(open(os.path.join(P, f"{tag}_ncu_launches.txt")).read())
print(json.dumps(d["phases"]))
