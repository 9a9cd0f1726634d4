"""Key metrics per kernel launch from an ncu report (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
I = {h: i for i, h in enumerate(hdr)}
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Grid Size", "Block Limit Registers", "Block Limit Shared Mem", "Dynamic Shared Memory Per Block"]
cur = None
for r in rows[1:]:
    k = r[I["Kernel Name"]][:40] + " #" + r[I["ID"]]
    if r[I["Metric Name"]] in want:
        if k != cur:
            print("==", k)
            cur = k
        print("   %-32s %s %s" % (r[I["Metric Name"]], r[I["Metric Value"]], r[I["Metric Unit"]]))
