"""Per-kernel ncu counters that justify the design: DRAM bytes and
throughput, L2 bytes, global load/store sector efficiency, occupancy, issue
activity and the full warp-stall breakdown (cycles per issued instruction).

    python scripts/ncu_counters.py gpurun_out/full_r02a.ncu-rep profiles/r02a_ncu_counters

writes <out>.csv (one row per captured launch, raw metric values) and <out>.txt
(a readable table; stall reasons sorted by weight per kernel).  The report must
come from an `ncu --set full` capture (MemoryWorkloadAnalysis + WarpStateStats).
"""
import csv
import io
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
I = {h: i for i, h in enumerate(hdr)}

BASE = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("lts__t_sectors_srcunit_tex_op_write_lookup_miss.sum", "l2_write_lookup_miss_sectors"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "l2_write_sectors"),
    ("smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio", "ld_bytes_per_sector"),
    ("smsp__sass_average_data_bytes_per_sector_mem_global_op_st.ratio", "st_bytes_per_sector"),
    ("smsp__sass_inst_executed_op_global_ld.sum", "global_ld_inst"),
    ("smsp__sass_inst_executed_op_global_st.sum", "global_st_inst"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local_ld_inst"),
    ("smsp__sass_inst_executed_op_local_st.sum", "local_st_inst"),
    ("smsp__inst_executed.sum", "inst_executed"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
STALL = sorted(h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"))


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return float("nan")


def kname(r):
    return r[I["Kernel Name"]].split("(")[0].replace("void ", "")


with open(out + ".csv", "w", newline="") as f:
    w = csv.writer(f)
    cols = [m for m, _ in BASE if m in I] + STALL
    w.writerow(["id", "kernel"] + cols)
    w.writerow(["", ""] + [units[I[m]] for m in cols])
    for r in data:
        w.writerow([r[I["ID"]], kname(r)] + [r[I[m]] for m in cols])

lines = [f"# ncu --set full counters from {rep.split('/')[-1]} (scripts/ncu_counters.py)", ""]
for r in data:
    v = {name: num(r[I[m]]) for m, name in BASE if m in I}
    u = {name: units[I[m]] for m, name in BASE if m in I}
    dur_us = v["duration"] * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[u["duration"]]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    rd = v["dram_read"] * scale.get(u["dram_read"], 1e-6)
    wr = v["dram_write"] * scale.get(u["dram_write"], 1e-6)
    lines.append(f"== {kname(r)}  (id {r[I['ID']]}, grid {int(v['grid'])} x {int(v['block'])}, {int(v['regs'])} regs)")
    lines.append(f"   duration {dur_us:8.2f} us   DRAM read {rd:8.2f} MB  write {wr:8.2f} MB  "
                 f"({1000 * (rd + wr) / dur_us:7.1f} GB/s, {v['dram_pct']:.1f}% of peak)")
    if "l2_write_sectors" in v:
        lines.append(f"   L2 write sectors {v['l2_write_sectors']:.4g}, lookup misses {v['l2_write_lookup_miss_sectors']:.4g}")
    lines.append(f"   global ld {v['ld_bytes_per_sector']:.2f} B/sector ({v['global_ld_inst']:.4g} inst)   "
                 f"st {v['st_bytes_per_sector']:.2f} B/sector ({v['global_st_inst']:.4g} inst)   "
                 f"local ld/st inst {v['local_ld_inst']:.4g}/{v['local_st_inst']:.4g}")
    lines.append(f"   inst {v['inst_executed']:.4g}   issue active {v['issue_active_pct']:.1f}%   occupancy {v['occupancy_pct']:.1f}%")
    st = sorted(((num(r[I[m]]), m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]) for m in STALL),
                reverse=True)
    tot = sum(x for x, _ in st if x == x)
    lines.append("   stalls (cycles per issued inst; share): " +
                 ", ".join(f"{n} {x:.2f} ({100 * x / tot:.0f}%)" for x, n in st if x >= 0.05 * tot))
    lines.append("")
open(out + ".txt", "w").write("\n".join(lines))
print("\n".join(lines))
