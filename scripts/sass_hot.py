"""Per-instruction execution counts / stall samples from `ncu --page source --csv --print-source sass`.
Usage: python scripts/sass_hot.py file.csv [kernel-substring] [min_exec]"""
import csv
import sys

path = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 1
rows = [r for r in csv.reader(open(path, errors="replace")) if r]
blocks, cur = [], None
for r in rows:
    if r[0] == "Kernel Name":
        cur = [r[1], None, []]
        blocks.append(cur)
    elif r[0] == "Address" and cur is not None:
        cur[1] = r
    elif cur is not None and cur[1] is not None and len(r) == len(cur[1]):
        cur[2].append(r)
seen = set()
for name, h, data in blocks:
    if want not in name or name in seen:
        continue
    seen.add(name)
    I = {x: i for i, x in enumerate(h)}
    num = lambda x: float(x) if x not in ("", "-") else 0.0
    tot = sum(num(r[I["Instructions Executed"]]) for r in data) or 1
    samp = sum(num(r[I["Warp Stall Sampling (All Samples)"]]) for r in data) or 1
    print("==", name[:90], "instr", int(tot), "samples", int(samp))
    for k, r in enumerate(data):
        e = num(r[I["Instructions Executed"]])
        if e >= mn:
            print("%5d %10d %5.1f%% %s" % (k, e, 100 * num(r[I["Warp Stall Sampling (All Samples)"]]) / samp,
                                          r[I["Source"]].strip()[:80]))
