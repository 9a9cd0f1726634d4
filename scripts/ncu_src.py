"""Summarise an ncu --page source CSV: SASS opcode mix + stall share, and
(with --cuda) per-CUDA-line instruction/stall hot spots."""
import csv
import sys
from collections import Counter

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Source" in r and ("Instructions Executed" in r))
hdr = rows[hdr_i]
I = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]


def num(x):
    try:
        return int(float(x))
    except Exception:
        return 0


tot = sum(num(r[I["Instructions Executed"]]) for r in data) or 1
samp = sum(num(r[I["Warp Stall Sampling (All Samples)"]]) for r in data) or 1
print("total warp instr", tot, "stall samples", samp)
if "--cuda" in sys.argv:
    items = sorted(data, key=lambda r: -num(r[I["Warp Stall Sampling (All Samples)"]]))[:30]
    for r in items:
        print("%6.1f%% stall %6.1f%% instr | %s" % (100 * num(r[I["Warp Stall Sampling (All Samples)"]]) / samp,
                                                  100 * num(r[I["Instructions Executed"]]) / tot,
                                                  r[I["Source"]].strip()[:110]))
else:
    op, st = Counter(), Counter()
    for r in data:
        toks = r[I["Source"]].split()
        if not toks:
            continue
        o = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        o = o.split(".")[0]
        op[o] += num(r[I["Instructions Executed"]])
        st[o] += num(r[I["Warp Stall Sampling (All Samples)"]])
    for o, c in op.most_common(28):
        print("%-10s %6.1f%% instr %6.1f%% stall" % (o, 100 * c / tot, 100 * st[o] / samp))
