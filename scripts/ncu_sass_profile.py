"""SASS-level profile of one captured launch: instruction mix, divergence,
stall share per opcode and the hottest 32-instruction windows.
    python scripts/ncu_sass_profile.py REP.ncu-rep LAUNCH_INDEX [KEYS]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, idx = sys.argv[1], int(sys.argv[2])
keys = float(sys.argv[3]) if len(sys.argv) > 3 else 1e7
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "--launch-skip", str(idx),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out)) if r]
print(rows[0][1][:100])
his = [i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r]
hi = his[0]
h = rows[hi]
I = {x: i for i, x in enumerate(h)}
data = [r for r in rows[hi + 1:] if len(r) == len(h)]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


samp = sum(num(r[I["Warp Stall Sampling (All Samples)"]]) for r in data) or 1
tot = sum(num(r[I["Instructions Executed"]]) for r in data) or 1
thr = sum(num(r[I["Thread Instructions Executed"]]) for r in data)
print("warp inst %.3g, thread inst %.3g (%.1f per key), avg active lanes %.1f" % (tot, thr, thr / keys, thr / tot))
op, st = Counter(), Counter()
for r in data:
    t = r[I["Source"]].strip().split()
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    op[o] += num(r[I["Instructions Executed"]])
    st[o] += num(r[I["Warp Stall Sampling (All Samples)"]])
print("mix (inst%/stall%): " + " ".join("%s %.1f/%.1f" % (o, 100 * c / tot, 100 * st[o] / samp) for o, c in op.most_common(24)))
acc = [(num(r[I["Warp Stall Sampling (All Samples)"]]), num(r[I["Instructions Executed"]]), r[I["Source"]].strip())
       for r in data]
W = 32
for k in range(0, len(acc), W):
    blk = acc[k:k + W]
    s = sum(b[0] for b in blk)
    ins = sum(b[1] for b in blk)
    if s / samp > 0.02 or ins / tot > 0.02:
        ops = " ".join(sorted(set(b[2].split()[1] if b[2].startswith("@") else b[2].split()[0] for b in blk if b[1] > 0)))
        print("%5d %5.1f%% stall %5.1f%% inst | %s" % (k, 100 * s / samp, 100 * ins / tot, ops[:150]))
