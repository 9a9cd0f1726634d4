"""Per-CUDA-line hot spots from `ncu --page source --csv --print-source cuda,sass`
(instructions executed, thread instructions, warp-stall samples), top N lines.
Usage: python scripts/ncu_lines.py file.csv [N]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path, errors="replace")))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
I = {}
for i, x in enumerate(h):
    I.setdefault(x, i)


def num(x):
    try:
        return float(x)
    except Exception:
        return 0.0


lines = []
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) != len(h) or not r[0] or not r[0].isdigit():
        continue
    lines.append((f"{fname}:{r[0]}", r[1].strip(), num(r[I["Instructions Executed"]]),
                  num(r[I["Thread Instructions Executed"]]), num(r[I["Warp Stall Sampling (All Samples)"]])))
ti = sum(x[2] for x in lines) or 1
tt = sum(x[3] for x in lines) or 1
ts = sum(x[4] for x in lines) or 1
print(f"warp inst {ti:.3e}  thread inst {tt:.3e}  stall samples {ts:.0f}")
print(" line                 inst%  thr%  stall%  source")
for ln in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{ln[0]:20s} {100*ln[2]/ti:6.1f} {100*ln[3]/tt:5.1f} {100*ln[4]/ts:6.1f}  {ln[1][:80]}")
