"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck), one
run each, checked against torch.sort / the oracle:
  C1 (100K uniform, fast engine: global pass + leaf queues + sorters),
  500 x 10K batch (segmented path), presorted 100K (stall guard, extra levels),
  skewed 300K (hand-backs), mixed signed zeros 30K (exact engine), heap sort exact 2K.
    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402

ok = True


def check(name, got, want):
    global ok
    same = bool(torch.equal(got.view(torch.int64), want.view(torch.int64)))
    ok &= same
    print(f"{name}: {'ok' if same else 'MISMATCH'}", flush=True)


x = K.generate_device(100_000, 20260816)
w = torch.sort(x).values
K.k_sort(x)
check("C1 100K uniform", x, w)

m, nseg = 10_000, 500
p = torch.cat([K.generate_device(m, 1000 + r) for r in range(nseg)])
off = torch.arange(0, (nseg + 1) * m, m, dtype=torch.int64, device="cuda")
w = torch.sort(p.view(nseg, m), dim=1).values.reshape(-1)
K.k_sort_segments(p, off)
check("500 x 10K batch", p, w)

x = torch.arange(100_000, dtype=torch.float64, device="cuda")
w = x.clone()
K.k_sort(x)
check("presorted 100K", x, w)

rng = np.random.default_rng(7)
x = torch.from_numpy(rng.lognormal(0.0, 4.0, 300_000)).cuda()
w = torch.sort(x).values
K.k_sort(x)
check("lognormal 300K", x, w)

a = rng.choice([0.0, -0.0, 1.0, -1.0, 0.5], size=30_000)
x = torch.from_numpy(a.copy()).cuda()
K.k_sort(x)
from oracle import oracle as O  # noqa: E402  (checker only)
b = a.copy()
O.k_sort(b)
check("mixed signed zeros 30K (exact)", x, torch.from_numpy(b).cuda())

a = rng.random(2_000)
x = torch.from_numpy(a.copy()).cuda()
c = K.OpCounts()
K.heap_sort(x, c)
b = a.copy()
O.heap_sort(b)
check("heap sort exact 2K", x, torch.from_numpy(b).cuda())
sys.exit(0 if ok else 1)
