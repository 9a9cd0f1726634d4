"""Device time of skewed 10M-key distributions (median of 5, L2 flushed)."""
import os, statistics, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1107_3622_b200 as K
from tests.test_gpu_parity import _skewed
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
n = 10_000_000
for kind in ("uniform", "exponential", "lognormal", "normal", "clusters", "powers_of_two", "small_integers", "bit_patterns"):
    rng = np.random.default_rng(1)
    a = rng.random(n) if kind == "uniform" else _skewed(kind, n, rng)
    p = torch.as_tensor(a).cuda(); k = torch.empty_like(p)
    ts = []
    for r in range(7):
        k.copy_(p); flush.zero_(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); K.k_sort(k); e1.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(e0.elapsed_time(e1))
    ok = bool(torch.equal(k, torch.sort(p).values))
    print("%-15s %.3f ms  levels %d  ok %s" % (kind, statistics.median(ts), K.last_stats.levels, ok), flush=True)
