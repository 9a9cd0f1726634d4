"""Device time of pathological inputs (looking for performance cliffs): median of 5, L2 flushed,
bytewise checked against torch.sort.   python scripts/pathological_time.py [n ...]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1107_3622_b200 as K

flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def make(kind, n, r):
    if kind == "sawtooth":
        return (np.arange(n) % 1000).astype(np.float64)
    if kind == "two_values":
        return r.integers(0, 2, n).astype(np.float64)
    if kind == "all_equal_but_one":
        a = np.full(n, 1.5); a[n // 3] = 0.25; return a
    if kind == "nearly_sorted":
        a = np.arange(n, dtype=np.float64); i = r.integers(0, n, n // 100); a[i] = a[i[::-1]]; return a
    if kind == "desc_blocks":
        return (np.arange(n) // 4096 * 4096 + (4095 - np.arange(n) % 4096)).astype(np.float64)
    if kind == "subnormals":
        return r.integers(1, 1 << 40, n).astype(np.int64).view(np.float64).copy()
    if kind == "huge":
        return r.random(n) * 1e300 + 1e299
    if kind == "negative":
        return -r.random(n) - 1e-3
    if kind == "million_distinct":
        return r.integers(0, 1_000_000, n).astype(np.float64)
    if kind == "same_pivots_then_uniform":
        a = r.random(n); a[:4096] = 0.5; return a
    if kind == "pivots_tiny_range":
        a = r.random(n); a[:4096] = 0.5 + r.random(4096) * 1e-12; return a
    if kind == "heavy_tail":
        return r.standard_cauchy(n)
    if kind == "zipf":
        return r.zipf(1.3, n).astype(np.float64)
    raise ValueError(kind)


KINDS = ["sawtooth", "two_values", "all_equal_but_one", "nearly_sorted", "desc_blocks", "subnormals", "huge",
         "negative", "million_distinct", "same_pivots_then_uniform", "pivots_tiny_range", "heavy_tail", "zipf"]
for n in [int(x) for x in sys.argv[1:]] or [10_000_000]:
    for kind in KINDS:
        r = np.random.default_rng(7)
        p = torch.as_tensor(make(kind, n, r)).cuda()
        k = torch.empty_like(p)
        ts = []
        for rep in range(7):
            k.copy_(p); flush.zero_(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); K.k_sort(k); e1.record(); torch.cuda.synchronize()
            if rep >= 2:
                ts.append(e0.elapsed_time(e1))
        ok = bool(torch.equal(k.view(torch.int64), torch.sort(p).values.view(torch.int64)))
        print("%9d %-26s %8.3f ms  levels %2d  launches %3d  syncs %d  ok %s" %
              (n, kind, statistics.median(ts), K.last_stats.levels, K.last_stats.launches, K.last_stats.host_syncs, ok),
              flush=True)
