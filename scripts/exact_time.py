"""Wall time of the exact paths (reference permutation / op counts) on the GPU:
k_sort(a, counts), k_sort on mixed signed zeros, heap_sort(a, counts).

    python scripts/exact_time.py > gpurun_out/exact_time.json

k_sort(a, counts) reproduces the reference recursion level by level (one CTA
per segment > 512 keys), heap_sort(a, counts) is the reference heap sort on
ONE device lane (inherently serial sift-downs): correctness paths, timed here
so that their cost is on record next to the reference's own Python timings.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for n in (100_000, 1_000_000, 10_000_000):
    p = K.generate_device(n, 20260816)
    want = torch.sort(p).values
    for rep in range(2):
        a = p.clone()
        c = K.OpCounts()
        s = timed(lambda: K.k_sort(a, c))
    print(json.dumps({"path": "k_sort(a, counts)", "n": n, "seconds": round(s, 4), "comparisons": c.comparisons,
                      "moves": c.moves, "max_pending_ranges": c.max_pending_ranges,
                      "levels": K.sort_core.last_stats.levels, "correct": bool(torch.equal(a, want))}), flush=True)
for n in (1_000_000, 10_000_000):
    p = K.generate_device(n, 20260816)
    p[::1000] = 0.0
    p[500::1000] = -0.0
    want = torch.sort(p).values
    for rep in range(2):
        a = p.clone()
        s = timed(lambda: K.k_sort(a))
    print(json.dumps({"path": "k_sort(a), mixed +0.0 / -0.0 (exact engine)", "n": n, "seconds": round(s, 4),
                      "levels": K.sort_core.last_stats.levels, "correct_values": bool(torch.equal(a, want))}), flush=True)
for n in (20_000, 100_000, 300_000):
    p = K.generate_device(n, 20260816)
    want = torch.sort(p).values
    a = p.clone()
    c = K.OpCounts()
    s = timed(lambda: K.heap_sort(a, c))
    print(json.dumps({"path": "heap_sort(a, counts) (one device lane)", "n": n, "seconds": round(s, 4),
                      "comparisons": c.comparisons, "moves": c.moves, "correct": bool(torch.equal(a, want))}), flush=True)
