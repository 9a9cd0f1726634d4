"""Device time of k_sort over array sizes up to 1e9 keys (8 GB): median of a few
sorts, L2 flushed before each; output checked sorted and as a permutation
(sum and sum of squares of the key bit patterns, int64 wrap-around)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def digest(x):
    b = x.view(torch.int64)
    return int(b.sum()), int((b * b).sum())


for n in [int(a) for a in (sys.argv[1:] or ["10000000", "100000000", "1000000000"])]:
    p = K.generate_device(n, 20260816)
    want = digest(p)
    k = torch.empty_like(p)
    ts = []
    for r in range(4 if n <= 100_000_000 else 3):
        k.copy_(p)
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        K.k_sort(k)
        b.record()
        torch.cuda.synchronize()
        if r:
            ts.append(a.elapsed_time(b))
    ok = K.is_sorted(k) and digest(k) == want
    ms = statistics.median(ts)
    print(json.dumps({"n": n, "ms": round(ms, 3), "Gkeys_s": round(n / ms / 1e6, 2), "ok": bool(ok),
                      "levels": K.last_stats.levels, "bytes_per_key": round(K.last_stats.bytes_moved / n, 1),
                      "mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1)}), flush=True)
    del p, k
    torch.cuda.empty_cache()
