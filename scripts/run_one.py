"""Sort one C0 workload a few times (for ncu / compute-sanitizer runs)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=10_000_000)
p.add_argument("--kind", default="uniform01")
p.add_argument("--reps", type=int, default=2)
p.add_argument("--batch", type=int, default=0, help="C4 shape: this many arrays of --n keys, one segmented call")
a = p.parse_args()
if a.batch:
    seg, nseg = a.n, a.batch
    p0 = torch.cat([K.generate_device(seg, 20260816 + r, a.kind) for r in range(nseg)])
    off = torch.arange(nseg + 1, dtype=torch.int64, device="cuda") * seg
    k = torch.empty_like(p0)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    for _ in range(a.reps):
        k.copy_(p0)
        flush.zero_()
        K.k_sort_segments(k, off)
    torch.cuda.synchronize()
    ok = all(K.is_sorted(k[r * seg:(r + 1) * seg]) for r in range(0, nseg, 97))
    print("sorted", ok, K.last_stats)
    sys.exit(0 if ok else 1)
pristine = K.generate_device(a.n, 20260816, a.kind)
keys = torch.empty_like(pristine)
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    keys.copy_(pristine)
    flush.zero_()   # L2 flushed before each sort, as in bench.py (ncu: run with --cache-control none)
    K.k_sort(keys)
torch.cuda.synchronize()
ok = K.is_sorted(keys)
print("sorted", ok, K.last_stats)
sys.exit(0 if ok else 1)
