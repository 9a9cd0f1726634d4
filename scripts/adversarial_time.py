"""Device time of the reference's adversarial shapes (tests/test_sort_core.py:163-177
of the reference: presorted, reversed, constant; plus organ-pipe and few distinct
values) at 1M and 10M keys, L2 flushed before each sort.  Reports levels (global
passes + leaf launches) and checks the output bytewise against torch.sort.

    python scripts/adversarial_time.py [--out gpurun_out/adversarial.json]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--out", default="gpurun_out/adversarial.json")
p.add_argument("--sizes", default="1000000,10000000")
p.add_argument("--reps", type=int, default=5)
a = p.parse_args()


def make(kind, n):
    if kind == "presorted":
        return torch.arange(n, dtype=torch.float64, device="cuda")
    if kind == "reversed":
        return torch.arange(n, 0, -1, dtype=torch.float64, device="cuda")
    if kind == "constant":
        return torch.full((n,), 0.5, dtype=torch.float64, device="cuda")
    if kind == "organ":
        h = n // 2
        return torch.cat([torch.arange(h, dtype=torch.float64, device="cuda"),
                          torch.arange(n - h, 0, -1, dtype=torch.float64, device="cuda")])
    if kind == "few_distinct":
        g = torch.Generator(device="cuda").manual_seed(n)
        return torch.randint(0, 3, (n,), generator=g, device="cuda").to(torch.float64)
    if kind == "uniform01":
        return K.generate_device(n, 20260816)
    raise ValueError(kind)


flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
res = []
for n in [int(x) for x in a.sizes.split(",")]:
    for kind in ("uniform01", "presorted", "reversed", "constant", "organ", "few_distinct"):
        src = make(kind, n)
        want = torch.sort(src).values
        x = torch.empty_like(src)
        ts, walls = [], []
        for r in range(a.reps + 1):
            x.copy_(src)
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.perf_counter()
            e0.record()
            K.k_sort(x)
            e1.record()
            torch.cuda.synchronize()
            w1 = time.perf_counter()
            if r > 0:
                ts.append(e0.elapsed_time(e1))
                walls.append(1e3 * (w1 - w0))
        ok = bool(torch.equal(x.view(torch.int64), want.view(torch.int64)))
        d = {"n": n, "kind": kind, "ms": statistics.median(ts), "wall_ms": statistics.median(walls),
             "levels": K.last_stats.levels, "bytes_per_key": K.last_stats.bytes_moved / n, "correct": ok}
        res.append(d)
        print(json.dumps(d), flush=True)
json.dump(res, open(a.out, "w"), indent=1)
