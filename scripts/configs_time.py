"""Device time of every BASELINE config (C0..C5): median of 10 warm sorts, L2 flushed before each."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def timeit(fn, prep, reps=10):
    ts = []
    for r in range(reps + 3):
        prep()
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if r >= 3:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


out = {}
for name, n, kind in (("C1", 100_000, "uniform01"), ("C2", 1_000_000, "uniform01"), ("C3", 7_000_000, "uniform01"),
                      ("C0", 10_000_000, "uniform01"), ("C5", 10_000_000, "dup256")):
    p = K.generate_device(n, 20260816, kind)
    k = torch.empty_like(p)
    ms = timeit(lambda: K.k_sort(k), lambda: k.copy_(p))
    ok = bool(torch.equal(k, torch.sort(p).values))
    out[name] = {"n": n, "kind": kind, "ms": round(ms, 4), "Gkeys_s": round(n / ms / 1e6, 2), "ok": ok}
    print(name, out[name], flush=True)
# C4: 500 x 100K independent arrays (one segmented call)
seg, nseg = 100_000, 500
p = torch.cat([K.generate_device(seg, 20260816 + r, "uniform01") for r in range(nseg)])
off = torch.arange(0, (nseg + 1) * seg, seg, dtype=torch.int64, device="cuda")
k = torch.empty_like(p)
ms = timeit(lambda: K.k_sort_segments(k, off), lambda: k.copy_(p))
ok = bool(torch.equal(k.view(nseg, seg), torch.sort(p.view(nseg, seg), dim=1).values))
out["C4"] = {"n": nseg * seg, "kind": "500x100K", "ms": round(ms, 4), "Gkeys_s": round(nseg * seg / ms / 1e6, 2), "ok": ok}
print("C4", out["C4"], flush=True)
json.dump(out, open(os.path.join("gpurun_out", "configs_time.json"), "w"), indent=1)
