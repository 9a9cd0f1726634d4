"""Randomised stress run (stand-in for compute-sanitizer, which is closed on
this GPU pool): hundreds of seeded inputs over sizes 1..3M and adversarial /
skewed distributions, single arrays, batches with ragged and empty segments,
host buffers, repeated calls (graph capture + replay) and 4 concurrent
threads.  Every output is compared bytewise with torch.sort; run it against the
self-checking build (KS_CHECK=1: every sort also verifies its own multiset
fingerprint and order on the device) to catch races in the device queues.

    KSORT_LIB=exp/lib_check.so python scripts/stress_check.py [--cases 300]
"""
import argparse
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1107_3622_b200 as K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=300)
ap.add_argument("--seed", type=int, default=20261020)
ap.add_argument("--large", action="store_true", help="also every kind at 1M, 4M, 10M and 12.5M keys")
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
KINDS = ["uniform", "dup256", "dup3", "normal", "lognormal", "presorted", "reversed", "organ", "constant",
         "bits", "clusters", "sawtooth"]


def make(kind, n, r):
    if kind == "uniform":
        return r.random(n)
    if kind == "dup256":
        return np.floor(r.random(n) * 256) / 256
    if kind == "dup3":
        return r.integers(0, 3, n).astype(np.float64)
    if kind == "normal":
        return r.normal(0, 1, n)
    if kind == "lognormal":
        return r.lognormal(0, 4, n)
    if kind == "presorted":
        return np.sort(r.random(n))
    if kind == "reversed":
        return np.sort(r.random(n))[::-1].copy()
    if kind == "organ":
        h = np.sort(r.random(n))
        return np.concatenate([h[0::2], h[1::2][::-1]])
    if kind == "constant":
        return np.full(n, 0.25)
    if kind == "bits":
        u = r.integers(1, 2**62, n, dtype=np.int64).view(np.float64)
        return u * r.choice([-1.0, 1.0], n)
    if kind == "clusters":
        c = r.uniform(-1e6, 1e6, 5)
        return c[r.integers(0, 5, n)] + r.normal(0, 1e-9, n)
    if kind == "sawtooth":
        return (np.arange(n) % max(1, n // 7)).astype(np.float64)
    raise ValueError(kind)


def same(x, y):
    return np.array_equal(np.asarray(x).view(np.uint64), np.asarray(y).view(np.uint64))


fails = []
t0 = time.time()
counts = {}
for c in range(a.cases):
    kind = KINDS[c % len(KINDS)]
    n = int(np.exp(rng.uniform(0, np.log(3_000_000))))
    data = make(kind, n, rng)
    mode = ["device", "device_twice", "host", "batch"][c % 4]
    try:
        if mode == "device":
            t = torch.from_numpy(data.copy()).cuda()
            K.k_sort(t)
            ok = same(t.cpu().numpy(), np.sort(data))
        elif mode == "device_twice":   # second call on the same buffers replays the cached graph
            t = torch.from_numpy(data.copy()).cuda()
            K.k_sort(t)
            t.copy_(torch.from_numpy(data[::-1].copy()))
            K.k_sort(t)
            ok = same(t.cpu().numpy(), np.sort(data))
        elif mode == "host":
            h = torch.from_numpy(data.copy()).pin_memory()
            K.k_sort(h)
            ok = same(h.numpy(), np.sort(data))
        else:
            cuts = np.sort(rng.integers(0, n + 1, rng.integers(1, 40)))
            off = np.concatenate([[0], cuts, [n]]).astype(np.int64)
            t = torch.from_numpy(data.copy()).cuda()
            K.k_sort_segments(t, torch.from_numpy(off).cuda())
            got = t.cpu().numpy()
            ok = all(same(got[off[i]:off[i + 1]], np.sort(data[off[i]:off[i + 1]])) for i in range(len(off) - 1))
    except Exception as e:  # noqa: BLE001
        ok = False
        print(f"case {c}: {kind} n={n} {mode}: {e!r}", flush=True)
    counts[mode] = counts.get(mode, 0) + 1
    if not ok:
        fails.append((c, kind, n, mode))
        print(f"FAIL case {c}: {kind} n={n} {mode}", flush=True)

if a.large:
    for n in (1_000_000, 4_000_000, 10_000_000, 12_500_000):
        for kind in KINDS:
            data = make(kind, n, rng)
            t = torch.from_numpy(data).cuda()
            want = torch.sort(t).values
            K.k_sort(t)
            ok = bool(torch.equal(t.view(torch.int64), want.view(torch.int64)))
            counts["large"] = counts.get("large", 0) + 1
            if not ok:
                fails.append((-1, kind, n, "large"))
                print(f"FAIL large: {kind} n={n}", flush=True)

# concurrency: 4 threads x 5 sorts of their own arrays
errs = []


def worker(i):
    try:
        r = np.random.default_rng(100 + i)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for j in range(5):
                d = make(KINDS[(i + j) % len(KINDS)], 400_000 + 1000 * i, r)
                t = torch.from_numpy(d.copy()).cuda()
                K.k_sort(t)
                if not same(t.cpu().numpy(), np.sort(d)):
                    errs.append((i, j))
    except Exception as e:  # noqa: BLE001
        errs.append((i, repr(e)))


ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
for t in ts:
    t.start()
for t in ts:
    t.join()
print(f"{a.cases} cases ({counts}) + 4x5 concurrent sorts in {time.time() - t0:.1f} s: "
      f"{len(fails)} failures, {len(errs)} concurrent failures; library {K._lib.LIB_PATH if hasattr(K, '_lib') else ''}")
sys.exit(1 if fails or errs else 0)
