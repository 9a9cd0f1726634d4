"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference's ``sortlab.sort_core`` and ``sortlab.workload``
through a namespace shim (``sortlab/__init__.py`` imports matplotlib, which is
absent), runs them on seeded inputs and writes the results as
JSON fixtures next to this script.  Floats are stored as 16-hex-digit IEEE-754
bit patterns so the fixtures are bit-exact (``-0.0`` vs ``+0.0`` included).

The fixtures pin the oracle (tests/test_oracle.py) and the device path
(tests/test_gpu_parity.py).  Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import struct
import sys
import types

import numpy as np

REF = "/root/reference/pkg/src/sortlab"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    pkg = types.ModuleType("sortlab")
    pkg.__path__ = [REF]
    sys.modules["sortlab"] = pkg
    from sortlab import sort_core, workload  # noqa: E402
    return sort_core, workload


def hx(v: float) -> str:
    return struct.pack(">d", v).hex()


def hxl(vs) -> list[str]:
    return [hx(v) for v in vs]


def sha(vs) -> str:
    return hashlib.sha256(np.asarray(vs, dtype="<f8").tobytes()).hexdigest()


def counts_dict(c) -> dict:
    return {"comparisons": c.comparisons, "moves": c.moves,
            "max_pending_ranges": c.max_pending_ranges}


def gen_arrays(rng: random.Random, count: int, max_n: int):
    """Seeded inputs covering the reference's tested shapes and the ±0 caveat."""
    pools = [
        lambda: rng.random(),
        lambda: float(rng.randint(0, 9)),                       # heavy duplicates
        lambda: rng.choice([0.0, -0.0, 0.5, -0.5, 1.0]),         # mixed signed zeros
        lambda: rng.choice([0.0, -0.0, 1e-310, -1e-310, 5e-324, 1.7976931348623157e308,
                            -1.7976931348623157e308, 2.5, -2.5]),  # extremes + subnormals
        lambda: rng.uniform(-1e6, 1e6),
        lambda: rng.randint(0, 255) / 256.0,                     # dup256 style
    ]
    out = []
    for t in range(count):
        n = rng.randint(0, max_n)
        draw = pools[t % len(pools)]
        out.append([draw() for _ in range(n)])
    return out


def main() -> None:
    sc, wl = _import_reference()

    # ---- workload: splitmix64 stream, derive_seed, generate --------------------
    work = {}
    streams = {}
    for seed in (0, 1, 7, 42, 1234, 20260816, 2**64 - 1):
        g = wl.SplitMix64(seed)
        streams[str(seed)] = [str(g.next_uint64()) for _ in range(8)]
    work["streams"] = streams
    work["derive_seed"] = [
        [s, i, st, str(wl.derive_seed(s, i, st))]
        for s in (0, 7, 11, 20260816) for i in (0, 1, 2, 499) for st in (0, 1, 2)
    ]
    work["generate"] = {
        "n": 257, "seed": 20260816,
        "bits": hxl(wl.generate(wl.WorkloadSpec(257, 20260816))),
    }
    big = wl.generate(wl.WorkloadSpec(100_000, 20260816))
    work["generate_100k_sha256"] = sha(big)
    with open(os.path.join(HERE, "workload.json"), "w") as fh:
        json.dump(work, fh, indent=0)

    # ---- partition: golden trace + seeded random cases -------------------------
    rng = random.Random(20260816)
    parts = []
    trace = [55.0, 66.0, 60.0, 78.0, 22.0, 50.0, 75.0, 5.0, 8.0, 94.0]
    a = list(trace)
    for left, right in ((0, 9), (0, 3), (2, 3)):
        before = list(a)
        c = sc.OpCounts()
        out = sc.ksort_partition(a, left, right, c)
        parts.append({"input": hxl(before), "left": left, "right": right,
                      "output": hxl(a), "pivot": out.pivot_index, "flag": out.flag_used,
                      "counts": counts_dict(c)})
    for arr in gen_arrays(rng, 600, 48):
        if len(arr) < 2:
            continue
        left = rng.randint(0, len(arr) - 2)
        right = rng.randint(left + 1, len(arr) - 1)
        b = list(arr)
        c = sc.OpCounts()
        out = sc.ksort_partition(b, left, right, c)
        parts.append({"input": hxl(arr), "left": left, "right": right, "output": hxl(b),
                      "pivot": out.pivot_index, "flag": out.flag_used,
                      "counts": counts_dict(c)})
    with open(os.path.join(HERE, "partition.json"), "w") as fh:
        json.dump(parts, fh)

    # ---- full sorts: k_sort and heap_sort outputs (bit patterns) + op counts ----
    sorts = []
    cases = [list(trace), [], [1.0], [2.0, 1.0], [1.0, 2.0], [3.0, 3.0, 3.0, 3.0],
             [0.0, -0.0, 0.0, -0.0, 1.0, -0.0], [float(v) for v in range(64)],
             [float(v) for v in range(64, 0, -1)], [0.5] * 50]
    cases += gen_arrays(rng, 420, 200)
    for arr in cases:
        k = list(arr)
        ck = sc.OpCounts()
        sc.k_sort(k, ck)
        h = list(arr)
        ch = sc.OpCounts()
        sc.heap_sort(h, ch)
        sorts.append({"input": hxl(arr), "ksort": hxl(k), "heapsort": hxl(h),
                      "ksort_counts": counts_dict(ck), "heapsort_counts": counts_dict(ch)})
    with open(os.path.join(HERE, "sorts.json"), "w") as fh:
        json.dump(sorts, fh)

    # ---- larger seeded sorts: digests only (inputs regenerate from the seed) ----
    large = []
    for n, seed, kind in ((20_000, 20260816, "uniform01"), (100_000, 20260816, "uniform01"),
                          (4096, 41, "sorted_ascending"), (4096, 41, "sorted_descending"),
                          (3000, 5, "constant"), (50_000, 20260816, "dup256")):
        if kind == "dup256":
            u = wl._bulk_uint64(seed, n)
            arr = ((u >> np.uint64(56)).astype(np.float64) / 256.0).tolist()
        else:
            arr = wl.generate(wl.WorkloadSpec(n, seed, kind))
        k = list(arr)
        ck = sc.OpCounts()
        sc.k_sort(k, ck)
        entry = {"n": n, "seed": seed, "kind": kind, "input_sha256": sha(arr),
                 "ksort_sha256": sha(k), "ksort_counts": counts_dict(ck)}
        if n <= 20_000:
            h = list(arr)
            ch = sc.OpCounts()
            sc.heap_sort(h, ch)
            entry["heapsort_sha256"] = sha(h)
            entry["heapsort_counts"] = counts_dict(ch)
        large.append(entry)
    with open(os.path.join(HERE, "large.json"), "w") as fh:
        json.dump(large, fh, indent=1)
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
