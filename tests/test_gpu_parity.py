"""Parity of the sm_100a engine against the reference (GPU; run with -m gpu).

Oracle: fixtures produced by the reference itself (tests/golden/*.json, made
by tests/golden/make_golden.py) and the C restatement in oracle/ (pinned to
those fixtures by tests/test_oracle.py).  Comparisons are BYTEWISE
(float64 bit patterns), never ``==``, so -0.0/+0.0 arrangements count.
Mirrors the reference's own hot-path tests (pkg/tests/test_sort_core.py,
test_acceptance.py C1/C2) through the drop-in API.
"""
import itertools
import math
import random
import threading
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1107_3622_b200 as K  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.golden_io import load, same_bits, sha256, unhex  # noqa: E402

TRACE_ARRAY = [55.0, 66.0, 60.0, 78.0, 22.0, 50.0, 75.0, 5.0, 8.0, 94.0]
TRACE_SORTED = [5.0, 8.0, 22.0, 50.0, 55.0, 60.0, 66.0, 75.0, 78.0, 94.0]


def dev(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float64)).cuda()


def host(t):
    return t.cpu().numpy()


def oracle_ksort(a):
    b = np.array(a, dtype=np.float64, copy=True)
    O.k_sort(b)
    return b


# ---- golden trace / partition (exact engine) --------------------------------------

def test_partition_golden_calls_1_to_3():
    # reference tests/test_sort_core.py:31-54, test_acceptance.py:63-69
    a = list(TRACE_ARRAY)
    out = K.ksort_partition(a, 0, 9)
    assert a == [8.0, 5.0, 50.0, 22.0, 55.0, 66.0, 75.0, 78.0, 60.0, 94.0]
    assert out.pivot_index == 4 and out.flag_used and a[5] == 66.0
    out = K.ksort_partition(a, 0, 3)
    assert a == [5.0, 8.0, 50.0, 22.0, 55.0, 66.0, 75.0, 78.0, 60.0, 94.0]
    assert out.pivot_index == 1 and out.flag_used and a[2] == 50.0
    out = K.ksort_partition(a, 2, 3)
    assert a == [5.0, 8.0, 22.0, 50.0, 55.0, 66.0, 75.0, 78.0, 60.0, 94.0]
    assert out.pivot_index == 3 and not out.flag_used


def test_partition_fixtures_bitwise():
    for case in load("partition.json"):
        a = dev(unhex(case["input"]))
        c = K.OpCounts()
        out = K.ksort_partition(a, case["left"], case["right"], c)
        assert same_bits(host(a), unhex(case["output"])), case
        assert out.pivot_index == case["pivot"] and out.flag_used == case["flag"]
        assert c.comparisons == case["counts"]["comparisons"]
        assert c.moves == case["counts"]["moves"]


def test_partition_edge_cases():
    a = [3.0, 3.0, 3.0, 3.0]
    assert K.ksort_partition(a, 0, 3).pivot_index == 0 and a == [3.0] * 4
    a = [2.0, 1.0]
    out = K.ksort_partition(a, 0, 1)
    assert a == [1.0, 2.0] and out.pivot_index == 1 and not out.flag_used
    b = [1.0, 2.0]
    out = K.ksort_partition(b, 0, 1)
    assert b == [1.0, 2.0] and out.pivot_index == 0 and out.flag_used
    for left, right in ((0, 0), (2, 1), (-1, 2), (0, 3), (3, 4)):
        with pytest.raises(ValueError):
            K.ksort_partition([1.0, 2.0, 3.0], left, right)
    with pytest.raises(K.NonFiniteKeyError):
        K.ksort_partition([1.0, float("nan"), 3.0], 0, 2)
    # NaN outside the segment is not inspected (sort_core.py:161)
    a = [float("nan"), 2.0, 1.0]
    K.ksort_partition(a, 1, 2)
    assert a[1:] == [1.0, 2.0]


def test_partition_large_segment_matches_oracle():
    rng = np.random.default_rng(3)
    for n, left, right in ((5000, 0, 4999), (100_000, 17, 99_000), (70_000, 5, 69_990)):
        a = np.floor(rng.random(n) * 50) / 7.0
        b = a.copy()
        piv, flag, c = O.partition(b, left, right, counts=True)
        t = dev(a)
        cc = K.OpCounts()
        out = K.ksort_partition(t, left, right, cc)
        assert same_bits(host(t), b)
        assert (out.pivot_index, out.flag_used) == (piv, flag)
        assert (cc.comparisons, cc.moves) == (c.comparisons, c.moves)


# ---- full sorts against reference outputs --------------------------------------------

def test_sort_fixtures_ksort_bitwise():
    for case in load("sorts.json"):
        a = dev(unhex(case["input"]))
        K.k_sort(a)
        assert same_bits(host(a), unhex(case["ksort"])), case["input"][:8]


def test_sort_fixtures_counts():
    for case in load("sorts.json"):
        a = dev(unhex(case["input"]))
        c = K.OpCounts()
        K.k_sort(a, c)
        assert same_bits(host(a), unhex(case["ksort"]))
        assert c.__dict__ == case["ksort_counts"], case["input"][:8]


def test_sort_fixtures_heapsort():
    for case in load("sorts.json"):
        a = dev(unhex(case["input"]))
        K.heap_sort(a)
        assert same_bits(host(a), unhex(case["heapsort"]))
        a = dev(unhex(case["input"]))
        c = K.OpCounts()
        K.heap_sort(a, c)
        assert same_bits(host(a), unhex(case["heapsort"]))
        want = dict(case["heapsort_counts"])
        assert c.__dict__ == want


@pytest.mark.parametrize("idx", range(6))
def test_large_fixtures(idx):
    case = load("large.json")[idx]
    n, seed, kind = case["n"], case["seed"], case["kind"]
    if kind in ("uniform01", "dup256"):
        a = K.generate_device(n, seed, kind)
    elif kind == "constant":
        a = torch.full((n,), 0.5, dtype=torch.float64, device="cuda")
    else:
        a = dev(np.sort(O.uniform01(seed, n)))
        if kind == "sorted_descending":
            a = a.flip(0).contiguous()
    assert sha256(host(a)) == case["input_sha256"]
    b = a.clone()
    K.k_sort(a)
    assert sha256(host(a)) == case["ksort_sha256"]
    c = K.OpCounts()
    K.k_sort(b, c)
    assert sha256(host(b)) == case["ksort_sha256"]
    assert c.__dict__ == case["ksort_counts"]


def test_golden_trace_counts():
    # reference tests/test_sort_core.py:129-137 (20 comparisons, 26 moves, 2 pending)
    a = list(TRACE_ARRAY)
    c = K.OpCounts()
    K.k_sort(a, c)
    assert a == TRACE_SORTED
    assert (c.comparisons, c.moves, c.max_pending_ranges) == (20, 26, 2)


# ---- the reference's correctness suite (test_sort_core.py:223-275, C2) ---------------

@pytest.mark.parametrize("sorter", ["ksort", "heapsort"])
def test_exhaustive_small_permutations(sorter):
    f = K.SORTERS[sorter]
    for n in range(1, 8):
        expect = [float(v) for v in range(1, n + 1)]
        perms = list(itertools.permutations(expect))
        if n <= 5:
            for perm in perms:
                a = list(perm)
                f(a)
                assert a == expect
        # all perms of this n through the batch API in one launch
        flat = torch.tensor([x for p in perms for x in p], dtype=torch.float64, device="cuda")
        off = torch.arange(0, len(perms) * n + 1, n, dtype=torch.int64, device="cuda")
        K.k_sort_segments(flat, off)
        assert same_bits(host(flat), np.tile(np.array(expect), len(perms)))


def test_exhaustive_binary_arrays():
    for n in range(1, 8):
        arrs = list(itertools.product((0.0, 1.0), repeat=n))
        flat = torch.tensor([x for p in arrs for x in p], dtype=torch.float64, device="cuda")
        off = torch.arange(0, len(arrs) * n + 1, n, dtype=torch.int64, device="cuda")
        K.k_sort_segments(flat, off)
        want = np.concatenate([np.sort(np.array(p)) for p in arrs])
        assert same_bits(host(flat), want)
        for p in arrs[:: max(1, len(arrs) // 16)]:
            a = list(p)
            K.k_sort(a)
            assert a == sorted(p)


def test_random_arrays_vs_oracle():
    # acceptance C2 (test_acceptance.py:108-124): seed 20260816, n <= 4096
    rng = random.Random(20260816)
    for _ in range(300):
        n = rng.randint(0, 4096)
        base = [rng.random() for _ in range(n)]
        a = dev(base)
        K.k_sort(a)
        assert same_bits(host(a), oracle_ksort(base))


def test_random_finite_doubles_incl_signed_zeros():
    # hypothesis-style (test_sort_core.py:253-275): arbitrary finite doubles,
    # including subnormals, extremes and mixed -0.0/+0.0
    rng = np.random.default_rng(7)
    specials = np.array([0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, -1.7976931348623157e308,
                         1.7976931348623157e308, 1.0, -1.0])
    for t in range(200):
        n = int(rng.integers(0, 300))
        bits = rng.integers(0, 2**64, size=n, dtype=np.uint64).view(np.float64)
        bits = np.where(np.isfinite(bits), bits, 0.0)
        mask = rng.random(n) < 0.3
        bits[mask] = rng.choice(specials, size=int(mask.sum()))
        a = dev(bits)
        K.k_sort(a)
        assert same_bits(host(a), oracle_ksort(bits)), t
        h = bits.copy()
        O.heap_sort(h)
        b = dev(bits)
        K.heap_sort(b)
        assert same_bits(host(b), h), t


# ---- errors and trivial inputs ------------------------------------------------------

def test_trivial_inputs():
    for a in ([], [1.0], [2.0, 1.0], [1.0, 2.0]):
        b = list(a)
        K.k_sort(b)
        assert b == sorted(a)
        c = list(a)
        K.heap_sort(c)
        assert c == sorted(a)


@pytest.mark.parametrize("n", [3, 5000, 8192, 8193, 100_000, 2_000_000])
def test_nonfinite_rejected_before_any_write(n):
    rng = np.random.default_rng(n)
    for bad in (float("nan"), float("inf"), float("-inf")):
        base = rng.random(n)
        pos = int(rng.integers(0, n))
        base[pos] = bad
        base[n - 1] = bad
        a = dev(base)
        before = host(a).copy()
        with pytest.raises(K.NonFiniteKeyError) as ei:
            K.k_sort(a)
        assert str(ei.value) == f"key at index {min(pos, n - 1)} is {bad!r}; keys must be finite"
        assert same_bits(host(a), before)
        with pytest.raises(K.NonFiniteKeyError):
            K.heap_sort(a)
        assert same_bits(host(a), before)
    with pytest.raises(K.NonFiniteKeyError):
        K.k_sort([float("nan")])


def test_list_and_numpy_and_cpu_tensor_inputs():
    rng = np.random.default_rng(1)
    base = rng.random(20000)
    want = np.sort(base)
    a = base.tolist()
    K.k_sort(a)
    assert same_bits(np.array(a), want)
    b = base.copy()
    K.k_sort(b)
    assert same_bits(b, want)
    c = torch.from_numpy(base.copy())
    K.k_sort(c)
    assert same_bits(c.numpy(), want)
    assert K.is_sorted(a) and K.is_sorted(c) and not K.is_sorted(base)


# ---- host buffers through ks_sort_f64_host (H2D, sort, D2H with one synchronisation) ----

def _host_inputs(base):
    yield "numpy", base.copy()
    yield "cpu", torch.from_numpy(base.copy())
    yield "pinned", torch.from_numpy(base.copy()).pin_memory()


def _bits(x):
    return x.numpy() if isinstance(x, torch.Tensor) else x


@pytest.mark.parametrize("n", [1, 2, 700, 20_000, 1_000_000, 3_000_000])
def test_host_buffers_bitexact(n):
    base = np.random.default_rng(n).random(n)
    want = np.sort(base)
    for name, x in _host_inputs(base):
        K.k_sort(x)
        assert same_bits(_bits(x), want), name


@pytest.mark.parametrize("n", [5000, 100_000, 2_000_000])
def test_host_buffers_nonfinite_untouched(n):
    rng = np.random.default_rng(n + 7)
    base = rng.random(n)
    pos = int(rng.integers(0, n))
    base[pos] = float("inf")
    for name, x in _host_inputs(base):
        with pytest.raises(K.NonFiniteKeyError) as ei:
            K.k_sort(x)
        assert str(ei.value) == f"key at index {pos} is inf; keys must be finite"
        assert same_bits(_bits(x), base), name


def test_host_buffers_signed_zeros_and_counts_match_oracle():
    rng = np.random.default_rng(11)
    base = rng.integers(-3, 4, size=50_000).astype(np.float64)
    base[rng.integers(0, base.size, size=500)] = -0.0   # both zeros: the exact engine
    want = oracle_ksort(base)
    for name, x in _host_inputs(base):
        K.k_sort(x)
        assert same_bits(_bits(x), want), name
    small = np.array(TRACE_ARRAY)
    c = K.OpCounts()
    K.k_sort(small, c)
    assert small.tolist() == TRACE_SORTED and (c.comparisons, c.moves, c.max_pending_ranges) == (20, 26, 2)


@pytest.mark.parametrize("kind", ["presorted", "few_distinct"])
def test_host_buffers_multi_pass_inputs(kind):
    # inputs that need the synchronising loop after the speculative schedule:
    # the copy back is rewritten after the extra passes
    n = 3_000_000
    a = np.arange(n, dtype=np.float64) if kind == "presorted" else \
        np.random.default_rng(5).integers(0, 3, size=n).astype(np.float64)
    for name, x in _host_inputs(a):
        K.k_sort(x)
        assert same_bits(_bits(x), np.sort(a)), name
        assert K.last_stats.levels >= 1


# ---- adversarial shapes (forward progress + parity) ----------------------------------

@pytest.mark.parametrize("kind", ["presorted", "reversed", "constant", "organ", "few_distinct"])
@pytest.mark.parametrize("n", [2048, 8193, 60_000])
def test_adversarial_inputs(kind, n):
    rng = np.random.default_rng(n)
    if kind == "presorted":
        a = np.arange(n, dtype=np.float64)
    elif kind == "reversed":
        a = np.arange(n, 0, -1, dtype=np.float64)
    elif kind == "constant":
        a = np.full(n, 0.5)
    elif kind == "organ":
        a = np.concatenate([np.arange(n // 2), np.arange(n - n // 2, 0, -1)]).astype(np.float64)
    else:
        a = rng.integers(0, 3, size=n).astype(np.float64)
    t = dev(a)
    K.k_sort(t)
    assert same_bits(host(t), np.sort(a))


def test_worklist_depth_bound():
    # test_sort_core.py:163-177
    rng = random.Random(41)
    cases = [[rng.random() for _ in range(1000)], [rng.random() for _ in range(4096)],
             [float(v) for v in range(2048)], [float(v) for v in range(2048, 0, -1)], [0.5] * 1024]
    for a in cases:
        n = len(a)
        want = O.k_sort(np.array(a), counts=True)
        c = K.OpCounts()
        K.k_sort(a, c)
        assert K.is_sorted(a)
        assert c.max_pending_ranges <= math.ceil(math.log2(n)) + 1
        assert c.__dict__ == want.__dict__


# ---- BASELINE.json configs at full size ----------------------------------------------

@pytest.mark.parametrize("n,kind", [(100_000, "uniform01"), (1_000_000, "uniform01"), (7_000_000, "uniform01"),
                                    (10_000_000, "uniform01"), (10_000_000, "dup256")])
def test_configs_full_size_bitexact(n, kind):
    seed = 20260816
    a = K.generate_device(n, seed, kind)
    K.k_sort(a)
    ref = O.uniform01(seed, n) if kind == "uniform01" else O.dup256(seed, n)
    # no -0.0 in these workloads: np.sort's bytes are the reference K-sort's
    # bytes (any correct sort of keys whose equal values are bitwise equal)
    assert np.signbit(ref).sum() == 0
    got = host(a)
    assert same_bits(got, np.sort(ref))
    assert K.last_stats.bytes_moved > 0
    if kind == "uniform01" and n >= 7_000_000:
        # and against the reference K-sort itself (C restatement, ~1 s at 1e7;
        # dup256's quadratic tie handling takes minutes there, so C5 stops at np.sort)
        assert same_bits(got, oracle_ksort(ref))


def test_config_1e5_against_oracle_ksort_and_heap():
    seed = 20260816
    base = O.uniform01(seed, 100_000)
    a = K.generate_device(100_000, seed)
    K.k_sort(a)
    assert same_bits(host(a), oracle_ksort(base))
    h = base.copy()
    O.heap_sort(h)
    b = K.generate_device(100_000, seed)
    K.heap_sort(b)
    assert same_bits(host(b), h)


def test_batch_config_500x100k():
    seed = 20260816
    m, nseg = 100_000, 500
    parts = [O.uniform01(O.derive_seed(seed, r, 0), m) for r in range(nseg)]
    flat = dev(np.concatenate(parts))
    off = torch.arange(0, m * nseg + 1, m, dtype=torch.int64, device="cuda")
    K.k_sort_segments(flat, off)
    got = host(flat)
    for r in range(nseg):
        assert same_bits(got[r * m:(r + 1) * m], np.sort(parts[r])), r


def test_batch_ragged_segments():
    rng = np.random.default_rng(11)
    sizes = [0, 1, 2, 3, 8192, 8193, 17, 0, 40_000, 1, 5, 123_457, 9000, 2]
    data = [np.floor(rng.random(s) * 97) / 13.0 for s in sizes]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    flat = dev(np.concatenate(data))
    K.k_sort_segments(flat, torch.from_numpy(off).cuda())
    got = host(flat)
    for i, d in enumerate(data):
        assert same_bits(got[off[i]:off[i + 1]], oracle_ksort(d)), i


def test_batch_signed_zeros_uses_exact_engine():
    rng = np.random.default_rng(5)
    segs = [rng.choice([0.0, -0.0, 0.5, -0.25], size=s) for s in (50, 9000, 3)]
    off = np.concatenate([[0], np.cumsum([len(s) for s in segs])]).astype(np.int64)
    flat = dev(np.concatenate(segs))
    K.k_sort_segments(flat, torch.from_numpy(off).cuda())
    got = host(flat)
    for i, s in enumerate(segs):
        assert same_bits(got[off[i]:off[i + 1]], oracle_ksort(s))


def test_signed_zero_large_input_exact_engine():
    rng = np.random.default_rng(9)
    a = rng.choice([0.0, -0.0, 1.0, -1.0, 0.5], size=30_000)
    t = dev(a)
    K.k_sort(t)
    assert same_bits(host(t), oracle_ksort(a))
    assert K.last_stats.exact_used


def test_device_generator_matches_reference_stream():
    for seed in (0, 7, 20260816):
        assert same_bits(host(K.generate_device(4097, seed)), O.uniform01(seed, 4097))
        assert same_bits(host(K.generate_device(4097, seed, "dup256")), O.dup256(seed, 4097))


def test_sizes_around_thresholds():
    rng = np.random.default_rng(2)
    for n in (8191, 8192, 8193, 16384, 16385, 32769, 65536 * 2 + 3, 300_001):
        a = rng.random(n)
        t = dev(a)
        K.k_sort(t)
        assert same_bits(host(t), np.sort(a)), n


def _skewed(kind, n, rng):
    if kind == "exponential":
        return rng.exponential(1.0, n)
    if kind == "lognormal":
        return rng.lognormal(0.0, 4.0, n)
    if kind == "normal":
        return rng.normal(0.0, 1.0, n)
    if kind == "clusters":   # a few very narrow clusters far apart
        centers = rng.uniform(-1e6, 1e6, 7)
        return centers[rng.integers(0, 7, n)] + rng.normal(0.0, 1e-9, n)
    if kind == "powers_of_two":   # exponentially spaced values: worst case for interpolation buckets
        return np.ldexp(1.0, rng.integers(-1000, 1000, n)) * rng.choice([-1.0, 1.0], n)
    if kind == "small_integers":
        return rng.integers(0, 1000, n).astype(np.float64)
    if kind == "bit_patterns":   # random finite doubles over the whole exponent range
        u = rng.integers(0, 2**63, n, dtype=np.int64).view(np.float64)
        u[~np.isfinite(u)] = 1.0
        u[u == 0.0] = 1.0   # keep signed zeros out of the fast-engine bitwise contract
        return u * rng.choice([-1.0, 1.0], n)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["exponential", "lognormal", "normal", "clusters", "powers_of_two",
                                  "small_integers", "bit_patterns"])
@pytest.mark.parametrize("n", [300_001, 3_000_000])
def test_skewed_distributions(kind, n):
    """Value distributions that defeat the segment sorter's interpolation buckets
    (oversized buckets, hand-backs to the first-key partitioner) must still sort exactly."""
    rng = np.random.default_rng(zlib.crc32(f"{kind}/{n}".encode()))   # fixed per case (hash() is salted per process)
    a = _skewed(kind, n, rng)
    t = dev(a)
    K.k_sort(t)
    assert same_bits(host(t), np.sort(a)), kind


@pytest.mark.parametrize("kind", ["exponential", "clusters", "powers_of_two", "bit_patterns"])
def test_skewed_large_inputs(kind):
    """Inputs of >= 8M keys take the single-buffer class-1 sorter (KS_SINGLE_MIN_N):
    skewed buckets, hand-backs and bounded items through that path."""
    n = 9_000_001
    rng = np.random.default_rng(zlib.crc32(f"{kind}/{n}".encode()))   # fixed per case (hash() is salted per process)
    a = _skewed(kind, n, rng)
    t = dev(a)
    K.k_sort(t)
    assert same_bits(host(t), np.sort(a)), kind


def test_sizes_around_engine_limits():
    """Sizes at every routing threshold (tiny gap, unit, sort classes, on-chip sort, local partition)."""
    rng = np.random.default_rng(3)
    for n in (16, 17, 512, 513, 2048, 2049, 6144, 6145, 12288, 12289, 131072, 131073, 262147):
        a = rng.random(n)
        t = dev(a)
        K.k_sort(t)
        assert same_bits(host(t), np.sort(a)), n


@pytest.mark.parametrize("n", [2_399_999, 2_400_001, 4_799_999, 4_800_001, 5_000_337, 7_399_999, 7_400_001])
def test_sizes_around_tile_count_thresholds(n):
    """One array gets 1 / 2 / 3 / 4 staged-scatter tiles per SM by its size (stage_items_per_sm in
    ks_fast.cu): sizes on both sides of each switch, uniform keys and a skewed distribution
    (chunks at the tile capacity, multi-level passes), sorted twice (direct launch, then the graph)."""
    rng = np.random.default_rng(n)
    for a in (rng.random(n), rng.exponential(1.0, n), np.floor(rng.random(n) * 300.0)):
        want = np.sort(a)
        t = dev(a)
        for _ in range(2):
            t.copy_(torch.from_numpy(a))
            K.k_sort(t)
            assert same_bits(host(t), want), n


def _small_case(kind, n, rng):
    if kind == "uniform":
        return rng.random(n)
    if kind == "dup256":
        return np.floor(rng.random(n) * 256.0) / 256.0
    if kind == "three_values":      # equality runs far longer than one CTA's range, empty gaps
        return rng.integers(0, 3, n).astype(np.float64)
    if kind == "constant":
        return np.full(n, 0.375)
    if kind == "presorted":
        return np.arange(n, dtype=np.float64)
    if kind == "reversed":
        return np.arange(n, 0, -1).astype(np.float64)
    if kind == "organ":
        h = n // 2
        return np.concatenate([np.arange(h), np.arange(n - h, 0, -1)]).astype(np.float64)
    if kind == "one_big_gap":       # 60% of the keys between two neighbouring pivots (not a stall: < 3/4)
        a = rng.random(n)
        m = rng.random(n) < 0.6
        m[:4096] = False
        a[m] = 0.5 + rng.random(int(m.sum())) * 1e-9
        return a
    if kind == "sorted_prefix":     # the first P keys are the smallest: ~P empty gaps in the first CTA's range
        a = rng.random(n) + 1.0
        m = min(4096, n // 2)
        a[:m] = np.sort(rng.random(m))
        return a
    if kind == "lognormal":
        return rng.lognormal(0.0, 4.0, n)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["uniform", "dup256", "three_values", "constant", "presorted", "reversed", "organ",
                                  "one_big_gap", "sorted_prefix", "lognormal"])
@pytest.mark.parametrize("n", [2049, 5000, 24_577, 150_001, 1_000_003, 1_999_999, 4_999_999, 5_000_001])
def test_small_array_cooperative_path(kind, n):
    """One array of 2K..5M keys sorts in one cooperative launch (k_small in ks_fast.cu): equality runs
    that span several CTAs' ranges, gaps above the on-chip sorter's capacity (next level), the stall
    bail-out (presorted / reversed / organ-pipe), batches of more than 128 gaps per CTA -- called three
    times (direct launch, graph capture, replay), bytewise against numpy."""
    rng = np.random.default_rng(zlib.crc32(f"small/{kind}/{n}".encode()))
    a = _small_case(kind, n, rng)
    want = np.sort(a)
    t = dev(a)
    for _ in range(3):
        t.copy_(torch.from_numpy(a))
        K.k_sort(t)
        assert same_bits(host(t), want), (kind, n)


@pytest.mark.parametrize("n", [3000, 100_000, 1_000_000, 5_000_000])
def test_small_array_takes_two_launches(n):
    """Uniform arrays of 2K..5M keys finish in two kernels (k_small + the reset / status kernel) and one
    host wait -- the general schedule takes eleven launches (ks_status_t.launches, host_syncs)."""
    from paper_1107_3622_b200.sort_core import _sort_device
    p = K.generate_device(n, 20260816)
    want = torch.sort(p).values
    for call in range(3):   # direct launch, graph capture, replay
        t = p.clone()
        st = _sort_device(t)
        assert torch.equal(t, want)
        assert int(st.launches) == 2 and int(st.host_syncs) == 1, (call, int(st.launches), int(st.host_syncs))
    big = K.generate_device(5_000_001, 20260816)
    st = _sort_device(big)
    assert int(st.launches) > 2


@pytest.mark.parametrize("n", [2049, 30_000, 400_000, 1_700_000])
def test_small_array_cooperative_path_rejections(n):
    """Non-finite keys (first, middle, last CTA's chunk) leave the buffer untouched; mixed signed
    zeros rerun in the exact engine (bytes equal to the reference K-sort's)."""
    rng = np.random.default_rng(n)
    for pos in (0, n // 2, n - 1):
        a = rng.random(n)
        a[pos] = np.nan if pos != n // 2 else np.inf
        t = dev(a)
        with pytest.raises(K.NonFiniteKeyError) as ei:
            K.k_sort(t)
        assert f"index {pos} " in str(ei.value)
        assert same_bits(host(t), a)
    if n <= 30_000:
        a = rng.random(n)
        a[::7] = 0.0
        a[3::7] = -0.0
        t = dev(a)
        K.k_sort(t)
        assert same_bits(host(t), oracle_ksort(a))


def test_sort_on_caller_side_stream():
    # the engine launches on the caller's current stream (sort_core._stream_ptr):
    # a sort issued under torch.cuda.stream(s) right after the input is produced
    # on s must see that input and finish before s's next op
    s = torch.cuda.Stream()
    n = 1_000_003
    with torch.cuda.stream(s):
        x = K.generate_device(n, 20260816)
        want = torch.sort(x).values
        K.k_sort(x)
        same = torch.equal(x, want)
    s.synchronize()
    assert bool(same)
    # and twice on the same buffers (the second call replays the cached graph) on another stream
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        y = K.generate_device(n, 7)
        want2 = torch.sort(y).values
        K.k_sort(y)
        y2 = K.generate_device(n, 7)
        y.copy_(y2)
        K.k_sort(y)
        same2 = torch.equal(y, want2)
    s2.synchronize()
    assert bool(same2)


# ---- concurrency (distinct arrays may be sorted from distinct threads) ----

def test_concurrent_threads_distinct_arrays():
    """Four threads each sort their own 1M-key array three times at once: the
    first call runs the launches directly, the second captures the CUDA graph,
    the third replays it -- all concurrently with the other threads' calls."""
    n, threads, reps = 1_000_000, 4, 3
    bases = [O.uniform01(1000 + i, n) for i in range(threads)]
    wants = [oracle_ksort(b) for b in bases]
    errors, results = [], [None] * threads
    barrier = threading.Barrier(threads)

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                src = dev(bases[i])
                x = torch.empty_like(src)
                for _ in range(reps):
                    x.copy_(src)
                    barrier.wait()
                    K.k_sort(x)
                results[i] = host(x)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    ts = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for i in range(threads):
        assert same_bits(results[i], wants[i]), i


# ---- batch offsets are validated before any write ---------------------------

@pytest.mark.parametrize("bad", ["decreasing", "negative", "past_end"])
def test_batch_invalid_offsets_rejected_untouched(bad):
    rng = np.random.default_rng(13)
    a = rng.random(60_000)
    off = {"decreasing": [0, 40_000, 30_000, 60_000], "negative": [-5, 30_000, 60_000],
           "past_end": [0, 30_000, 60_001]}[bad]
    t = dev(a)
    with pytest.raises(ValueError):
        K.k_sort_segments(t, torch.tensor(off, dtype=torch.int64, device="cuda"))
    assert same_bits(host(t), a)
    # the library is usable afterwards
    K.k_sort_segments(t, torch.tensor([0, 30_000, 60_000], dtype=torch.int64, device="cuda"))
    got = host(t)
    assert same_bits(got[:30_000], np.sort(a[:30_000])) and same_bits(got[30_000:], np.sort(a[30_000:]))


# ---- the reference's KeyArray (list[float]) path -------------------------------------------

def test_list_keyarray_path_bitexact_and_errors():
    base = O.uniform01(20260816, 200_000)
    a = base.tolist()
    K.k_sort(a)
    assert isinstance(a, list) and len(a) == 200_000
    assert same_bits(np.array(a), oracle_ksort(base))
    b = base.tolist()
    K.heap_sort(b)
    h = base.copy()
    O.heap_sort(h)
    assert same_bits(np.array(b), h)
    # NaN: the reference's error, the list untouched (sort_core.py:178)
    c = base[:1000].tolist()
    c[777] = float("nan")
    before = list(c)
    with pytest.raises(K.NonFiniteKeyError, match="key at index 777 is nan; keys must be finite"):
        K.k_sort(c)
    assert c[:777] == before[:777] and c[778:] == before[778:]
    # mixed signed zeros through heap_sort's list path: the reference heap sort's bytes
    d = [0.0, -0.0, 0.5, -0.0, 0.0, -1.0, 0.0]
    want = np.array(d)
    O.heap_sort(want)
    K.heap_sort(d)
    assert same_bits(np.array(d), want)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_tensor_on_non_current_device():
    x = K.generate_device(300_000, 5).to("cuda:1")
    want = torch.sort(x).values
    with torch.cuda.device(0):
        K.k_sort(x)
    assert torch.equal(x, want)


@pytest.mark.parametrize("kind", ["presorted", "reversed", "organ", "uniform01"])
def test_device_resident_recursion_one_sync(kind):
    """The reference's worklist (sort_core.py:182-198) runs on the device: once a
    call's schedule is a cached graph, inputs needing extra global passes and
    leaf launches (presorted, reversed, organ-pipe: the reference's adversarial
    shapes, tests/test_sort_core.py:163-177) finish behind ONE host wait."""
    n = 1_000_000
    base = np.sort(O.uniform01(20260816, n))
    if kind == "reversed":
        base = base[::-1].copy()
    elif kind == "organ":
        base = np.concatenate([base[0::2], base[1::2][::-1]])
    elif kind == "uniform01":
        base = O.uniform01(20260816, n)
    want = np.sort(base)
    p = dev(base)
    t = torch.empty_like(p)
    for call in range(3):   # eager, capture, replay
        t.copy_(p)
        K.k_sort(t)
        assert same_bits(host(t), want), (kind, call)
        if call >= 1:
            assert K.last_stats.host_syncs == 1, (kind, call, K.last_stats)
    if kind != "uniform01":
        assert K.last_stats.levels > 2, K.last_stats


def test_device_loop_recaptured_when_a_cached_schedule_falls_short():
    """A buffer set first sorted with uniform keys gets a graph without the
    device loop; a presorted input on the same buffers then runs the host loop
    once (correct output), and the next call recaptures with the loop."""
    n = 1_000_000
    uni = dev(O.uniform01(7, n))
    pre = torch.sort(uni).values
    t = torch.empty_like(uni)
    for _ in range(3):
        t.copy_(uni)
        K.k_sort(t)
        assert torch.equal(t, pre)
    syncs = []
    for _ in range(3):
        t.copy_(pre)
        K.k_sort(t)
        assert torch.equal(t, pre)
        syncs.append(K.last_stats.host_syncs)
    assert syncs[-1] == 1 and syncs[-2] == 1, syncs
