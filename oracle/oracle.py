"""CPU oracle for the K-sort hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and only
as the checker / the timed CPU baseline.  The product package
``paper_1107_3622_b200`` never imports it.

Two layers:

* ``libksort_oracle.so`` (``ksort_oracle.c``): a line-by-line C restatement of
  ``sort_core._partition`` / ``k_sort`` / ``heap_sort`` and ``workload``'s
  splitmix64 (file:line cited in the C source).  Fast enough for 1e7 keys.
* pure-Python restatements of the exact K-sort partition in data-parallel
  closed form and of a level-order (BFS) K-sort driver,
  used to check the device's level-synchronous exact mode level by level.

Parity status: pinned.  ``tests/golden/*.json`` hold outputs of the reference
itself (generated in the build container by ``tests/golden/make_golden.py``)
and ``tests/test_oracle.py`` checks this module against them.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libksort_oracle.so")


class _Counts(ctypes.Structure):
    _fields_ = [
        ("comparisons", ctypes.c_uint64),
        ("moves", ctypes.c_uint64),
        ("max_pending_ranges", ctypes.c_uint64),
    ]


@dataclass
class Counts:
    comparisons: int = 0
    moves: int = 0
    max_pending_ranges: int = 0


def build() -> str:
    """Compile the C restatement (make -C oracle); returns the .so path."""
    src = os.path.join(_HERE, "ksort_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        path = _LIB_PATH if os.path.exists(_LIB_PATH) else build()
        L = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        cp = ctypes.POINTER(_Counts)
        L.ko_check_finite.argtypes = [dp, ctypes.c_int64]
        L.ko_check_finite.restype = ctypes.c_int64
        L.ko_is_sorted.argtypes = [dp, ctypes.c_int64]
        L.ko_is_sorted.restype = ctypes.c_int
        L.ko_partition.argtypes = [dp, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.POINTER(ctypes.c_int), cp]
        L.ko_partition.restype = ctypes.c_int64
        L.ko_k_sort.argtypes = [dp, ctypes.c_int64, cp]
        L.ko_k_sort.restype = None
        L.ko_heap_sort.argtypes = [dp, ctypes.c_int64, cp]
        L.ko_heap_sort.restype = None
        L.ko_mix64.argtypes = [ctypes.c_uint64]
        L.ko_mix64.restype = ctypes.c_uint64
        L.ko_bulk_uint64.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
        L.ko_bulk_uint64.restype = None
        L.ko_uniform01.argtypes = [ctypes.c_uint64, ctypes.c_int64, dp]
        L.ko_uniform01.restype = None
        L.ko_dup256.argtypes = [ctypes.c_uint64, ctypes.c_int64, dp]
        L.ko_dup256.restype = None
        L.ko_derive_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.ko_derive_seed.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _to_counts(c: _Counts) -> Counts:
    return Counts(int(c.comparisons), int(c.moves), int(c.max_pending_ranges))


# ---- sort_core restatement (C) ------------------------------------------------

def k_sort(a: np.ndarray, counts: bool = False):
    """In-place K-sort of a float64 array (sort_core.py:169).  Returns Counts if asked."""
    c = _Counts()
    lib().ko_k_sort(_dptr(a), a.size, ctypes.byref(c) if counts else None)
    return _to_counts(c) if counts else None


def heap_sort(a: np.ndarray, counts: bool = False):
    """In-place heap sort (sort_core.py:262).  Returns Counts if asked."""
    c = _Counts()
    lib().ko_heap_sort(_dptr(a), a.size, ctypes.byref(c) if counts else None)
    return _to_counts(c) if counts else None


def partition(a: np.ndarray, left: int, right: int, counts: bool = False):
    """One K-sort partition of a[left..right] (sort_core.py:81-143).

    Returns (pivot_index, flag_used[, Counts]).
    """
    flag = ctypes.c_int(0)
    c = _Counts()
    piv = lib().ko_partition(_dptr(a), left, right, ctypes.byref(flag),
                             ctypes.byref(c) if counts else None)
    if counts:
        return int(piv), bool(flag.value), _to_counts(c)
    return int(piv), bool(flag.value)


def check_finite(a: np.ndarray) -> int:
    return int(lib().ko_check_finite(_dptr(a), a.size))


def is_sorted(a: np.ndarray) -> bool:
    return bool(lib().ko_is_sorted(_dptr(a), a.size))


# ---- workload restatement (C) ---------------------------------------------------

def mix64(x: int) -> int:
    return int(lib().ko_mix64(x & 0xFFFFFFFFFFFFFFFF))


def bulk_uint64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().ko_bulk_uint64(seed & 0xFFFFFFFFFFFFFFFF, count,
                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return out


def uniform01(seed: int, count: int) -> np.ndarray:
    """workload.generate(WorkloadSpec(count, seed)) as a float64 array."""
    out = np.empty(count, dtype=np.float64)
    lib().ko_uniform01(seed & 0xFFFFFFFFFFFFFFFF, count, _dptr(out))
    return out


def dup256(seed: int, count: int) -> np.ndarray:
    """BASELINE configs[4]: k/256, k = (splitmix64 output >> 56)."""
    out = np.empty(count, dtype=np.float64)
    lib().ko_dup256(seed & 0xFFFFFFFFFFFFFFFF, count, _dptr(out))
    return out


def derive_seed(seed: int, index: int, stream: int = 0) -> int:
    if index < 0 or stream < 0:
        raise ValueError("index and stream must be nonnegative")
    return int(lib().ko_derive_seed(seed & 0xFFFFFFFFFFFFFFFF, index, stream))


# ---- data-parallel restatements (pure Python, small cases) -----------------------

def partition_closed_form(a, left: int, right: int):
    """Exact K-sort partition in closed form.

    Same output permutation as sort_core.py:81-105 but every destination is a
    function of prefix counts, which is what the device exact mode computes.
    Returns (new list, pivot_index, flag_used).
    """
    key = a[left]
    nl = sum(1 for p in range(left + 1, right + 1) if a[p] < key)
    piv = left + nl
    B = [p for p in range(left + 1, piv + 1) if not (a[p] < key)]     # ge in A, increasing
    G = [q for q in range(right, piv, -1) if a[q] < key]              # lt in Z, decreasing
    c = len(B)
    out = list(a)
    rb = 0
    for p in range(left + 1, piv + 1):
        if a[p] < key:
            out[p - 1] = a[p]
        else:
            out[p - 1] = a[G[rb]]
            rb += 1
    out[piv] = key
    e = piv + 1
    if c >= 1:
        for k in range(c - 1):
            out[G[k]] = a[B[k + 1]]
        if not (a[e] < key):
            out[G[c - 1]] = a[e]
        out[e] = a[B[0]]
    return out, piv, piv < right


def k_sort_levels(a):
    """Level-order (BFS) K-sort driver over the exact partition.

    Partitions of disjoint segments commute, so processing the reference's
    recursion tree level by level yields the same final array and the same
    comparison/move totals as the LIFO driver (sort_core.py:182-198).
    Returns (final list, [array state after each level]).
    """
    a = list(a)
    n = len(a)
    states = []
    level = [(0, n - 1)] if n >= 2 else []
    while level:
        nxt = []
        for left, right in level:
            a, piv, _ = partition_closed_form(a, left, right)
            if piv - left >= 2:
                nxt.append((left, piv - 1))
            if right - piv >= 2:
                nxt.append((piv + 1, right))
        states.append(list(a))
        level = nxt
    return a, states
