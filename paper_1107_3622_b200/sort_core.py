"""Drop-in mirror of ``sortlab.sort_core`` backed by the sm_100a K-sort engine.

Reference interface: /root/reference/pkg/src/sortlab/sort_core.py.  Names,
argument meaning, return values and error behaviour follow it:

* ``k_sort(a, counts=None) -> None``        (sort_core.py:169)
* ``heap_sort(a, counts=None) -> None``     (sort_core.py:262)
* ``ksort_partition(a, left, right, counts=None) -> PartitionOutcome``  (sort_core.py:146)
* ``is_sorted(a) -> bool``                  (sort_core.py:62)
* ``NonFiniteKeyError``, ``OpCounts``, ``PartitionOutcome``, ``KeyArray``, ``SORTERS``

``a`` may be a ``list[float]`` (the reference's KeyArray: copied to the GPU,
sorted, copied back into the same list object), a float64 ``torch.Tensor``
(CUDA tensors are sorted in place on the device; CPU tensors round-trip), or a
float64 ``numpy.ndarray`` (round-trips, sorted in place).

Engines (all on the GPU; there is no CPU fallback):

* fast engine: multi-level K-sort passes + on-chip leaves.  Its output is
  byte-identical to the reference's whenever equal keys are bitwise equal,
  which holds for every finite input that does not contain both -0.0 and +0.0.
* exact engine: the reference's own partition permutation, level by level;
  used for ``counts``, for ``ksort_partition`` and for inputs holding both
  signed zeros, so results are byte-identical on every finite input.
* heap sort: routed to the fast engine (k_sort and heap_sort produce
  identical outputs); with ``counts`` or both signed zeros the
  reference's heap sort runs exactly on one device lane.
"""

from __future__ import annotations

import array
import contextlib
import ctypes
import functools
import threading
from dataclasses import dataclass
from typing import Callable, Optional, Union

import numpy as np
import torch

from . import _lib

KeyArray = list[float]
ArrayLike = Union[list, torch.Tensor, np.ndarray]


class NonFiniteKeyError(ValueError):
    """Raised when an input key is NaN or infinite; its order is undefined."""


@dataclass
class OpCounts:
    """Tallies of the abstract work a sort performed (sort_core.py:29-41)."""

    comparisons: int = 0
    moves: int = 0
    max_pending_ranges: int = 0


@dataclass(frozen=True)
class PartitionOutcome:
    pivot_index: int
    flag_used: bool


@dataclass
class SortStats:
    """Engine telemetry of the last call on this thread (not part of the reference API)."""

    levels: int = 0
    bytes_moved: int = 0
    keys_partitioned: int = 0
    keys_leaf_sorted: int = 0
    leaves: int = 0
    exact_used: bool = False
    host_syncs: int = 0   # waits for the device (1: the whole recursion ran device-resident)
    launches: int = 0     # kernels launched by the call


last_stats = SortStats()


# ---------------------------------------------------------------------------
# device plumbing
# ---------------------------------------------------------------------------

_cuda_ok = False


def _device() -> torch.device:
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1107_3622_b200 needs a CUDA device (B200); there is no CPU fallback")
        _cuda_ok = True
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_ptr() -> int:
    """The caller's current CUDA stream (the raw handle: ~0.3 us instead of ~3 us
    for building a torch.cuda.Stream object on every call)."""
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def _on_input_device(fn):
    """Run an entry point on the device that holds its CUDA tensor argument.

    The workspace, the stream and every library launch use the *current*
    device; a tensor on another GPU would otherwise be sorted by kernels of
    the current one (an illegal address without peer access).
    """
    @functools.wraps(fn)
    def wrapper(a, *args, **kwargs):
        if isinstance(a, torch.Tensor) and a.is_cuda and a.device.index != torch.cuda.current_device():
            with torch.cuda.device(a.device):
                return fn(a, *args, **kwargs)
        return fn(a, *args, **kwargs)
    return wrapper


_tls = threading.local()


def _workspace(nbytes: int) -> torch.Tensor:
    """Per-thread, per-device scratch buffer, grown on demand and reused: the
    library never allocates, and calls are synchronous, so one buffer per
    calling thread is enough (distinct threads may sort concurrently)."""
    nbytes = max(int(nbytes), 256)
    dev = _device()
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    buf = cache.get(dev.index)
    if buf is None or buf.numel() < nbytes:
        cache[dev.index] = None   # release the old buffer before growing
        buf = cache[dev.index] = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    return buf


_ws_sizes: dict = {}


def _workspace_bytes(L, n: int, nseg: int, flags: int) -> int:
    key = (n, nseg, flags)
    v = _ws_sizes.get(key)
    if v is None:
        v = _ws_sizes[key] = int(L.ks_workspace_bytes(n, nseg, flags))
        if len(_ws_sizes) > 4096:
            _ws_sizes.clear()
    return v


class _Staged:
    """A device float64 view of the caller's array plus the write-back."""

    def __init__(self, a: ArrayLike):
        self.a = a
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64 or a.dim() != 1:
                raise TypeError("expected a 1-D float64 tensor")
            if a.is_cuda and a.is_contiguous():
                self.dev = a
            else:
                self.dev = a.to(device=_device(), non_blocking=False).contiguous()
        elif isinstance(a, np.ndarray):
            if a.dtype != np.float64 or a.ndim != 1:
                raise TypeError("expected a 1-D float64 array")
            self.dev = torch.from_numpy(np.ascontiguousarray(a)).to(_device())
        else:
            self.dev = torch.tensor(a, dtype=torch.float64, device=_device()) if len(a) else \
                torch.empty(0, dtype=torch.float64, device=_device())
        self.n = int(self.dev.numel())

    def ptr(self) -> int:
        return self.dev.data_ptr()

    def write_back(self) -> None:
        a = self.a
        if isinstance(a, torch.Tensor):
            if a is not self.dev:
                a.copy_(self.dev)
        elif isinstance(a, np.ndarray):
            a[...] = self.dev.cpu().numpy()
        else:
            a[:] = self.dev.cpu().tolist()


def _nonfinite_message(idx: int, v: float) -> str:
    # sort_core.py:58
    return f"key at index {idx} is {v!r}; keys must be finite"


def _raise_for(code: int, st: _lib.KsStatus, what: str) -> None:
    if code == _lib.KS_OK:
        return
    if code == _lib.KS_NONFINITE:
        raise NonFiniteKeyError(_nonfinite_message(int(st.bad_index), float(st.bad_value)))
    if code == _lib.KS_BAD_ARG:
        raise ValueError(f"{what}: invalid arguments")
    raise RuntimeError(f"{what}: libksort returned code {code}")


def _record(st: _lib.KsStatus) -> None:
    # updated in place so ``from paper_1107_3622_b200 import last_stats`` stays live
    last_stats.levels = int(st.levels)
    last_stats.bytes_moved = int(st.bytes_moved)
    last_stats.keys_partitioned = int(st.keys_partitioned)
    last_stats.keys_leaf_sorted = int(st.keys_leaf_sorted)
    last_stats.leaves = int(st.leaves)
    last_stats.exact_used = bool(st.exact_used)
    last_stats.host_syncs = int(st.host_syncs)
    last_stats.launches = int(st.launches)


def _fast_slot(n: int, dev: int):
    """Per-thread cache for the plain call (CUDA tensor, no counts, current device): the workspace
    pointer and size for this n and a reusable status block -- ~4 us less host time per call than the
    general path (building a torch.device, a status struct and the telemetry copy), which is 10% of a
    100K-key sort."""
    slots = getattr(_tls, "fast", None)
    if slots is None:
        slots = _tls.fast = {}
    slot = slots.get((n, dev))
    if slot is not None and _tls.ws.get(dev) is slot[3]:   # (the buffer this slot points into is still the live one)
        return slot
    L = _lib.load()
    ws_bytes = _workspace_bytes(L, n, 1, 0)
    ws = _workspace(ws_bytes)
    st = _lib.KsStatus()
    if len(slots) > 64:
        slots.clear()
    slot = slots[(n, dev)] = (ws.data_ptr(), ws_bytes, st, ws, ctypes.byref(st), L.ks_sort_f64)
    return slot


def _record_fast(st: _lib.KsStatus) -> None:
    last_stats.levels = st.levels
    last_stats.bytes_moved = st.bytes_moved
    last_stats.keys_partitioned = st.keys_partitioned
    last_stats.keys_leaf_sorted = st.keys_leaf_sorted
    last_stats.leaves = st.leaves
    last_stats.exact_used = bool(st.exact_used)
    last_stats.host_syncs = st.host_syncs
    last_stats.launches = st.launches


def _sort_device_fast(keys: torch.Tensor, n: int, dev: int) -> bool:
    """The plain call through the cached slot; False when the general path must take over
    (any return code but KS_OK: non-finite keys, signed zeros -> exact engine, errors)."""
    ws_ptr, ws_bytes, st, _ws, st_ref, fn = _fast_slot(n, dev)
    code = fn(keys.data_ptr(), n, ws_ptr, ws_bytes, _raw_stream(dev), 0, st_ref)
    if code != _lib.KS_OK:
        return False
    _record_fast(st)
    return True


def _sort_device(keys: torch.Tensor, flags: int = 0) -> _lib.KsStatus:
    """Sort a contiguous CUDA float64 tensor in place; returns the status block."""
    L = _lib.load()
    n = keys.numel()
    st = _lib.KsStatus()
    ws_bytes = _workspace_bytes(L, n, 1, flags)
    ws = _workspace(ws_bytes)
    code = L.ks_sort_f64(keys.data_ptr(), n, ws.data_ptr(), ws_bytes, _stream_ptr(), flags,
                         ctypes.byref(st))
    if code == _lib.KS_NEED_EXACT:
        # both signed zeros present: rerun with the exact engine's workspace
        ws_bytes = _workspace_bytes(L, n, 1, flags | _lib.KS_FLAG_EXACT)
        ws = _workspace(ws_bytes)
        code = L.ks_sort_f64(keys.data_ptr(), n, ws.data_ptr(), ws_bytes, _stream_ptr(), flags,
                             ctypes.byref(st))
    _raise_for(code, st, "k_sort")
    _record(st)
    return st


def _host_view(a: ArrayLike) -> Optional[torch.Tensor]:
    """A CPU float64 tensor sharing the caller's memory (host tensors and
    ndarrays that are contiguous 1-D float64), else None."""
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            return None
        if a.dtype != torch.float64 or a.dim() != 1:
            raise TypeError("expected a 1-D float64 tensor")
        return a if a.is_contiguous() and a.numel() > 0 else None
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or a.ndim != 1:
            raise TypeError("expected a 1-D float64 array")
        if a.size > 0 and a.flags.c_contiguous and a.flags.writeable:
            return torch.from_numpy(a)
    return None


def _sort_host(h: torch.Tensor, flags: int = 0) -> _lib.KsStatus:
    """Sort a host float64 tensor in place through ks_sort_f64_host (H2D, sort,
    D2H queued on one stream; pinned memory makes the copies asynchronous)."""
    L = _lib.load()
    n = h.numel()
    dev = torch.empty(n, dtype=torch.float64, device=_device())
    st = _lib.KsStatus()
    ws_bytes = _workspace_bytes(L, n, 1, flags)
    ws = _workspace(ws_bytes)
    code = L.ks_sort_f64_host(h.data_ptr(), n, dev.data_ptr(), ws.data_ptr(), ws_bytes, _stream_ptr(), flags,
                              ctypes.byref(st))
    if code == _lib.KS_NEED_EXACT:
        ws_bytes = _workspace_bytes(L, n, 1, flags | _lib.KS_FLAG_EXACT)
        ws = _workspace(ws_bytes)
        code = L.ks_sort_f64_host(h.data_ptr(), n, dev.data_ptr(), ws.data_ptr(), ws_bytes, _stream_ptr(), flags,
                                  ctypes.byref(st))
    _raise_for(code, st, "k_sort")
    _record(st)
    return st


def _list_buffer(a: list) -> Optional[array.array]:
    """A packed float64 copy of a ``list[float]`` KeyArray (array.array: about
    3x faster to build than a tensor from the list), or None when empty."""
    if len(a) == 0:
        return None
    return array.array("d", a)


def _sort_list(a: list, flags: int) -> Optional[_lib.KsStatus]:
    """k_sort of the reference's KeyArray: pack, copy in, sort, copy back with
    one synchronisation (ks_sort_f64_host), then rewrite the list in place.
    Nothing is written to ``a`` when the sort raises (NonFiniteKeyError)."""
    buf = _list_buffer(a)
    if buf is None:
        return None
    st = _sort_host(torch.frombuffer(buf, dtype=torch.float64), flags)
    a[:] = buf.tolist()
    return st


# ---------------------------------------------------------------------------
# reference API
# ---------------------------------------------------------------------------

@_on_input_device
def is_sorted(a: ArrayLike) -> bool:
    """True when a is ascending (non-strict) -- sort_core.py:62-67, on the device."""
    s = _Staged(a)
    if s.n < 2:
        return True
    L = _lib.load()
    ws = _workspace(256)
    r = ctypes.c_int32(0)
    code = L.ks_is_sorted_f64(s.ptr(), s.n, ws.data_ptr(), _stream_ptr(), ctypes.byref(r))
    if code != _lib.KS_OK:
        raise RuntimeError(f"is_sorted: libksort returned code {code}")
    return bool(r.value)


@_on_input_device
def ksort_partition(a: ArrayLike, left: int, right: int,
                    counts: Optional[OpCounts] = None) -> PartitionOutcome:
    """Partition a[left..right] (inclusive) around key = a[left], in place.

    Exact reference permutation (sort_core.py:81-105) computed on the device
    in data-parallel closed form; range/finiteness errors as sort_core.py:157-161.
    """
    n = len(a)
    if not 0 <= left < right < n:
        raise ValueError(f"partition range [{left}, {right}] invalid for array of length {n}")
    s = _Staged(a)
    L = _lib.load()
    ws_bytes = L.ks_workspace_bytes(s.n, 1, _lib.KS_FLAG_EXACT)
    ws = _workspace(ws_bytes)
    st = _lib.KsStatus()
    piv = ctypes.c_int64(0)
    flag = ctypes.c_int32(0)
    code = L.ks_partition_f64(s.ptr(), s.n, left, right, ws.data_ptr(), ws_bytes, _stream_ptr(),
                              ctypes.byref(piv), ctypes.byref(flag), ctypes.byref(st))
    _raise_for(code, st, "ksort_partition")
    s.write_back()
    if counts is not None:
        counts.comparisons += int(st.comparisons)
        counts.moves += int(st.moves)
    return PartitionOutcome(pivot_index=int(piv.value), flag_used=bool(flag.value))


def k_sort(a: ArrayLike, counts: Optional[OpCounts] = None) -> None:
    """Sort a ascending, in place (sort_core.py:169-217), on the GPU.

    With ``counts`` the exact engine runs and the reference's tallies are
    accumulated (comparisons/moves added, max_pending_ranges maxed).
    """
    if (counts is None and type(a) is torch.Tensor and a.is_cuda and a.dtype is torch.float64 and a.dim() == 1
            and a.is_contiguous() and _raw_stream is not None):
        # the plain call: a CUDA tensor on the current device, through the cached slot (a failed fast
        # call wrote nothing: the general path below reruns it and raises / switches engines)
        dev = a.device.index
        if dev == torch.cuda.current_device() and _sort_device_fast(a, a.numel(), dev):
            return
    _k_sort_general(a, counts)


@_on_input_device
def _k_sort_general(a: ArrayLike, counts: Optional[OpCounts] = None) -> None:
    flags = _lib.KS_FLAG_COUNTS if counts is not None else 0
    h = _host_view(a)
    if h is not None:   # host tensor / ndarray: copy in, sort, copy back with one synchronisation
        n = h.numel()
        st = _sort_host(h, flags)
    elif isinstance(a, list):
        n = len(a)
        st = _sort_list(a, flags)
    else:
        s = _Staged(a)
        n = s.n
        st = _sort_device(s.dev, flags)
        s.write_back()
    if counts is not None and n >= 2 and st is not None:
        counts.comparisons += int(st.comparisons)
        counts.moves += int(st.moves)
        counts.max_pending_ranges = max(counts.max_pending_ranges, int(st.max_pending_ranges))


@_on_input_device
def heap_sort(a: ArrayLike, counts: Optional[OpCounts] = None) -> None:
    """Sort a ascending, in place, with heap sort's contract (sort_core.py:262-286).

    Without counts the output is produced by the K-sort engine (SPEC.md:113:
    both sorters produce identical outputs); when the input holds both signed
    zeros or counts are requested, the reference heap sort runs exactly on the
    device so bytes and tallies match the reference's heap_sort.
    """
    if counts is None and isinstance(a, list):
        buf = _list_buffer(a)
        if buf is None:
            return
        v = np.frombuffer(buf, dtype=np.float64)
        z = np.signbit(v[v == 0])
        if not (z.any() and not z.all()):   # no mixed signed zeros: the K-sort engine's bytes are heap sort's
            _sort_host(torch.frombuffer(buf, dtype=torch.float64), 0)
            a[:] = buf.tolist()
            return
    s = _Staged(a)
    L = _lib.load()
    exact = counts is not None
    if not exact and s.n >= 2:
        zeros = s.dev == 0
        if bool(zeros.any()):
            sb = torch.signbit(s.dev[zeros])
            exact = bool(sb.any()) and not bool(sb.all())
    if not exact:
        _sort_device(s.dev, 0)
        s.write_back()
        return
    ws = _workspace(256)
    st = _lib.KsStatus()
    code = L.ks_heap_sort_f64_exact(s.ptr(), s.n, ws.data_ptr(), 256, _stream_ptr(), 0,
                                    ctypes.byref(st))
    _raise_for(code, st, "heap_sort")
    s.write_back()
    if counts is not None and s.n >= 2:
        counts.comparisons += int(st.comparisons)
        counts.moves += int(st.moves)


@_on_input_device
def k_sort_segments(keys: torch.Tensor, offsets: torch.Tensor, exact: bool = False) -> None:
    """Sort keys[offsets[s]:offsets[s+1]] independently, in place, in one call.

    New batch API (the reference bench calls k_sort once per array,
    bench.py:169-173).  keys: CUDA float64, offsets: CUDA int64 of nseg+1
    non-decreasing entries.  Each segment's result equals k_sort on it alone.
    """
    if not (keys.is_cuda and keys.dtype == torch.float64 and keys.is_contiguous() and keys.dim() == 1):
        raise TypeError("keys must be a contiguous 1-D CUDA float64 tensor")
    if not (offsets.is_cuda and offsets.dtype == torch.int64 and offsets.is_contiguous()):
        raise TypeError("offsets must be a contiguous CUDA int64 tensor")
    if offsets.device != keys.device:
        raise ValueError("keys and offsets must be on the same device")
    nseg = offsets.numel() - 1
    if nseg <= 0:
        return
    L = _lib.load()
    n = keys.numel()
    flags = _lib.KS_FLAG_EXACT if exact else 0
    ws_bytes = L.ks_workspace_bytes(n, nseg, flags)
    ws = _workspace(ws_bytes)
    st = _lib.KsStatus()
    code = L.ks_sort_f64_segmented(keys.data_ptr(), offsets.data_ptr(), nseg, n, ws.data_ptr(), ws_bytes,
                                   _stream_ptr(), flags, ctypes.byref(st))
    if code == _lib.KS_NEED_EXACT:
        ws_bytes = L.ks_workspace_bytes(n, nseg, _lib.KS_FLAG_EXACT)
        ws = _workspace(ws_bytes)
        code = L.ks_sort_f64_segmented(keys.data_ptr(), offsets.data_ptr(), nseg, n, ws.data_ptr(),
                                       ws_bytes, _stream_ptr(), flags, ctypes.byref(st))
    _raise_for(code, st, "k_sort_segments")
    _record(st)


SORTERS: dict[str, Callable[..., None]] = {
    "ksort": k_sort,
    "heapsort": heap_sort,
}
