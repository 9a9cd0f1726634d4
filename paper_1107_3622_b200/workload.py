"""Device twin of the reference workload generator (workload.py:43-121).

``generate_device(n, seed, kind)`` fills a CUDA float64 tensor with exactly the
bits ``sortlab.workload.generate(WorkloadSpec(n, seed))`` produces
(counter-based splitmix64, ``(u >> 11) * 2**-53``), without host generation or
an H2D copy.  ``kind="dup256"`` is BASELINE.json configs[4] (k/256 with
k = u >> 56 on the same stream).
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib

_KINDS = {"uniform01": 0, "dup256": 1}


def generate_device(n: int, seed: int, kind: str = "uniform01",
                    out: torch.Tensor | None = None) -> torch.Tensor:
    if kind not in _KINDS:
        raise ValueError(f"unknown workload kind {kind!r}; choose from {tuple(_KINDS)}")
    if n < 0:
        raise ValueError(f"n must be nonnegative, got {n}")
    if not torch.cuda.is_available():
        raise RuntimeError("generate_device needs a CUDA device")
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device="cuda")
    L = _lib.load()
    code = L.ks_generate_f64(out.data_ptr(), n, seed & 0xFFFFFFFFFFFFFFFF, _KINDS[kind],
                             torch.cuda.current_stream().cuda_stream)
    if code != _lib.KS_OK:
        raise RuntimeError(f"ks_generate_f64 returned {code}")
    return out


# ---------------------------------------------------------------------------
# Array files straight to / from the device.
# Same formats, validation order and messages as the reference
# (workload.py:129-174): binary = 8-byte little-endian count + count
# little-endian float64; text = one repr() per line.  Reads land in a pinned
# host buffer and go to the GPU in one copy; the finiteness check
# (workload._require_finite, :129-134) runs on the device.
# ---------------------------------------------------------------------------
import os
import struct

import numpy as np


def _nonfinite_error(source: str, t: int, v: float):
    from .sort_core import NonFiniteKeyError
    return NonFiniteKeyError(f"{source}: value at position {t} is {v!r}; keys must be finite")


def _require_finite_device(t: torch.Tensor, source: str) -> torch.Tensor:
    L = _lib.load()
    ws = torch.empty(256, dtype=torch.uint8, device=t.device)
    bad = ctypes.c_int64(-1)
    code = L.ks_first_nonfinite_f64(t.data_ptr(), t.numel(), ws.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream, ctypes.byref(bad))
    if code != _lib.KS_OK:
        raise RuntimeError(f"ks_first_nonfinite_f64 returned {code}")
    if bad.value >= 0:
        raise _nonfinite_error(source, int(bad.value), float(t[bad.value].item()))
    return t


def _host_f64(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        return a.detach().to("cpu", torch.float64).contiguous().numpy()
    return np.asarray(a, dtype=np.float64)


def write_binary(path, a) -> None:
    """workload.write_binary (workload.py:137-140) for a list, ndarray or tensor."""
    x = _host_f64(a)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", x.size))
        fh.write(x.astype("<f8", copy=False).tobytes())


def read_binary(path) -> torch.Tensor:
    """workload.read_binary (workload.py:143-153), returning a CUDA float64 tensor."""
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(8)
        if len(head) < 8:
            raise ValueError(f"{path}: truncated header, {len(head)} bytes")
        (count,) = struct.unpack("<Q", head)
        expected = 8 + 8 * count
        if size != expected:
            raise ValueError(f"{path}: expected {expected} bytes for {count} values, found {size}")
        if not torch.cuda.is_available():
            raise RuntimeError("read_binary needs a CUDA device; there is no CPU fallback")
        host = torch.empty(count, dtype=torch.float64, pin_memory=True)
        if count:
            view = host.numpy().view(np.uint8)
            got = fh.readinto(memoryview(view))
            if got != 8 * count:
                raise ValueError(f"{path}: expected {expected} bytes for {count} values, found {8 + got}")
    if host.numpy().dtype.byteorder == ">":   # (big-endian hosts only)
        host.copy_(torch.from_numpy(host.numpy().byteswap()))
    dev = host.to("cuda", non_blocking=True)
    return _require_finite_device(dev, str(path))


def write_text(path, a) -> None:
    """workload.write_text (workload.py:156-160): one repr() per line."""
    x = _host_f64(a)
    with open(path, "w", encoding="ascii") as fh:
        for v in x.tolist():
            fh.write(repr(v))
            fh.write("\n")


def read_text(path) -> torch.Tensor:
    """workload.read_text (workload.py:163-174), returning a CUDA float64 tensor."""
    values = []
    with open(path, "r", encoding="ascii") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                values.append(float(line))
            except ValueError as exc:
                raise ValueError(f"{path}:{lineno}: not a float: {line!r}") from exc
    if not torch.cuda.is_available():
        raise RuntimeError("read_text needs a CUDA device; there is no CPU fallback")
    dev = torch.tensor(values, dtype=torch.float64).pin_memory().to("cuda", non_blocking=True)
    return _require_finite_device(dev, str(path))
