"""Device twin of the reference workload generator (workload.py:43-121).

``generate_device(n, seed, kind)`` fills a CUDA float64 tensor with exactly the
bits ``sortlab.workload.generate(WorkloadSpec(n, seed))`` produces
(counter-based splitmix64, ``(u >> 11) * 2**-53``), without host generation or
an H2D copy.  ``kind="dup256"`` is BASELINE.json configs[4] (k/256 with
k = u >> 56 on the same stream).
"""
from __future__ import annotations

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
