"""ctypes binding of libksort.so (include/ksort.h).

The product path has no fallback: if the library or a CUDA device is missing,
every entry point raises.  Nothing here imports the test oracle.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KSORT_LIB") or os.path.join(_HERE, "libksort.so")   # KSORT_LIB: experiment builds

KS_OK = 0
KS_NONFINITE = 1
KS_BAD_ARG = 2
KS_CUDA_ERROR = 3
KS_WORKSPACE_SMALL = 4
KS_NOT_SUPPORTED = 5
KS_NEED_EXACT = 6

KS_FLAG_EXACT = 1
KS_FLAG_COUNTS = 2
KS_FLAG_PROFILE = 4
PHASES = ("gate", "pivots", "count", "scan", "scatter", "plan", "leaf", "local")

EXPORTED = (
    "ks_workspace_bytes", "ks_sort_f64", "ks_sort_f64_host", "ks_sort_f64_segmented", "ks_partition_f64",
    "ks_heap_sort_f64_exact", "ks_is_sorted_f64", "ks_first_nonfinite_f64", "ks_generate_f64", "ks_version",
)


class KsStatus(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("levels", ctypes.c_int32),
        ("bad_index", ctypes.c_int64),
        ("bad_value", ctypes.c_double),
        ("comparisons", ctypes.c_uint64),
        ("moves", ctypes.c_uint64),
        ("max_pending_ranges", ctypes.c_uint64),
        ("bytes_moved", ctypes.c_uint64),
        ("keys_partitioned", ctypes.c_uint64),
        ("keys_leaf_sorted", ctypes.c_uint64),
        ("leaves", ctypes.c_int64),
        ("exact_used", ctypes.c_int32),
        ("launches", ctypes.c_int32),
        ("phase_ms", ctypes.c_float * 8),
        ("phase_launches", ctypes.c_int32 * 8),
        ("phase_bytes", ctypes.c_uint64 * 8),
        ("host_syncs", ctypes.c_int32),
        ("reserved_", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = list(v) if not isinstance(v, (int, float)) else v
        return d


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libksort.so once; raise loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build the CUDA engine first "
            "(python -m paper_1107_3622_b200.build); there is no CPU fallback")
    L = ctypes.CDLL(path)
    vp, i64, u32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
    st = ctypes.POINTER(KsStatus)
    L.ks_workspace_bytes.argtypes = [i64, i64, u32]
    L.ks_workspace_bytes.restype = sz
    L.ks_sort_f64.argtypes = [vp, i64, vp, sz, vp, u32, st]
    L.ks_sort_f64.restype = ctypes.c_int
    L.ks_sort_f64_host.argtypes = [vp, i64, vp, vp, sz, vp, u32, st]
    L.ks_sort_f64_host.restype = ctypes.c_int
    L.ks_sort_f64_segmented.argtypes = [vp, vp, i64, i64, vp, sz, vp, u32, st]
    L.ks_sort_f64_segmented.restype = ctypes.c_int
    L.ks_partition_f64.argtypes = [vp, i64, i64, i64, vp, sz, vp, ctypes.POINTER(i64),
                                   ctypes.POINTER(ctypes.c_int32), st]
    L.ks_partition_f64.restype = ctypes.c_int
    L.ks_heap_sort_f64_exact.argtypes = [vp, i64, vp, sz, vp, u32, st]
    L.ks_heap_sort_f64_exact.restype = ctypes.c_int
    L.ks_is_sorted_f64.argtypes = [vp, i64, vp, vp, ctypes.POINTER(ctypes.c_int32)]
    L.ks_is_sorted_f64.restype = ctypes.c_int
    L.ks_first_nonfinite_f64.argtypes = [vp, i64, vp, vp, ctypes.POINTER(ctypes.c_int64)]
    L.ks_first_nonfinite_f64.restype = ctypes.c_int
    L.ks_generate_f64.argtypes = [vp, i64, ctypes.c_uint64, ctypes.c_int32, vp]
    L.ks_generate_f64.restype = ctypes.c_int
    L.ks_version.argtypes = []
    L.ks_version.restype = ctypes.c_char_p
    _lib = L
    return L
