"""paper_1107_3622_b200 -- K-sort (arXiv:1107.3622) on one B200, sm_100a CUDA.

Drop-in for the hot path of the reference package ``sortlab``: the sort
entry points of ``sortlab.sort_core`` (k_sort, heap_sort, ksort_partition,
is_sorted, SORTERS, OpCounts, PartitionOutcome, NonFiniteKeyError) backed by
libksort.so (include/ksort.h).  See DESIGN.md.
"""

from .sort_core import (  # noqa: F401
    SORTERS,
    KeyArray,
    NonFiniteKeyError,
    OpCounts,
    PartitionOutcome,
    SortStats,
    heap_sort,
    is_sorted,
    k_sort,
    k_sort_segments,
    ksort_partition,
    last_stats,
)
from .workload import generate_device, read_binary, read_text, write_binary, write_text  # noqa: F401

__all__ = [
    "SORTERS", "KeyArray", "NonFiniteKeyError", "OpCounts", "PartitionOutcome", "SortStats",
    "heap_sort", "is_sorted", "k_sort", "k_sort_segments", "ksort_partition", "generate_device", "last_stats",
    "read_binary", "write_binary", "read_text", "write_text",
]
