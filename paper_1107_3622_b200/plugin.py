"""Registration of the B200 sorters into the reference's plugin registry.

The reference's plug-in point for this path is ``sortlab.sort_core.SORTERS``
(sort_core.py:289-292), a ``name -> sorter(a, counts=None) -> None`` map read
by ``bench.run_cell`` (bench.py:138-155), ``cli.cmd_sort`` (cli.py:99-104) and
the CLI's argparse choices (built from ``sorted(SORTERS)`` when the parser is
built, cli.py:258,269).  ``bench`` and ``cli`` import the same dict object, so
one registration is seen everywhere -- provided it happens before
``cli.build_parser()`` runs; ``BenchConfig.algorithms`` defaults to the keys
captured at import time (bench.py:93), so pass ``algorithms=`` explicitly.
"""
from __future__ import annotations

from typing import Callable, MutableMapping, Optional

from .sort_core import heap_sort, k_sort

NAMES = {"ksort": k_sort, "heapsort": heap_sort}


def register(sorters: Optional[MutableMapping[str, Callable[..., None]]] = None, *, suffix: str = "_b200",
             replace: bool = False) -> dict:
    """Add the GPU sorters to ``sorters`` (default: ``sortlab.sort_core.SORTERS``).

    ``replace=False`` adds ``ksort<suffix>`` / ``heapsort<suffix>`` next to the
    reference's own entries (A/B runs through the reference harness);
    ``replace=True`` rebinds ``ksort`` / ``heapsort`` themselves (drop-in).
    Returns the names registered.
    """
    if sorters is None:
        from sortlab.sort_core import SORTERS as sorters  # the reference must be importable
    added = {}
    for name, fn in NAMES.items():
        key = name if replace else name + suffix
        sorters[key] = fn
        added[key] = fn
    return added
