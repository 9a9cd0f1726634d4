"""Import the UNMODIFIED reference package installed under baseline/_ref.

    python -m pip install --no-index --no-build-isolation --no-deps \
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

(baseline/_ref is git-ignored; it travels to the GPU box with the gpurun
snapshot.)  The reference's ``sortlab/__init__.py`` imports ``figures.py``,
which needs matplotlib -- absent from this image and irrelevant to the sort
path -- so a stub module providing the one imported name (``Figure``) is
registered first (workaround 2).  Nothing in the reference
is patched.  Used by the reference arm / CPU baseline of bench.py and by
tests/test_sortlab_plugin.py; the product package never imports it.
"""
from __future__ import annotations

import os
import sys
import types

REF_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref")


def available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "sortlab", "sort_core.py"))


def _stub_matplotlib() -> None:
    try:
        import matplotlib.figure  # noqa: F401
        return
    except ImportError:
        pass
    mpl = types.ModuleType("matplotlib")
    fig = types.ModuleType("matplotlib.figure")

    class Figure:  # never instantiated on the sort / bench / cli-sort paths
        def __init__(self, *a, **k):
            raise RuntimeError("matplotlib is not installed (figure rendering is out of scope)")

    fig.Figure = Figure
    mpl.figure = fig
    sys.modules.setdefault("matplotlib", mpl)
    sys.modules.setdefault("matplotlib.figure", fig)


def import_sortlab():
    """The reference package ``sortlab`` (whole package, stock code)."""
    if not available():
        raise ImportError(f"reference not installed under {REF_DIR}")
    _stub_matplotlib()
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import sortlab  # noqa: E402
    import sortlab.bench  # noqa: F401,E402
    import sortlab.cli  # noqa: F401,E402
    import sortlab.sort_core  # noqa: F401,E402
    import sortlab.workload  # noqa: F401,E402
    return sortlab
