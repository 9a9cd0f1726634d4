"""CPU checks of the drop-in boundary: libksort.so loads and exports every
symbol include/ksort.h declares; host-only entry points answer; the product
package refuses to run without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ksort.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ks_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1107_3622_b200 import _lib
    from paper_1107_3622_b200.build import build
    build()
    return _lib.load()


def test_header_lists_the_abi():
    syms = declared_symbols()
    assert "ks_sort_f64" in syms and "ks_partition_f64" in syms and "ks_heap_sort_f64_exact" in syms
    from paper_1107_3622_b200 import _lib
    assert sorted(_lib.EXPORTED) == syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_nm_exports(lib):
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_host_only_entry_points(lib):
    assert lib.ks_version().startswith(b"ksort sm_100a")
    w0 = lib.ks_workspace_bytes(10_000_000, 1, 0)
    assert w0 >= 8 * 10_000_000             # scratch ping-pong buffer
    assert lib.ks_workspace_bytes(10_000_000, 1, 1) > w0   # exact engine keeps position lists
    assert lib.ks_workspace_bytes(-1, 1, 0) == 0


def test_host_entry_argument_checks(lib):
    # ks_sort_f64_host validates before any CUDA call: bad sizes / null buffers -> KS_BAD_ARG,
    # an empty array -> KS_OK, and the status block carries the code
    import ctypes
    from paper_1107_3622_b200 import _lib
    _lib.load()   # sets argtypes
    st = _lib.KsStatus()
    assert lib.ks_sort_f64_host(None, -1, None, None, 0, None, 0, ctypes.byref(st)) == _lib.KS_BAD_ARG
    assert st.code == _lib.KS_BAD_ARG
    h = (ctypes.c_double * 4)(3.0, 1.0, 2.0, 0.5)
    assert lib.ks_sort_f64_host(ctypes.addressof(h), 4, None, None, 0, None, 0, ctypes.byref(st)) == _lib.KS_BAD_ARG
    assert list(h) == [3.0, 1.0, 2.0, 0.5]   # untouched
    assert lib.ks_sort_f64_host(None, 0, None, None, 0, None, 0, ctypes.byref(st)) == _lib.KS_OK


def test_status_struct_layout(tmp_path):
    # the ctypes mirror must match the C compiler's layout of ks_status_t
    import subprocess
    from paper_1107_3622_b200._lib import KsStatus
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "ksort.h"\n'
                   'int main(void){printf("%zu %zu %zu\\n", sizeof(ks_status_t),'
                   ' offsetof(ks_status_t, leaves), offsetof(ks_status_t, phase_bytes));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    size, off_leaves, off_pb = map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split())
    assert ctypes.sizeof(KsStatus) == size
    assert KsStatus.leaves.offset == off_leaves and KsStatus.phase_bytes.offset == off_pb


def test_sass_is_sm100a(lib):
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "-lelf", lib._name], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1107_3622_b200 as K
    with pytest.raises(RuntimeError):
        K.k_sort([3.0, 1.0, 2.0])
