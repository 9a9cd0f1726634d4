"""The reference's own callers, unmodified, driving the B200 sorters (GPU).

The reference package is installed stock under baseline/_ref (see
baseline/ref_import.py); the GPU sorters are registered into its
``sortlab.sort_core.SORTERS`` (paper_1107_3622_b200.plugin.register) and run
through ``bench.run_cell`` / ``bench.run_grid`` (bench.py:122-217) and
``cli.main(["sort", ...])`` (cli.py:88-117) on ``list[float]`` KeyArrays --
exactly the objects the reference passes.  Outputs are compared bytewise with
the reference's own Python sorters on the same inputs.
"""
import os
import struct

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from baseline import ref_import  # noqa: E402

if not ref_import.available():
    pytest.skip("reference not installed under baseline/_ref", allow_module_level=True)

import paper_1107_3622_b200 as K  # noqa: E402
from paper_1107_3622_b200 import plugin  # noqa: E402

sortlab = ref_import.import_sortlab()
sc, bench, cli, workload = sortlab.sort_core, sortlab.bench, sortlab.cli, sortlab.workload


@pytest.fixture(autouse=True)
def registered():
    names = plugin.register(sc.SORTERS)
    yield names
    for k in names:
        sc.SORTERS.pop(k, None)


def bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def test_registry_is_the_one_the_callers_read(registered):
    assert set(registered) == {"ksort_b200", "heapsort_b200"}
    assert bench.SORTERS is sc.SORTERS and cli.SORTERS is sc.SORTERS
    assert sc.SORTERS["ksort_b200"] is K.k_sort


@pytest.mark.parametrize("algo", ["ksort_b200", "heapsort_b200"])
def test_run_cell_wall_time_sorts_reference_inputs(algo):
    # run_cell raises SortIntegrityError if the sorter leaves the list unsorted (bench.py:157-160)
    rec = bench.run_cell(algo, 100_000, reps=3, seed=20260816, warmup=1)
    assert rec.algorithm == algo and rec.n == 100_000 and rec.reps == 3 and rec.mean_seconds > 0


def test_run_cell_inputs_bytewise_equal_reference_ksort():
    # the same data run_cell builds (bench.py:147), sorted by both
    for rep in range(2):
        data = workload.generate(workload.WorkloadSpec(n=50_000, seed=workload.derive_seed(20260816, rep, 0)))
        ref = list(data)
        sc.k_sort(ref)
        K.k_sort(data)
        assert isinstance(data, list)
        assert np.array_equal(bits(data), bits(ref))


def test_run_cell_op_counts_match_reference():
    got = bench.run_cell("ksort_b200", 5_000, reps=2, seed=7, mode="op_counts")
    want = bench.run_cell("ksort", 5_000, reps=2, seed=7, mode="op_counts")
    assert (got.comparisons_mean, got.moves_mean) == (want.comparisons_mean, want.moves_mean)
    got = bench.run_cell("heapsort_b200", 3_000, reps=2, seed=7, mode="op_counts")
    want = bench.run_cell("heapsort", 3_000, reps=2, seed=7, mode="op_counts")
    assert (got.comparisons_mean, got.moves_mean) == (want.comparisons_mean, want.moves_mean)


def test_run_grid_with_explicit_algorithms():
    cfg = bench.BenchConfig(sizes=(20_000, 60_000), reps=2, seed=3, algorithms=("ksort", "ksort_b200"))
    recs = bench.run_grid(cfg)
    assert [(r.algorithm, r.n) for r in recs] == [("ksort", 20_000), ("ksort_b200", 20_000),
                                                 ("ksort", 60_000), ("ksort_b200", 60_000)]


def test_cli_sort_binary_file_matches_reference(tmp_path, capsys):
    src = tmp_path / "w.bin"
    assert cli.main(["generate", "--n", "70000", "--seed", "20260816", "--out", str(src)]) == 0
    out_gpu, out_ref = tmp_path / "gpu.bin", tmp_path / "ref.bin"
    assert cli.main(["sort", "--algo", "ksort_b200", "--in", str(src), "--out", str(out_gpu)]) == 0
    assert cli.main(["sort", "--algo", "ksort", "--in", str(src), "--out", str(out_ref)]) == 0
    assert out_gpu.read_bytes() == out_ref.read_bytes()
    text = capsys.readouterr().out
    assert "sorted 70000 keys with ksort_b200" in text


def test_cli_sort_counts_and_text_format(tmp_path, capsys):
    src = tmp_path / "w.txt"
    keys = [55.0, 66.0, 60.0, 78.0, 22.0, 50.0, 75.0, 5.0, 8.0, 94.0]   # the paper's trace
    workload.write_text(str(src), keys)
    out = tmp_path / "o.txt"
    assert cli.main(["sort", "--algo", "ksort_b200", "--in", str(src), "--format", "text", "--out", str(out),
                     "--counts"]) == 0
    text = capsys.readouterr().out
    assert "comparisons=20 moves=26 max_pending_ranges=2" in text   # tests/test_sort_core.py:129-137
    assert workload.read_text(str(out)) == sorted(keys)


def test_cli_sort_nonfinite_file_exit_1(tmp_path, capsys):
    src = tmp_path / "bad.bin"
    # reference binary layout (workload.py:137-150): 8-byte LE count + LE float64
    vals = [0.5, 0.25, float("nan"), 0.75]
    src.write_bytes(struct.pack("<Q", len(vals)) + struct.pack("<4d", *vals))
    assert cli.main(["sort", "--algo", "ksort_b200", "--in", str(src)]) == 1
    err = capsys.readouterr().err
    assert "error:" in err


def test_replace_registers_drop_in_names():
    reg = {}
    plugin.register(reg, replace=True)
    assert reg == {"ksort": K.k_sort, "heapsort": K.heap_sort}
