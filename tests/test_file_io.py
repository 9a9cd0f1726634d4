"""Array files: the reference's binary/text formats read
straight to the device.  Formats and messages follow workload.py:129-174."""
import math
import struct

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1107_3622_b200 as K  # noqa: E402


def _ref_write_binary(path, a):   # workload.py:137-140, restated
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", len(a)))
        fh.write(struct.pack(f"<{len(a)}d", *a))


def test_binary_truncated_header(tmp_path):
    p = tmp_path / "x.bin"
    p.write_bytes(b"\x01\x02\x03")
    with pytest.raises(ValueError, match=r"truncated header, 3 bytes"):
        K.read_binary(p)


def test_binary_size_mismatch(tmp_path):
    p = tmp_path / "x.bin"
    p.write_bytes(struct.pack("<Q", 3) + struct.pack("<2d", 1.0, 2.0))
    with pytest.raises(ValueError, match=r"expected 32 bytes for 3 values, found 24"):
        K.read_binary(p)


def test_text_not_a_float(tmp_path):
    p = tmp_path / "x.txt"
    p.write_text("1.0\n\nabc\n", encoding="ascii")
    with pytest.raises(ValueError, match=r"x.txt:3: not a float: 'abc'"):
        K.read_text(p)


def test_write_formats_match_reference(tmp_path):
    a = [0.1, 1e-310, -2.5, 1.7976931348623157e308, 3.0]
    ours, ref = tmp_path / "o.bin", tmp_path / "r.bin"
    K.write_binary(ours, a)
    _ref_write_binary(ref, a)
    assert ours.read_bytes() == ref.read_bytes()
    t = tmp_path / "o.txt"
    K.write_text(t, np.array(a))
    assert t.read_text(encoding="ascii") == "".join(repr(v) + "\n" for v in a)


gpu = pytest.mark.gpu
needs_cuda = pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")


@gpu
@needs_cuda
def test_binary_round_trip_to_device_and_sort(tmp_path):
    rng = np.random.default_rng(7)
    a = rng.random(100_003)
    p = tmp_path / "a.bin"
    _ref_write_binary(p, a.tolist())
    t = K.read_binary(p)
    assert t.is_cuda and t.dtype == torch.float64
    assert np.array_equal(t.cpu().numpy().view(np.int64), a.view(np.int64))
    K.k_sort(t)
    q = tmp_path / "s.bin"
    K.write_binary(q, t)
    _ref_write_binary(tmp_path / "r.bin", sorted(a.tolist()))
    assert q.read_bytes() == (tmp_path / "r.bin").read_bytes()


@gpu
@needs_cuda
@pytest.mark.parametrize("bad", [math.nan, math.inf, -math.inf])
def test_binary_nonfinite_rejected_on_device(tmp_path, bad):
    a = [0.5, 0.25, 0.75, bad, 0.125, bad]
    p = tmp_path / "bad.bin"
    _ref_write_binary(p, a)
    with pytest.raises(K.NonFiniteKeyError, match=rf"bad.bin: value at position 3 is {bad!r}; keys must be finite"):
        K.read_binary(p)


@gpu
@needs_cuda
def test_text_round_trip(tmp_path):
    a = [3.5, -0.0, 1e-300, 2.0 ** 0.5, 123456789.125]
    p = tmp_path / "a.txt"
    p.write_text("".join(repr(v) + "\n" for v in a) + "\n", encoding="ascii")
    t = K.read_text(p)
    assert np.array_equal(t.cpu().numpy().view(np.int64), np.array(a).view(np.int64))
    p.write_text("1.0\ninf\n", encoding="ascii")
    with pytest.raises(K.NonFiniteKeyError, match=r"value at position 1 is inf"):
        K.read_text(p)
