"""TSB1 / CSV series files (reference seriesio.py:20-95)."""
import struct

import numpy as np
import pytest
import torch

import paper_2305_00332_b200 as mm
from paper_2305_00332_b200 import seriesio


def _write_ref_bin(path, x, y):
    # the reference's writer, seriesio.py:75-81
    inter = np.empty(2 * x.shape[0], dtype="<f8")
    inter[0::2] = x
    inter[1::2] = y
    with open(path, "wb") as fh:
        fh.write(struct.pack("<4sQ", b"TSB1", x.shape[0]))
        fh.write(inter.tobytes())


def test_header_errors(tmp_path):
    p = tmp_path / "a.bin"
    p.write_bytes(b"TSB1\x01")
    with pytest.raises(ValueError, match="truncated"):
        seriesio._read_bin_host(p)
    p.write_bytes(struct.pack("<4sQ", b"XXXX", 3))
    with pytest.raises(ValueError, match="bad magic"):
        seriesio._read_bin_host(p)
    p.write_bytes(struct.pack("<4sQ", b"TSB1", 3) + b"\0" * 16)
    with pytest.raises(ValueError, match="short"):
        seriesio._read_bin_host(p)
    assert seriesio.detect_format(p) == "bin"


def test_host_roundtrips(tmp_path):
    rng = np.random.Generator(np.random.PCG64(0))
    x = np.cumsum(rng.exponential(1.0, 1000))
    y = rng.standard_normal(1000)
    _write_ref_bin(tmp_path / "s.bin", x, y)
    ts = seriesio._read_bin_host(tmp_path / "s.bin")
    assert np.array_equal(ts.xs, x) and np.array_equal(ts.ys, y)
    mm.write_series(tmp_path / "s.csv", ts, "csv")
    assert seriesio.detect_format(tmp_path / "s.csv") == "csv"
    back = mm.read_series(tmp_path / "s.csv")
    assert np.array_equal(back.xs, x) and np.array_equal(back.ys, y)
    mm.write_series(tmp_path / "t.bin", ts, "bin")
    assert (tmp_path / "t.bin").read_bytes() == (tmp_path / "s.bin").read_bytes()


@pytest.mark.gpu
def test_device_ingest(tmp_path):
    rng = np.random.Generator(np.random.PCG64(1))
    n = 3_000_003
    x = np.cumsum(rng.exponential(1.0, n))
    y = np.cumsum(rng.standard_normal(n))
    _write_ref_bin(tmp_path / "s.bin", x, y)
    old = seriesio._CHUNK_PAIRS
    seriesio._CHUNK_PAIRS = 1 << 20  # several pipelined chunks
    try:
        ts = mm.read_series(tmp_path / "s.bin", device="cuda:0")
    finally:
        seriesio._CHUNK_PAIRS = old
    assert not ts.is_host and ts.x_data.is_cuda
    assert np.array_equal(ts.x_data.cpu().numpy(), x) and np.array_equal(ts.y_data.cpu().numpy(), y)
    assert np.array_equal(ts.xs, x) and ts.ys.dtype == np.float64  # reference surface: host float64
    from oracle import oracle as O

    out = mm.minmaxlttb(ts, 1000, 4)
    assert np.array_equal(out.cpu().numpy(), O.minmaxlttb(x, y, 1000, 4))
    y[17] = np.nan
    _write_ref_bin(tmp_path / "bad.bin", x, y)
    with pytest.raises(mm.errors.NonFiniteValue):
        mm.read_series(tmp_path / "bad.bin", device="cuda:0")
    (tmp_path / "short.bin").write_bytes((tmp_path / "s.bin").read_bytes()[:-8])
    with pytest.raises(ValueError, match="short"):
        mm.read_series(tmp_path / "short.bin", device="cuda:0")
