"""CPU-only tests: the C-ABI library, host-side API logic and error parity.

No GPU and no reference needed; expected values come from the golden files
made by the reference (tests/golden/make_golden.py).
"""
import gzip
import json
import re
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2305_00332_b200 as mm
from paper_2305_00332_b200 import _native, errors

ROOT = Path(__file__).resolve().parent.parent
GOLD = ROOT / "tests" / "golden"


def test_library_exports_every_header_symbol():
    hdr = (ROOT / "include" / "mmlttb.h").read_text()
    declared = set(re.findall(r"\b(mmlttb_\w+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    L = _native.load()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_native.EXPORTED)
    assert L.mmlttb_version() == 1


def test_library_is_sm100a():
    import subprocess

    so = _native.LIB_PATH
    r = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_workspace_sizes_are_small_and_independent_of_n():
    # P12 / SPEC acceptance #11: aux memory O(k + m), not O(N)
    L = _native.load()
    a = L.mmlttb_workspace_bytes(_native.OP_MINMAXLTTB, 1, 10_000_000, 2000, 4, _native.MM_F32)
    b = L.mmlttb_workspace_bytes(_native.OP_MINMAXLTTB, 1, 1_000_000, 2000, 4, _native.MM_F32)
    assert 0 < a < 4 << 20 and 0 < b < 4 << 20
    assert abs(a - b) / b < 0.10


def test_workspace_bytes_memo_matches_library():
    """The hot path's memoised mmlttb_workspace_bytes returns the library's value."""
    L = _native.load()
    for op, B, n, n_out, r, ydt in [(_native.OP_MINMAXLTTB, 1, 1_000_000, 1000, 4, _native.MM_F64),
                                    (_native.OP_MINMAXLTTB, 3, 1_000_000, 1000, 32, _native.MM_F32),
                                    (_native.OP_LTTB, 1, 10_000_000, 2000, 0, _native.MM_F64),
                                    (_native.OP_LTTB, 4, 300_000, 700, 0, _native.MM_F32),
                                    (_native.OP_PRESELECT, 2, 5_000_000, 2000, 8, _native.MM_F32)]:
        want = L.mmlttb_workspace_bytes(op, B, n, n_out, r, ydt)
        assert _native.workspace_bytes(op, B, n, n_out, r, ydt) == want > 0
        assert _native.workspace_bytes(op, B, n, n_out, r, ydt) == want  # cached


def test_flat_k3c_workspace_is_bounded():
    """The single-series K3c flat passes add O(k3) workspace, not O(N)."""
    L = _native.load()
    a = L.mmlttb_workspace_bytes(_native.OP_LTTB, 1, 10_000_000, 2000, 0, _native.MM_F64)
    b = L.mmlttb_workspace_bytes(_native.OP_LTTB, 1, 1_000_000_000, 2000, 0, _native.MM_F64)
    assert 0 < a < 32 << 20 and a == b
    # the K3s group summaries (1 KB per bucket) are carved only up to K3S_K3MAX buckets:
    # a large n_out pays the K3c arrays (~1.5 KB per bucket) and no more
    c = L.mmlttb_workspace_bytes(_native.OP_LTTB, 1, 100_000_000, 200_000, 0, _native.MM_F64)
    assert c < 1700 * 200_000 + (32 << 20)


def test_error_hierarchy_matches_reference_names():
    for name in ("NonMonotonicX", "NonFiniteValue", "NOutOfRange", "BadPreselectionRatio", "InvalidPartition",
                 "OddNOut", "NOutNotDivisibleBy4", "RatioTooLargeForSeries", "NotParallelizable"):
        cls = getattr(errors, name)
        assert issubclass(cls, errors.ValidationError) and issubclass(cls, ValueError)
    assert issubclass(errors.OutOfMemory, errors.TsdownError)


def test_partition_kats():
    k = json.loads((GOLD / "kats.json").read_text())["partition"]
    for key, b in k.items():
        s, e, n = map(int, key.split(","))
        assert mm.partition(s, e, n).boundaries.tolist() == b
    with pytest.raises(errors.InvalidPartition):
        mm.partition(0, 3, 4)
    with pytest.raises(errors.InvalidPartition):
        mm.partition(0, 3, 0)


def test_partition_sizes_exhaustive():
    for length in range(1, 120):
        for k in range(1, length + 1):
            s = mm.partition(5, 5 + length, k).sizes()
            assert s.max() - s.min() <= 1 and s.sum() == length


def test_timeseries_invariants():
    with pytest.raises(errors.NonFiniteValue):
        mm.TimeSeries([0, 1, 2], [0.0, np.nan, 1.0])
    with pytest.raises(errors.NonFiniteValue):
        mm.TimeSeries([0.0, np.inf, 2.0], [0.0, 1.0, 1.0])
    with pytest.raises(errors.NonMonotonicX):
        mm.TimeSeries([0, 2, 1], [1, 2, 3])
    with pytest.raises(ValueError):
        mm.TimeSeries([0, 1], [1, 2, 3])
    with pytest.raises(ValueError):
        mm.TimeSeries([0], [1])
    with pytest.raises(ValueError):
        mm.TimeSeries(np.zeros((2, 2)), np.zeros((2, 2)))
    ts = mm.TimeSeries([0, 1, 1, 2], [1, 2, 3, 4])  # non-decreasing x is fine
    assert len(ts) == 4 and ts.ys.dtype == np.float64  # ints -> float64 like core.py:49
    t32 = mm.TimeSeries(np.arange(3), np.ones(3, np.float32))
    assert t32.y_data.dtype == np.float32 and t32.ys.dtype == np.float64  # stored f32, exposed f64 (core.py:48-53)
    assert not t32.xs.flags.writeable and not t32.ys.flags.writeable
    with pytest.raises(AttributeError):
        ts.foo = 1
    big = np.array([2**53 + 1, 2**53], dtype=np.int64)  # equal once converted to f64
    mm.TimeSeries(big, [0.0, 1.0])


def _golden_config_cases():
    with gzip.open(GOLD / "config_errors.json.gz", "rt") as f:
        return json.load(f)


def test_config_and_validate_parity():
    rng = np.random.Generator(np.random.PCG64(77))
    series = {}
    for n in (3, 4, 5, 10, 57):
        x = np.arange(n)
        series[n] = mm.TimeSeries(x, rng.standard_normal(n))
    for rec in _golden_config_cases():
        args = (rec["algo"], rec["n_out"], rec["r_ps"], rec["parallel"], rec["threads"])
        if "config_error" in rec:
            with pytest.raises(Exception) as ei:
                mm.DownsampleConfig(*args)
            assert type(ei.value).__name__ == rec["config_error"], rec
            continue
        cfg = mm.DownsampleConfig(*args)
        try:
            mm.validate(series[rec["n"]], cfg)
            got = "ok"
        except errors.TsdownError as e:
            got = type(e).__name__
        assert got == rec["validate"], rec


def test_checks_raise_before_any_device_work():
    # argument errors surface in the reference's order even with no GPU
    ts = mm.TimeSeries(np.arange(20), np.arange(20.0))
    with pytest.raises(errors.NOutOfRange):
        mm.minmaxlttb(ts, 2, 4)
    with pytest.raises(errors.BadPreselectionRatio):
        mm.minmaxlttb(ts, 5, 3)
    with pytest.raises(errors.RatioTooLargeForSeries):
        mm.minmaxlttb(ts, 10, 8)
    with pytest.raises(errors.OddNOut):
        mm.minmax(ts, 5)
    with pytest.raises(errors.OddNOut):
        mm.minmaxlttb(ts, 5, 1)
    with pytest.raises(errors.NOutNotDivisibleBy4):
        mm.m4(ts, 6)
    with pytest.raises(errors.NOutOfRange):
        mm.lttb(ts, 21)
    with pytest.raises(errors.NotParallelizable):
        mm.downsample(ts, mm.DownsampleConfig("lttb", 5, parallel=True))
    with pytest.raises(ValueError):
        mm.run_parallel(ts, mm.DownsampleConfig("minmax", 6))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    ts = mm.TimeSeries(np.arange(20), np.arange(20.0))
    with pytest.raises(errors.CudaError):
        mm.minmaxlttb(ts, 6, 2)
    with pytest.raises(errors.CudaError):
        mm.lttb(np.arange(20), np.arange(20.0), 6)


def test_timeseries_owns_its_arrays():
    """the caller's arrays stay writable and later writes do not reach the series."""
    x = np.arange(5, dtype=np.int64)
    y = np.linspace(0.0, 1.0, 5)
    ts = mm.TimeSeries(x, y)
    assert x.flags.writeable and y.flags.writeable
    x[0] = 100  # would make x non-monotonic if it were shared
    y[1] = -7.0
    assert ts.xs[0] == 0.0 and ts.ys[1] == 0.25
    assert ts.xs.dtype == np.float64 and ts.ys.dtype == np.float64
    with pytest.raises(ValueError):
        ts.ys[0] = 1.0  # read-only like the reference's frozen arrays
    base = np.arange(10, dtype=np.float64)
    ts2 = mm.TimeSeries(base[::2], base[1::2])
    base[:] = -1.0
    assert ts2.xs[0] == 0.0 and ts2.ys[0] == 1.0


def test_flat_and_reference_forms_never_rebind():
    """Mixing the flat form (x, y, n_out, minmax_ratio) with the reference form
    (series, n_out, r_ps, parallel) raises TypeError instead of misbinding."""
    x = np.arange(100, dtype=np.int64)
    y = np.zeros(100)
    with pytest.raises(TypeError):
        mm.minmaxlttb(x, y, 10, True)  # a bool in the ratio slot
    with pytest.raises(TypeError):
        mm.minmaxlttb(x, y, 10, 4, minmax_ratio=4)  # ratio twice
    with pytest.raises(TypeError):
        mm.minmax(x, y)  # flat minmax without n_out
    with pytest.raises(TypeError):
        mm.minmax(x, y, 10, True)
    with pytest.raises(TypeError):
        mm.lttb(x, y)
    with pytest.raises(TypeError):
        mm.minmax_preselect(x, y, 10)  # flat preselect without r_ps
    ts = mm.TimeSeries(x, y)
    with pytest.raises(TypeError):
        mm.minmaxlttb(ts, y, 10)  # an array in the n_out slot
    with pytest.raises(TypeError):
        mm.lttb(ts, 10, 4)
