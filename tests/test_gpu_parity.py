"""Device parity: the sm_100a path vs the reference's golden outputs and the oracle.

Index-exact equality everywhere (integer/index work; LTTB fp64 parity is
bit-exact by construction, so the tolerance is zero).  Inputs are the
seeded recipes of tests/recipes.py and tests/fuzzgen.py.
"""
import ctypes
import gzip
import json
import os
from pathlib import Path

import numpy as np
import pytest
import torch

import fuzzgen
import recipes
import paper_2305_00332_b200 as mm
from paper_2305_00332_b200 import _native, errors
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
DEV = torch.device("cuda", 0)


def _cfg():
    return json.loads((GOLD / "configs.json").read_text())


def _call(op, series, n_out, r_ps):
    try:
        if op == "minmaxlttb":
            out = mm.minmaxlttb(series, n_out, r_ps)
        elif op == "lttb":
            out = mm.lttb(series, n_out)
        elif op == "minmax":
            out = mm.minmax(series, n_out)
        elif op == "minmax_preselect":
            out = mm.minmax_preselect(series, n_out, r_ps)
        elif op == "m4":
            out = mm.m4(series, n_out)
        else:
            raise ValueError(op)
    except errors.TsdownError as e:
        return {"error": type(e).__name__}
    if isinstance(out, torch.Tensor):
        out = out.cpu().numpy()
    return {"out": [int(v) for v in out]}


def test_kats():
    k = json.loads((GOLD / "kats.json").read_text())
    ts = mm.TimeSeries
    a = [1, 3, 2, 0, 5, 4, 9, 8]
    xa = list(range(8))
    assert mm.minmax(ts(xa, a), 4).tolist() == k["minmax"]
    assert mm.m4(ts(xa, a), 8).tolist() == k["m4"]
    assert mm.lttb(ts(list(range(6)), [0, 0, 10, 0, 0, 0]), 3).tolist() == k["lttb_spike"]
    assert mm.minmax(ts(list(range(10)), [3.0] * 10), 4).tolist() == k["minmax_constant_n10"]
    assert mm.lttb(ts(list(range(20)), list(range(20))), 6).tolist() == k["lttb_collinear_n20"]
    assert mm.minmax_preselect(ts(list(range(10)), np.sin(np.arange(10.0))), 4, 2).tolist() == k["preselect_sin10"]
    assert mm.minmaxlttb(ts(xa, a), 4, r_ps=1).tolist() == k["minmaxlttb_r1"]
    assert mm.every_nth(ts(list(range(10)), [0.0] * 10), 5).tolist() == k["every_nth_10_5"]
    assert mm.every_nth(ts(list(range(7)), [0.0] * 7), 3).tolist() == k["every_nth_7_3"]
    assert mm.minmax(ts([0, 1, 2, 3], [0.0, -0.0, 0.0, -0.0]), 4).tolist() == k["signed_zero_minmax"]


def _fuzz():
    with gzip.open(GOLD / "fuzz.json.gz", "rt") as f:
        return json.load(f)


@pytest.mark.parametrize("home", ["host", "device"])
def test_fuzz_matches_reference(home):
    bad = []
    for rec in _fuzz():
        c = fuzzgen.make_case(rec["i"])
        x, y = c["x"], c["y"]
        if home == "device":
            x, y = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
        got = _call(rec["op"], mm.TimeSeries(x, y), rec["n_out"], rec["r_ps"])
        want = {k: rec[k] for k in ("out", "error") if k in rec}
        if got != want:
            bad.append((rec["i"], rec["op"], rec["kind"], rec["n"], rec["n_out"], rec["r_ps"]))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:8]}"


def test_downsample_config_parity():
    with gzip.open(GOLD / "config_errors.json.gz", "rt") as f:
        recs = json.load(f)
    rng = np.random.Generator(np.random.PCG64(77))
    series = {n: mm.TimeSeries(np.arange(n), rng.standard_normal(n)) for n in (3, 4, 5, 10, 57)}
    for rec in recs:
        if "config_error" in rec:
            continue
        cfg = mm.DownsampleConfig(rec["algo"], rec["n_out"], rec["r_ps"], rec["parallel"], rec["threads"])
        try:
            got = {"out": [int(v) for v in mm.downsample(series[rec["n"]], cfg)]}
        except (errors.TsdownError, ValueError) as e:
            got = {"downsample_error": type(e).__name__}
        want = {k: rec[k] for k in ("out", "downsample_error") if k in rec}
        assert got == want, rec


def test_c1_full():
    x, y = recipes.c1()
    g = _cfg()["C1"]["r4"]["out"]
    assert mm.minmaxlttb(mm.TimeSeries(x, y), 1000, 4).tolist() == g
    out = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 1000, minmax_ratio=4)
    assert out.cpu().tolist() == g


def test_c2_full_lttb():
    x, y = recipes.c2()
    g = _cfg()["C2"]["lttb"]["out"]
    out = mm.lttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 2000)
    assert out.cpu().tolist() == g


def test_c3_full_all_ratios():
    x, y = recipes.c3()
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    cfg = _cfg()["C3"]
    for r in recipes.CONFIGS["C3"]["r_ps"]:
        out = mm.minmaxlttb(xd, yd, 2000, minmax_ratio=r)
        assert out.cpu().tolist() == cfg[f"r{r}"]["out"], r


def _c4_device(ids, n, dev):
    """Rows `ids` of the C4 batch generated on host threads (numpy releases the
    GIL in its generators and cumsum) and staged into one device matrix."""
    from concurrent.futures import ThreadPoolExecutor

    yd = torch.empty((len(ids), n), dtype=torch.float32, device=dev)
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 4)) as ex:
        for i, row in enumerate(ex.map(lambda s: recipes.c4_series(s, n), ids)):
            yd[i].copy_(torch.from_numpy(row))
    return yd


def test_c4_full_batch():
    """All 4,096 series of C4 in ONE batched call, every row against the
    reference's output SHA (downsamplers.py:182-209 per series)."""
    import hashlib

    g = json.loads((GOLD / "c4.json").read_text())
    n, B = 1_000_000, 4096
    ids = list(range(B))
    yd = _c4_device(ids, n, DEV)
    xd = torch.arange(n, dtype=torch.int64, device=DEV)
    out = mm.minmaxlttb(xd, yd, 1000, minmax_ratio=4).cpu().numpy()
    assert out.shape == (B, 1000)
    bad = [s for s in ids if hashlib.sha256(out[s].astype(np.int64).tobytes()).hexdigest() != g["sha"][s]]
    assert not bad, bad[:20]
    for s, o in g["full"].items():
        assert out[int(s)].tolist() == o


@pytest.mark.slow
def test_c5_full():
    g = _cfg()["C5"]["r4"]["out"]
    n = recipes.CONFIGS["C5"]["n"]
    xd = torch.empty(n, dtype=torch.float64, device=DEV)
    yd = torch.empty(n, dtype=torch.float32, device=DEV)
    for lo, xc, yc in recipes.c5_chunks(n):
        xd[lo:lo + xc.shape[0]].copy_(torch.from_numpy(xc))
        yd[lo:lo + yc.shape[0]].copy_(torch.from_numpy(yc))
    out = mm.minmaxlttb(xd, yd, 4000, minmax_ratio=4)
    assert out.cpu().tolist() == g


def test_batch_equals_per_series():
    rng = np.random.Generator(np.random.PCG64(5))
    B, n = 37, 20_011
    y = np.cumsum(rng.standard_normal((B, n)), axis=1)
    x = np.cumsum(rng.exponential(1.0, n))
    for dt in (np.float32, np.float64):
        yb = torch.from_numpy(y.astype(dt)).to(DEV)
        out = mm.minmaxlttb(torch.from_numpy(x).to(DEV), yb, 300, minmax_ratio=6).cpu().numpy()
        for i in range(B):
            assert np.array_equal(out[i], O.minmaxlttb(x, y[i].astype(dt), 300, 6)), (dt, i)
        lt = mm.lttb(torch.from_numpy(x).to(DEV), yb, 200).cpu().numpy()
        for i in range(0, B, 6):
            assert np.array_equal(lt[i], O.lttb(x, y[i].astype(dt), 200))


@pytest.mark.parametrize("n,n_out", [(10, 3), (100, 98), (1000, 500), (65_537, 40), (300_000, 3),
                                     # K3s below one bucket per SM (G = k3 CTAs) / K3c for wide buckets
                                     (20_000, 4), (50_000, 5), (200_000, 60), (1_000_000, 150), (2_000_000, 40)])
def test_lttb_shapes(n, n_out):
    rng = np.random.Generator(np.random.PCG64(n))
    x = np.cumsum(rng.exponential(1.0, n))
    y = rng.standard_normal(n)
    got = mm.lttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out).cpu().numpy()
    assert np.array_equal(got, O.lttb(x, y, n_out))


@pytest.mark.parametrize("r", [2, 4, 8, 16, 32, 64, 100])
def test_minmaxlttb_ratios_small(r):
    rng = np.random.Generator(np.random.PCG64(r))
    n = 200_000
    x = np.arange(n, dtype=np.int64)
    y = np.cumsum(rng.standard_normal(n)).astype(np.float32)
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 700, minmax_ratio=r)
    assert np.array_equal(got.cpu().numpy(), O.minmaxlttb(x, y, 700, r))


def test_degeneracy_to_lttb():
    # SPEC acceptance #2: sub-buckets of <= 2 points -> minmaxlttb == lttb
    rng = np.random.Generator(np.random.PCG64(2))
    for n in (10, 57, 200, 500):
        x = np.arange(n)
        y = rng.standard_normal(n)
        ts = mm.TimeSeries(x, y)
        for n_out in range(3, n + 1, max(1, n // 17)):
            for r in (2, 4, 6, 8):
                k = (n_out - 2) * (r // 2)
                if k > n - 2 or -(-(n - 2) // k) > 2:
                    continue
                assert np.array_equal(mm.minmaxlttb(ts, n_out, r), mm.lttb(ts, n_out)), (n, n_out, r)


def test_pinned_host_inputs_zero_copy_x():
    x, y = recipes.c1(500_000)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.from_numpy(y.astype(np.float32)).pin_memory()
    out = mm.minmaxlttb(xp, yp, 1000, minmax_ratio=4)
    assert not out.is_cuda
    assert np.array_equal(out.numpy(), O.minmaxlttb(x, y.astype(np.float32), 1000, 4))


def test_reference_kernel_entry_points():
    """mmlttb_extrema_by_bucket / mmlttb_lttb_select vs the oracle's restatement."""
    L = _native.lib()
    rng = np.random.Generator(np.random.PCG64(9))
    n = 100_003
    y = np.cumsum(rng.standard_normal(n))
    y[::97] = -0.0
    bounds = mm.partition(1, n - 1, 777).boundaries
    yd = torch.from_numpy(y).to(DEV)
    bd = torch.from_numpy(np.ascontiguousarray(bounds)).to(DEV)
    mn = torch.empty(777, dtype=torch.int64, device=DEV)
    mx = torch.empty(777, dtype=torch.int64, device=DEV)
    smax = int(np.diff(bounds).max())
    wsb = L.mmlttb_extrema_workspace_bytes(777, smax)
    ws = torch.empty(wsb, dtype=torch.uint8, device=DEV)
    st = torch.cuda.current_stream().cuda_stream
    _native.check(L.mmlttb_extrema_by_bucket(yd.data_ptr(), 1, bd.data_ptr(), 777, smax, mn.data_ptr(),
                                             mx.data_ptr(), ws.data_ptr(), wsb, st), "extrema")
    omn, omx = O.extrema_by_bucket(y, bounds)
    assert np.array_equal(mn.cpu().numpy(), omn) and np.array_equal(mx.cpu().numpy(), omx)
    x = np.arange(n, dtype=np.int64)
    lb = mm.partition(1, n - 1, 398).boundaries
    lbd = torch.from_numpy(np.ascontiguousarray(lb)).to(DEV)
    out = torch.empty(400, dtype=torch.int64, device=DEV)
    wsb = L.mmlttb_lttb_select_workspace_bytes(n, 399)
    ws = torch.empty(wsb, dtype=torch.uint8, device=DEV)
    xd = torch.from_numpy(x).to(DEV)
    _native.check(L.mmlttb_lttb_select(xd.data_ptr(), 2, yd.data_ptr(), 1, n, lbd.data_ptr(), 399, out.data_ptr(),
                                       ws.data_ptr(), wsb, st), "lttb_select")
    assert np.array_equal(out.cpu().numpy(), O.lttb(x, y, 400))


def test_device_validation():
    x = torch.arange(100, device=DEV, dtype=torch.int64)
    y = torch.randn(100, device=DEV)
    mm.TimeSeries(x, y)
    y2 = y.clone()
    y2[50] = float("nan")
    with pytest.raises(errors.NonFiniteValue):
        mm.TimeSeries(x, y2)
    x2 = x.clone()
    x2[10] = 3
    with pytest.raises(errors.NonMonotonicX):
        mm.TimeSeries(x2, y)


@pytest.mark.parametrize("case", ["ok", "neg_zero_after_pos_zero", "i64_equal_after_rounding", "i64_decreasing",
                                  "last_pair", "first_pair", "nan_x", "inf_y32", "inf_y64", "f32x_decreasing"])
def test_device_validation_cases(case):
    """Device TimeSeries validation against the reference's own rules (core.py:89-92:
    np.isfinite on the float64 conversions, then np.diff(xs) < 0), across dtypes,
    +-0.0, int64 beyond 2^53 and grid-stride boundaries."""
    n = 3_000_003
    rng = np.random.Generator(np.random.PCG64(5))
    x = np.arange(n, dtype=np.int64)
    y = rng.standard_normal(n).astype(np.float32)
    if case == "neg_zero_after_pos_zero":
        x = np.arange(n, dtype=np.float64) - 1000.0
        x[1000] = 0.0
        x[1001] = -0.0
        x[1002] = 1.0
    elif case == "i64_equal_after_rounding":
        x = np.arange(n, dtype=np.int64) * 4096 + (1 << 60)
        x[777], x[778] = (1 << 60) + 777 * 4096 + 1, (1 << 60) + 777 * 4096  # equal as float64
    elif case == "i64_decreasing":
        x[2_500_000] = x[2_499_999] - 1
    elif case == "last_pair":
        x[-1] = x[-2] - 1
    elif case == "first_pair":
        x[0] = 5
    elif case == "nan_x":
        x = np.arange(n, dtype=np.float64)
        x[123_456] = np.nan
    elif case == "inf_y32":
        y[n - 1] = np.inf
    elif case == "inf_y64":
        y = y.astype(np.float64)
        y[17] = -np.inf
    elif case == "f32x_decreasing":
        x = np.arange(n, dtype=np.float32)
        x[2_999_000] = 1.0
    xf, yf = x.astype(np.float64), y.astype(np.float64)
    if not (np.isfinite(xf).all() and np.isfinite(yf).all()):
        want = errors.NonFiniteValue
    elif np.any(np.diff(xf) < 0):
        want = errors.NonMonotonicX
    else:
        want = None
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    for off in (0, 1):  # aligned (16-byte vector path) and an unaligned view (scalar path)
        if off and case in ("first_pair",):
            continue
        xo, yo = xd[off:], yd[off:]
        if want is None:
            mm.TimeSeries(xo, yo)
        else:
            with pytest.raises(want):
                mm.TimeSeries(xo, yo)


def test_large_properties_1e9():
    """Size-independent properties at the headline size (C3 recipe, N=1e9)."""
    n = 1_000_000_000
    g = torch.Generator(device=DEV).manual_seed(3)
    y = torch.randn(n, device=DEV, dtype=torch.float32, generator=g)
    x = torch.arange(n, device=DEV, dtype=torch.int64)
    out = mm.minmaxlttb(x, y, 2000, minmax_ratio=4)
    o = out.cpu().numpy()
    assert o.shape == (2000,) and o[0] == 0 and o[-1] == n - 1 and np.all(np.diff(o) > 0)
    # the preselected set contains the global extrema (every LTTB pick comes from it)
    pre = mm.minmax_preselect(x, y, 2000, 4)
    p = pre.cpu().numpy()
    assert int(torch.argmin(y[1:-1])) + 1 in set(p.tolist())
    assert set(o.tolist()) <= set(p.tolist())
    # chunked oracle on the same data agrees exactly
    yh = y.cpu().numpy()
    assert np.array_equal(o, O.minmaxlttb_typed(np.arange(n, dtype=np.int64), yh, 2000, 4))


@pytest.mark.parametrize("n_out,r", [(5000, 2), (5000, 4), (3001, 6), (3001, 8), (4500, 16), (2100, 32)])
def test_lttb_scan_multi_chunk(n_out, r):
    """k3 > 2048 buckets: several scan chunks with a carried prefix map."""
    rng = np.random.Generator(np.random.PCG64(n_out + r))
    n = 3_000_000
    x = np.cumsum(rng.exponential(1.0, n))
    y = np.cumsum(rng.standard_normal(n)).astype(np.float32)
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out, minmax_ratio=r)
    assert np.array_equal(got.cpu().numpy(), O.minmaxlttb(x, y, n_out, r))


def test_lttb_large_bucket_repair_path():
    """K3c with the candidate sets cut to 1-2 points: verification must flag
    the wrong picks and the repair walk must still reproduce the reference."""
    import subprocess
    import sys

    code = (
        "import numpy as np, torch, sys; sys.path.insert(0, '.');"
        "import paper_2305_00332_b200 as mm; from oracle import oracle as O;"
        "rng = np.random.Generator(np.random.PCG64(8)); n = 300_000;"
        "x = np.cumsum(rng.exponential(1.0, n)); y = np.cumsum(rng.standard_normal(n));"
        "g = mm.lttb(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), 700).cpu().numpy();"
        "assert np.array_equal(g, O.lttb(x, y, 700)), 'mismatch';"
        "x2 = np.arange(n, dtype=np.int64); y2 = np.repeat(rng.standard_normal(n // 100), 100);"
        "g = mm.lttb(torch.from_numpy(x2).cuda(), torch.from_numpy(y2).cuda(), 300).cpu().numpy();"
        "assert np.array_equal(g, O.lttb(x2, y2, 300)), 'mismatch2'; print('ok')"
    )
    for cap in ("1", "2"):
        env = dict(__import__("os").environ, MMLTTB_K3C_CAND_CAP=cap)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           cwd=str(GOLD.parent.parent), timeout=300)
        assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_lttb_large_bucket_certification_ties():
    """K3c means are any-order sums certified against an error bound; duplicated
    points tie in every bucket, so every certification fails and each bucket
    falls back to the reference's in-order mean (exact re-scan)."""
    rng = np.random.Generator(np.random.PCG64(11))
    n = 200_000
    x = np.repeat(np.arange(n // 2, dtype=np.float64) * 0.37, 2)
    y = np.repeat(np.cumsum(rng.standard_normal(n // 2)), 2)
    for n_out in (100, 1001):
        got = mm.lttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out).cpu().numpy()
        assert np.array_equal(got, O.lttb(x, y, n_out))
    # integer-valued data: the means are exact (no certification needed)
    xi = np.arange(n, dtype=np.int64)
    yi = np.cumsum(rng.integers(-5, 6, n)).astype(np.float64)
    got = mm.lttb(torch.from_numpy(xi).to(DEV), torch.from_numpy(yi).to(DEV), 150).cpu().numpy()
    assert np.array_equal(got, O.lttb(xi, yi, 150))


@pytest.mark.parametrize("xkind", ["f64_even", "f32_even", "i64_irregular", "i32_arange", "f64_large"])
def test_lttb_large_bucket_x_kinds(xkind):
    """K3c flat passes across x layouts: evenly spaced float timestamps (affine by
    formula), irregular integers (x loaded), int32 and large-magnitude float x
    (inexact x means, so x certification matters too)."""
    rng = np.random.Generator(np.random.PCG64(hash(xkind) % 2**32))
    n = 400_003
    if xkind == "f64_even":
        x = 1.7e9 + 0.25 * np.arange(n, dtype=np.float64)
    elif xkind == "f32_even":
        x = (np.arange(n, dtype=np.float64) * 0.5).astype(np.float32)
    elif xkind == "i64_irregular":
        x = np.cumsum(rng.integers(1, 5, n)).astype(np.int64)
    elif xkind == "i32_arange":
        x = np.arange(n, dtype=np.int32) * 3
    else:
        x = np.cumsum(rng.exponential(1.0, n)) * 1e12
    for ydt in (np.float64, np.float32):
        y = (np.cumsum(rng.standard_normal(n)) * 1e3).astype(ydt)
        for n_out in (300, 1234):
            got = mm.lttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out).cpu().numpy()
            assert np.array_equal(got, O.lttb(x, y, n_out)), (xkind, ydt, n_out)


def test_lttb_large_bucket_degenerate():
    """Ties everywhere (constant / collinear / duplicated points) through K3c."""
    n = 100_000
    x = np.arange(n, dtype=np.int64)
    for y in (np.zeros(n), 3.0 * x + 1.0, np.repeat(np.arange(n // 1000, dtype=np.float64), 1000)):
        got = mm.lttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 90).cpu().numpy()
        assert np.array_equal(got, O.lttb(x, y, 90))
    xr = np.repeat(np.arange(n // 4, dtype=np.float64), 4)  # repeated x
    yr = np.random.Generator(np.random.PCG64(1)).standard_normal(n)
    got = mm.lttb(torch.from_numpy(xr).to(DEV), torch.from_numpy(yr).to(DEV), 120).cpu().numpy()
    assert np.array_equal(got, O.lttb(xr, yr, 120))


@pytest.mark.parametrize("r,ydt,xkind", [(2, np.float32, "i64"), (4, np.float64, "f64"), (6, np.float32, "f32"),
                                          (8, np.float64, "i32")])
def test_fused_batch_path(r, ydt, xkind):
    """B >= 148 series, r_ps <= 8: the one-CTA-per-series fused kernel."""
    rng = np.random.Generator(np.random.PCG64(r * 7))
    B, n, n_out = 160, 30_011, 257
    y = np.cumsum(rng.standard_normal((B, n)), axis=1).astype(ydt)
    y[3, ::7] = -0.0
    y[5] = 1.0  # constant row: every argmin == argmax
    x = {"i64": np.arange(n, dtype=np.int64), "f64": np.cumsum(rng.exponential(1.0, n)),
         "f32": np.arange(n, dtype=np.float32), "i32": np.arange(n, dtype=np.int32) * 3}[xkind]
    out = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out, minmax_ratio=r).cpu().numpy()
    for i in range(B):
        assert np.array_equal(out[i], O.minmaxlttb(x, y[i].astype(np.float64), n_out, r)), i


def test_flat_api_nonfinite_parity():
    """The reference rejects NaN/inf at TimeSeries construction (core.py:89-90);
    the flat form detects it for free from the K1 keys: at once for host inputs
    and validate=True, deferred (no host sync) for device inputs."""
    n = 50_000
    x = np.arange(n, dtype=np.int64)
    for ydt in (np.float32, np.float64):
        for bad in (np.nan, np.inf, -np.inf):
            for pos in (0, 777, n - 1):
                y = np.cumsum(np.ones(n)).astype(ydt)
                y[pos] = bad
                with pytest.raises(errors.NonFiniteValue):
                    mm.minmaxlttb(x, y, 100, minmax_ratio=4)
                with pytest.raises(errors.NonFiniteValue):
                    mm.minmax(x, y, 100)
                with pytest.raises(errors.NonFiniteValue):
                    mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 100, minmax_ratio=4,
                                  validate=True)
    yb = torch.randn(4, n, device=DEV)
    yb[2, 5] = float("nan")
    with pytest.raises(errors.NonFiniteValue):
        mm.minmaxlttb(torch.from_numpy(x).to(DEV), yb, 100, minmax_ratio=4, validate=True)
    xd = torch.from_numpy(x.copy()).to(DEV)
    xd[100] = 5
    with pytest.raises(errors.NonMonotonicX):
        mm.minmaxlttb(xd, torch.randn(n, device=DEV), 100, minmax_ratio=4, validate=True)
    # device inputs without validate: no host sync in the call; the status
    # word comes back asynchronously and the error surfaces at check_deferred()
    mm.check_deferred()
    xd = torch.from_numpy(x).to(DEV)
    out = mm.minmaxlttb(xd, yb, 100, minmax_ratio=4)
    assert out.shape == (4, 100)
    with pytest.raises(errors.NonFiniteValue, match="earlier minmaxlttb call"):
        mm.check_deferred()
    mm.check_deferred()  # reported once
    # ... or at the next call, once the copy has landed
    for fn, args in ((mm.minmaxlttb, (100,)), (mm.minmax, (100,)), (mm.m4, (100,)), (mm.minmax_preselect, (100, 4))):
        fn(xd, yb, *args)
        torch.cuda.synchronize()
        with pytest.raises(errors.NonFiniteValue):
            mm.minmaxlttb(xd, torch.randn(n, device=DEV), 100, minmax_ratio=4)
        mm.check_deferred()
    # clean device calls, validate=False and graph-free streams never raise
    for _ in range(3):
        mm.minmaxlttb(xd, torch.randn(4, n, device=DEV), 100, minmax_ratio=4)
    mm.minmaxlttb(xd, yb, 100, minmax_ratio=4, validate=False)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        mm.minmaxlttb(xd, torch.randn(n, device=DEV), 100, minmax_ratio=4)
    mm.check_deferred()
    # the 1e8-class single-series path (K23 / cooperative) reports it too
    yl = torch.randn(3_000_000, device=DEV)
    yl[2_999_999] = float("inf")
    mm.minmaxlttb(torch.arange(3_000_000, device=DEV), yl, 2000, minmax_ratio=4)
    with pytest.raises(errors.NonFiniteValue):
        mm.check_deferred()


def test_plan_graph_replay():
    x, y = recipes.c1(200_000)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    plan = mm.MinMaxLTTBPlan(200_000, 500, 4, y_dtype=torch.float64, device=DEV)
    a = plan(xd, yd).clone()
    assert np.array_equal(a.cpu().numpy(), O.minmaxlttb(x, y, 500, 4))
    y2 = np.cumsum(np.random.default_rng(1).standard_normal(200_000))
    yd.copy_(torch.from_numpy(y2))  # same buffer, new contents: graph replays on the new data
    b = plan(xd, yd).clone()
    assert np.array_equal(b.cpu().numpy(), O.minmaxlttb(x, y2, 500, 4))
    yd3 = torch.from_numpy(y).to(DEV)  # new buffer: new graph
    assert np.array_equal(plan(xd, yd3).cpu().numpy(), a.cpu().numpy())
    with pytest.raises(errors.ValidationError):
        plan(xd, yd.float())
    with pytest.raises(errors.NOutOfRange):
        mm.MinMaxLTTBPlan(100, 101, 4)


def _minmaxlttb_abi(x, y2d, n, n_out, r, y_ld):
    """mmlttb_minmaxlttb through the C ABI on a [B, y_ld] buffer (rows padded)."""
    from paper_2305_00332_b200 import _native as NN
    B = y2d.shape[0]
    out = torch.empty((B, n_out), dtype=torch.int64, device=DEV)
    ydt = NN.DTYPE_CODE[y2d.dtype]
    L = NN.lib()
    wsb = L.mmlttb_workspace_bytes(NN.OP_MINMAXLTTB, B, n, n_out, r, ydt)
    ws = NN.workspace(wsb, DEV, n)
    NN.check(L.mmlttb_minmaxlttb(x.data_ptr(), NN.DTYPE_CODE[x.dtype], 0, y2d.data_ptr(), ydt, y_ld, B, n, n_out, r,
                                 out.data_ptr(), None, ws.data_ptr(), wsb, NN.stream_ptr(DEV)), "minmaxlttb", n)
    return out.cpu().numpy()


def test_status_arm_abi():
    """mmlttb_status_arm / _poll through the C ABI: every status-producing path
    (K23 single series, fused batch, per-stage batch, preselect, minmax/m4)
    delivers its NaN bit to the armed slot; a failed call and a captured call
    are reported as such; unarmed calls leave the ring alone."""
    from paper_2305_00332_b200 import _native as NN
    L = NN.lib()
    st = NN.stream_ptr(DEV)

    def run(op, y, n_out, r=4, B=1, n=None):
        n = n or y.shape[-1]
        x = torch.arange(n, device=DEV)
        ydt = NN.DTYPE_CODE[y.dtype]
        code = {"mml": NN.OP_MINMAXLTTB, "pre": NN.OP_PRESELECT, "mm": NN.OP_MINMAX, "m4": NN.OP_M4}[op]
        wsb = L.mmlttb_workspace_bytes(code, B, n, n_out, r if op in ("mml", "pre") else 0, ydt)
        ws = torch.empty(wsb, dtype=torch.uint8, device=DEV)
        cap = 2 + 2 * (n_out - 2) * (r // 2)
        out = torch.empty((B, max(n_out, cap)), dtype=torch.int64, device=DEV)
        cnt = torch.empty(B, dtype=torch.int64, device=DEV)
        if op == "mml":
            return L.mmlttb_minmaxlttb(x.data_ptr(), NN.DTYPE_CODE[x.dtype], 0, y.data_ptr(), ydt, n, B, n, n_out, r,
                                       out.data_ptr(), None, ws.data_ptr(), wsb, st)
        if op == "pre":
            return L.mmlttb_minmax_preselect(y.data_ptr(), ydt, n, B, n, n_out, r, out.data_ptr(), out.shape[1],
                                             cnt.data_ptr(), ws.data_ptr(), wsb, st)
        fn = L.mmlttb_minmax if op == "mm" else L.mmlttb_m4
        return fn(y.data_ptr(), ydt, n, B, n, n_out, out.data_ptr(), cnt.data_ptr(), ws.data_ptr(), wsb, st)

    cases = [("mml", 1, 3_000_000, 2000), ("mml", 1, 200_000, 1000), ("mml", 200, 20_000, 100),
             ("mml", 3, 400_000, 40), ("pre", 2, 100_000, 100), ("mm", 2, 100_000, 100), ("m4", 2, 100_000, 100)]
    for op, B, n, n_out in cases:
        for bad in (False, True):
            y = torch.randn(B, n, device=DEV)
            if bad:
                y[B - 1, n // 3] = float("nan")
            t = L.mmlttb_status_arm()
            assert t >= 0
            assert run(op, y, n_out, B=B, n=n) == 0
            assert L.mmlttb_status_poll(t, 1) == int(bad), (op, B, n, bad)
    # a failing call marks its slot failed
    t = L.mmlttb_status_arm()
    y = torch.randn(1, 1000, device=DEV)
    ws = torch.empty(1 << 20, dtype=torch.uint8, device=DEV)
    assert L.mmlttb_minmaxlttb(None, 2, 0, y.data_ptr(), 9, 1000, 1, 1000, 100, 4, ws.data_ptr(), None,
                               ws.data_ptr(), 1 << 20, st) != 0  # bad y dtype
    assert L.mmlttb_status_poll(t, 0) < 0
    # unarmed calls do not write the ring
    ring = np.ctypeslib.as_array((ctypes.c_uint64 * 1024).from_address(L.mmlttb_status_ring()))
    before = ring.copy()
    run("mml", torch.randn(1, 3_000_000, device=DEV), 2000)
    torch.cuda.synchronize()
    assert np.array_equal(ring, before)
    # a captured call delivers "no status" and its graph never touches the slot
    y = torch.randn(1, 200_000, device=DEV)
    y[0, 5] = float("inf")
    run("mml", y, 1000)  # warm the workspace paths before capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x = torch.arange(200_000, device=DEV)
        wsb = L.mmlttb_workspace_bytes(NN.OP_MINMAXLTTB, 1, 200_000, 1000, 4, 0)
        ws = torch.empty(wsb, dtype=torch.uint8, device=DEV)
        out = torch.empty((1, 1000), dtype=torch.int64, device=DEV)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            t = L.mmlttb_status_arm()
            rc = L.mmlttb_minmaxlttb(x.data_ptr(), NN.DTYPE_CODE[x.dtype], 0, y.data_ptr(), 0, 200_000, 1, 200_000,
                                     1000, 4, out.data_ptr(), None, ws.data_ptr(), wsb, s.cuda_stream)
    assert rc == 0
    assert L.mmlttb_status_poll(t, 1) == 0
    slot = int(ring[t % 1024])
    g.replay()
    torch.cuda.synchronize()
    assert int(ring[t % 1024]) == slot


@pytest.mark.parametrize("ydt,n,pad,r,n_out", [(np.float32, 20_000, 0, 4, 257), (np.float32, 20_003, 1, 2, 300),
                                               (np.float64, 16_001, 1, 8, 130), (np.float64, 24_000, 2, 6, 201),
                                               (np.float32, 9_001, 3, 4, 1000)])
def test_fused_padded_rows(ydt, n, pad, r, n_out):
    """Fused per-series kernel through the C ABI with B > resident CTAs and a
    padded row stride (y_ld > n, padding = NaN that must never be read)."""
    rng = np.random.Generator(np.random.PCG64(n + r))
    B, y_ld = 420, n + pad
    y = np.zeros((B, y_ld), dtype=ydt)
    y[:, :n] = np.cumsum(rng.standard_normal((B, n)), axis=1)
    y[:, n:] = np.nan  # padding must never be read
    y[7, ::5] = -0.0
    y[9, :n] = 2.5
    y[11, n - 1] = 1e30
    x = np.arange(n, dtype=np.int64)
    out = _minmaxlttb_abi(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n, n_out, r, y_ld)
    for i in range(B):
        assert np.array_equal(out[i], O.minmaxlttb(x, y[i, :n].astype(np.float64), n_out, r)), i


def test_batch_above_grid_limit():
    """B > 65,535 series (past the grid.y limit of the per-series kernels): the
    C entries run stream-ordered chunks over one workspace."""
    rng = np.random.Generator(np.random.PCG64(70))
    B, n = 70_001, 64
    y = np.cumsum(rng.standard_normal((B, n)), axis=1).astype(np.float32)
    x = np.arange(n, dtype=np.int64)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    rows = [0, 1, 65_534, 65_535, 65_536, 70_000]
    out = mm.minmaxlttb(xd, yd, 10, minmax_ratio=2).cpu().numpy()
    for i in rows:
        assert np.array_equal(out[i], O.minmaxlttb(x, y[i].astype(np.float64), 10, 2)), i
    out = mm.lttb(xd, yd, 12).cpu().numpy()
    for i in rows:
        assert np.array_equal(out[i], O.lttb(x, y[i], 12)), i
    mmx = mm.minmax(xd, yd, 8)
    for i in rows:
        assert np.array_equal(mmx[i].cpu().numpy(), O.minmax(y[i], 8)), i
    y[65_600, 3] = np.nan  # the status word ORs over every chunk
    with pytest.raises(errors.NonFiniteValue):
        mm.minmaxlttb(x, y, 10, minmax_ratio=2)


def test_batched_validate_row_order():
    """validate=True checks every row in one launch; the first failing row decides
    and within it NaN is reported before a decreasing x (core.py:89-92)."""
    n = 1000
    x = torch.arange(n, dtype=torch.int64, device=DEV).repeat(6, 1)
    y = torch.randn(6, n, device=DEV)
    x[2, 10] = 5  # row 2: decreasing x
    y[4, 7] = float("nan")  # row 4: NaN (later row)
    with pytest.raises(errors.NonMonotonicX):
        mm.minmaxlttb(x, y, 50, minmax_ratio=4, validate=True)
    y[1, 7] = float("inf")  # now an earlier row has a non-finite value
    with pytest.raises(errors.NonFiniteValue):
        mm.minmaxlttb(x, y, 50, minmax_ratio=4, validate=True)
    x2 = torch.arange(n, dtype=torch.int64, device=DEV)[:, None].repeat(1, 3)[:, 0]  # shared x, fine
    mm.minmaxlttb(x2, torch.randn(3, n, device=DEV), 50, minmax_ratio=4, validate=True)


K3S_CASE = """
import sys
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2305_00332_b200 as mm
from oracle import oracle as O
rng = np.random.Generator(np.random.PCG64(21))
n = 700_001
x = np.arange(n, dtype=np.int64)
y = np.cumsum(rng.standard_normal(n)) + rng.normal(0, 0.5, n)
xi = np.cumsum(rng.integers(1, 4, n)).astype(np.int64)
yd = np.repeat(np.cumsum(rng.standard_normal(n // 2 + 1)), 2)[:n].copy()
cases = [(x, y, 2000), (xi, y.astype(np.float32), 1500), (x, yd, 1800), (x.astype(np.float64) * 0.25, y, 3001)]
# group pruning / fixed-point passes: smooth, constant and stepped data (many
# mismatches or whole-group ties), decreasing-magnitude negative float x, and
# buckets of > 8192 points (groups of 2^s warp-loads, s > 0) in f64 and f32
i = np.arange(n, dtype=np.float64)
cases += [(x, np.sin(i / 3000.0) * 100 + np.sin(i / 17.0), 1400), (x, np.full(n, 3.25), 1300),
          (x, np.repeat(rng.integers(-5, 5, n // 1000 + 1), 1000)[:n].astype(np.float64), 1250),
          (-0.25 * i[::-1].copy() - 7.0, y, 1300)]
nb = 12_000_011
yb = np.cumsum(rng.standard_normal(nb))
cases += [(np.arange(nb, dtype=np.int64), yb, 1186), (np.arange(nb, dtype=np.int32), yb.astype(np.float32), 1190)]
for xx, yy, k in cases:
    got = mm.lttb(torch.from_numpy(xx).cuda(), torch.from_numpy(yy).cuda(), k).cpu().numpy()
    if not np.array_equal(got, O.lttb(xx, yy.astype(np.float64), k)):
        sys.exit('mismatch at n=%d n_out=%d' % (len(xx), k))
print('ok')
"""


@pytest.mark.parametrize("knobs", [{}, {"MMLTTB_K3C_CAND_CAP": "1"}, {"MMLTTB_K3C_CAND_CAP": "2"},
                                   {"MMLTTB_K3C_CERT_FORCE": "1"}, {"MMLTTB_K3S": "0"},
                                   {"MMLTTB_K3S_PRUNE": "0"}, {"MMLTTB_K3S_JMAX": "0"},
                                   {"MMLTTB_K3S_JMIN": "0", "MMLTTB_K3S_JMAX": "2"},
                                   {"MMLTTB_K3C_CAND_CAP": "1", "MMLTTB_K3S_JMAX": "0"},
                                   {"MMLTTB_K3C_CERT_FORCE": "1", "MMLTTB_K3S_JMIN": "0"}])
def test_lttb_k3s_single_launch(knobs):
    """K3s (one cooperative launch for full LTTB over >= 8 x SMs large buckets):
    arange / irregular integer / duplicated-point / float x, f64 and f32 y,
    smooth / constant / stepped data and buckets beyond one group size, at
    its default (group-pruned candidate search and verification, fixed-point
    passes when many buckets mismatch), with the candidate sets cut to 1-2 points
    (every bucket's pick missed: mismatches, fixed-point passes, 4b deviation
    walks and the sequential repair walk all run), with every certification
    failing (in-order exact means), without pruning, with the fixed-point passes
    off (walks only) or cut short after 2 passes, and the multi-kernel K3c
    fallback (MMLTTB_K3S=0) -- all index-exact vs the oracle."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, **knobs)
    r = subprocess.run([sys.executable, "-c", K3S_CASE], env=env, capture_output=True, text=True,
                       cwd=str(GOLD.parent.parent), timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-500:] + r.stderr[-2000:]


def test_lttb_k3s_repeatable():
    """The cross-CTA protocols of the single-launch kernel (neighbour flags,
    grid barriers, aggregate exchange, last-CTA repair) must be deterministic:
    30 back-to-back calls give identical indices."""
    rng = np.random.Generator(np.random.PCG64(5))
    n = 3_000_000
    x = torch.arange(n, dtype=torch.int64, device=DEV)
    y = torch.from_numpy(np.cumsum(rng.standard_normal(n))).to(DEV)
    first = mm.lttb(x, y, 2500)
    for _ in range(30):
        assert torch.equal(mm.lttb(x, y, 2500), first)
    assert np.array_equal(first.cpu().numpy(), O.lttb(x.cpu().numpy(), y.cpu().numpy(), 2500))


def test_lttb_tie_with_tail_element_regression():
    """Found by tools/lttb_fuzz.py (seed 2, case 42): stepped float32 y over a repeating int64 x,
    328-point buckets.  K3s's warp-level exact scan visits a lane's head / tail element before
    its vector elements; an exact area tie between the tail and an earlier element of the same
    lane kept the later index (78 of 6,429 picks off).  The scan now breaks ties by index."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, LTTB_FUZZ_ONLY="42")
    r = subprocess.run([sys.executable, "tools/lttb_fuzz.py", "43", "2"], env=env, capture_output=True, text=True,
                       cwd=str(GOLD.parent.parent), timeout=900)
    assert r.returncode == 0 and "0 mismatches" in r.stdout, r.stdout[-800:] + r.stderr[-1500:]
