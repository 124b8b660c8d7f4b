"""Randomised parity sweep over every device dispatch path (hypothesis-style,
seeded): K1 flat / chunked / 8-lane / warp-per-bucket, the fused batch
kernel, the fused and cooperative post kernels, K3a tables+scan / jump, K3c
large-bucket LTTB, minmax / m4 / preselect, f32/f64 y and all x dtypes.
Each case runs in a fresh interpreter only when it needs an env knob."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_2305_00332_b200 as mm
from oracle import oracle as O

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)
XT = [np.int64, np.int32, np.float64, np.float32]


def _series(rng, B, n, ydt, xdt, kind):
    if kind == "walk":
        y = np.cumsum(rng.standard_normal((B, n)), axis=1)
    elif kind == "ties":
        y = rng.integers(-3, 4, (B, n)).astype(np.float64)
        y[:, ::5] = -0.0
    else:
        y = rng.standard_normal((B, n))
    y = y.astype(ydt)
    if xdt in (np.float64, np.float32):
        x = np.cumsum(rng.exponential(1.0, n)).astype(xdt)
        x = np.maximum.accumulate(x)  # float32 rounding must stay non-decreasing
    else:
        x = (np.arange(n) * int(rng.integers(1, 4))).astype(xdt)
    return x, y


def _check_case(seed):
    rng = np.random.Generator(np.random.PCG64(1000 + seed))
    B = int(rng.choice([1, 1, 3, 150, 160]))
    n = int(rng.choice([50, 3_001, 40_000, 300_000])) if B > 3 else int(rng.choice([50, 9_001, 600_000, 3_000_000]))
    ydt = rng.choice([np.float32, np.float64])
    xdt = XT[int(rng.integers(0, 4))]
    kind = str(rng.choice(["walk", "ties", "noise"]))
    x, y = _series(rng, B, n, ydt, xdt, kind)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    op = str(rng.choice(["minmaxlttb", "minmaxlttb", "lttb", "minmax", "m4", "preselect"]))
    hi = min(n, 2500)
    if op == "minmaxlttb":
        r = int(rng.choice([2, 4, 6, 8, 16, 32, 80]))
        kmax = (n - 2) // (r // 2)
        n_out = int(rng.integers(3, max(4, min(hi, kmax + 2)) + 1))
        if (n_out - 2) * (r // 2) > n - 2:
            return
        got = mm.minmaxlttb(xd, yd, n_out, minmax_ratio=r).cpu().numpy().reshape(B, -1)
        for i in range(B):
            want = O.minmaxlttb(x, y[i].astype(np.float64), n_out, r)
            assert np.array_equal(got[i], want), (seed, op, B, n, n_out, r, i)
    elif op == "lttb":
        n_out = int(rng.integers(3, hi + 1))
        got = mm.lttb(xd, yd, n_out).cpu().numpy().reshape(B, -1)
        for i in range(0, B, max(1, B // 7)):
            assert np.array_equal(got[i], O.lttb(x, y[i], n_out)), (seed, op, B, n, n_out, i)
    elif op in ("minmax", "m4"):
        step = 2 if op == "minmax" else 4
        n_out = step * int(rng.integers(1, max(2, hi // step)))
        if n_out < 3 or n_out > n:
            return
        fn = mm.minmax if op == "minmax" else mm.m4
        orc = O.minmax if op == "minmax" else O.m4
        got = fn(xd, yd, n_out)
        rows = got if isinstance(got, list) else list(got.reshape(B, -1))
        for i in range(0, B, max(1, B // 7)):
            assert np.array_equal(rows[i].cpu().numpy().reshape(-1), orc(y[i], n_out)), (seed, op, B, n, n_out, i)
    else:
        r = int(rng.choice([2, 4, 8]))
        kmax = (n - 2) // (r // 2)
        n_out = int(rng.integers(3, max(4, min(hi, kmax + 2)) + 1))
        if (n_out - 2) * (r // 2) > n - 2:
            return
        got = mm.minmax_preselect(xd, yd, n_out, r)
        rows = got if isinstance(got, list) else list(got.reshape(B, -1))
        for i in range(0, B, max(1, B // 7)):
            assert np.array_equal(rows[i].cpu().numpy().reshape(-1), O.minmax_preselect(y[i], n_out, r)), (seed, op, i)


@pytest.mark.parametrize("seed", range(60))
def test_random_paths(seed):
    _check_case(seed)


@pytest.mark.parametrize("knob", ["MMLTTB_NO_FUSED=1", "MMLTTB_NO_POST_FUSED=1", "MMLTTB_K1_FLAT_WARPS=0",
                                  "MMLTTB_K3C_FLAT=0", "MMLTTB_K3C_CERT_FORCE=1", "MMLTTB_K3C_XAFF=0",
                                  "MMLTTB_K3C_REPAIR_SMEM=0"])
def test_random_paths_with_knobs(knob):
    """The alternative kernels behind the A/B knobs stay exact too."""
    k, v = knob.split("=")
    code = ("import sys; sys.path[:0] = ['.', 'tests'];"
            "import test_gpu_random as T\nfor s in range(0, 60, 3): T._check_case(s)\nprint('ok')")
    env = dict(os.environ, **{k: v})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=root, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
