"""Deterministic adversarial small cases.

``make_case(i)`` regenerates case i bit-for-bit from its index, so the golden
file only stores parameters, an input digest and the reference's output.
Kinds cover: random walks, float32 with ties, +-0.0 runs, denormals, constant
series, collinear series (all LTTB areas tie), huge magnitudes (areas overflow
to inf/NaN), irregular and repeated x, large int64 x.
"""
from __future__ import annotations

import hashlib

import numpy as np

KINDS = (
    "walk64", "walk32", "ties32", "signed_zero", "denormal", "constant", "collinear",
    "huge", "irregular_x", "repeated_x", "bigint_x", "steps",
)
OPS = ("minmaxlttb", "lttb", "minmax", "minmax_preselect", "m4")
N_CASES = 1200


def _n(rng, i):
    if i % 10 == 0:
        return int(rng.integers(1000, 4000))
    if i % 3 == 0:
        return int(rng.integers(3, 12))
    return int(rng.integers(12, 600))


def _series(kind, n, rng):
    if kind == "walk64":
        return np.arange(n, dtype=np.int64), np.cumsum(rng.standard_normal(n))
    if kind == "walk32":
        return np.arange(n, dtype=np.int64), np.cumsum(rng.standard_normal(n)).astype(np.float32)
    if kind == "ties32":
        return np.arange(n, dtype=np.int64), rng.integers(-2, 3, n).astype(np.float32)
    if kind == "signed_zero":
        y = np.where(rng.random(n) < 0.5, -0.0, 0.0)
        y[rng.random(n) < 0.05] = 1.0
        return np.arange(n, dtype=np.int64), y.astype(np.float64)
    if kind == "denormal":
        vals = np.array([5e-324, -5e-324, 0.0, -0.0, 1e-310, -1e-310, 2.5e-320], dtype=np.float64)
        return np.arange(n, dtype=np.int64), vals[rng.integers(0, vals.shape[0], n)]
    if kind == "constant":
        return np.arange(n, dtype=np.int64), np.full(n, float(rng.integers(-5, 5)))
    if kind == "collinear":
        x = np.arange(n, dtype=np.int64)
        return x, 2.0 * x.astype(np.float64) + 1.0
    if kind == "huge":
        vals = np.array([1e300, -1e300, 1.7e308, -1.7e308, 0.0, 1.0], dtype=np.float64)
        return np.arange(n, dtype=np.int64), vals[rng.integers(0, vals.shape[0], n)]
    if kind == "irregular_x":
        return np.cumsum(rng.exponential(1.0, n)), np.cumsum(rng.standard_normal(n)).astype(np.float32)
    if kind == "repeated_x":
        x = np.sort(rng.integers(0, max(2, n // 3), n)).astype(np.float64)
        return x, rng.standard_normal(n)
    if kind == "bigint_x":
        return (np.int64(10**15) + 7 * np.arange(n, dtype=np.int64)), rng.standard_normal(n)
    if kind == "steps":
        return np.arange(n, dtype=np.int64), np.repeat(rng.standard_normal(n // 4 + 1), 4)[:n].copy()
    raise ValueError(kind)


def _params(op, n, rng):
    """n_out / r_ps, mostly valid, ~8% deliberately invalid (error parity)."""
    bad = rng.random() < 0.08
    if op == "lttb":
        n_out = int(rng.integers(3, min(n, 200) + 1)) if n >= 3 else 3
        if bad:
            n_out = int(rng.choice([2, n + 1]))
        return n_out, 0
    if op in ("minmax", "m4"):
        step = 2 if op == "minmax" else 4
        hi = min(n, 200)
        n_out = step * int(rng.integers(1, max(2, hi // step + 1)))
        if n_out < 3:
            n_out = 4 if step == 2 or n >= 4 else 4
        if bad:
            n_out = int(rng.choice([n_out + 1, n + 2, 2]))
        return n_out, 0
    # minmaxlttb / minmax_preselect
    r_ps = int(rng.choice([1, 2, 2, 4, 4, 6, 8, 16, 32])) if op == "minmaxlttb" else int(rng.choice([2, 4, 6, 8, 16]))
    if r_ps == 1:
        hi = min(n, 200)
        n_out = 2 * int(rng.integers(2, max(3, hi // 2 + 1)))
        n_out = min(n_out, n - (n % 2)) if n >= 4 else 4
    else:
        kmax = (n - 2) // (r_ps // 2)
        hi = min(n, 200, kmax + 2)
        n_out = int(rng.integers(3, hi + 1)) if hi >= 3 else 3
    if bad:
        r_ps = int(rng.choice([0, 3, 5, 64, 128]))
    return n_out, r_ps


def make_case(i: int) -> dict:
    rng = np.random.Generator(np.random.PCG64(10_000 + i))
    kind = KINDS[i % len(KINDS)]
    op = OPS[(i // len(KINDS)) % len(OPS)]
    n = _n(rng, i)
    x, y = _series(kind, n, rng)
    n_out, r_ps = _params(op, n, rng)
    return dict(i=i, kind=kind, op=op, n=n, n_out=n_out, r_ps=r_ps, x=x, y=y)


def digest(x: np.ndarray, y: np.ndarray) -> str:
    h = hashlib.sha256()
    for a in (x, y):
        h.update(str(a.dtype).encode())
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]
