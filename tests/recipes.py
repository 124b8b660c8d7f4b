"""Seeded synthetic inputs for BASELINE.json's five configs (C1-C5).

The reference's own datagen uses numpy PCG64 (``datagen.py:105``); these
recipes follow BASELINE.json's config strings, with the open choices (seeds,
noise sigma, spike law, chunking) fixed here and recorded in DESIGN.md.
Everything is generated on the host with numpy so the GPU path and the oracle
see bit-identical inputs.  C5 is defined chunk-by-chunk (fixed chunk size) so
it can be streamed to the device without a 24 GB host copy.
"""
from __future__ import annotations

import numpy as np

C5_CHUNK = 1 << 25

CONFIGS = {
    "C1": dict(n=1_000_000, n_out=1000, r_ps=(4,), op="minmaxlttb"),
    "C2": dict(n=10_000_000, n_out=2000, r_ps=(), op="lttb"),
    "C3": dict(n=100_000_000, n_out=2000, r_ps=(2, 4, 8, 16, 32), op="minmaxlttb"),
    "C4": dict(n=1_000_000, n_out=1000, r_ps=(4,), op="minmaxlttb", batch=4096),
    "C5": dict(n=2_000_000_000, n_out=4000, r_ps=(4,), op="minmaxlttb"),
}


def c1(n: int = 1_000_000):
    """int64 arange x; float64 random walk y (cumsum N(0,1)), PCG64(0)."""
    rng = np.random.Generator(np.random.PCG64(0))
    return np.arange(n, dtype=np.int64), np.cumsum(rng.standard_normal(n))


def c2(n: int = 10_000_000):
    """float64 walk + N(0, 0.5) noise + 0.1% spikes of +-50 sigma (sigma = 0.5), PCG64(2)."""
    rng = np.random.Generator(np.random.PCG64(2))
    walk = np.cumsum(rng.standard_normal(n))
    noise = rng.normal(0.0, 0.5, n)
    spike = rng.random(n) < 0.001
    sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    y = walk + noise + np.where(spike, sign * 50.0 * 0.5, 0.0)
    return np.arange(n, dtype=np.int64), y


def c3_y(n: int = 100_000_000, seed: int = 3, chunk: int = 1 << 26) -> np.ndarray:
    """float32 sin(2 pi i/1e3) + sin(2 pi i/1e5) + sin(2 pi i/1e7) + N(0,1), computed in f64."""
    rng = np.random.Generator(np.random.PCG64(seed))
    y = np.empty(n, dtype=np.float32)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        i = np.arange(lo, hi, dtype=np.float64)
        v = np.sin(2.0 * np.pi * i / 1e3)
        v += np.sin(2.0 * np.pi * i / 1e5)
        v += np.sin(2.0 * np.pi * i / 1e7)
        v += rng.standard_normal(hi - lo)
        y[lo:hi] = v
    return y


def c3(n: int = 100_000_000):
    return np.arange(n, dtype=np.int64), c3_y(n)


def c4_series(s: int, n: int = 1_000_000) -> np.ndarray:
    """Series s of the C4 batch: float32 random walk from PCG64(s)."""
    rng = np.random.Generator(np.random.PCG64(s))
    return np.cumsum(rng.standard_normal(n)).astype(np.float32)


def c4(batch: int = 4096, n: int = 1_000_000, series=None):
    ids = range(batch) if series is None else series
    y = np.stack([c4_series(s, n) for s in ids])
    return np.arange(n, dtype=np.int64), y


def c5_chunks(n: int = 2_000_000_000, chunk: int = C5_CHUNK):
    """Yield (lo, x_f64, y_f32) chunks of C5, PCG64(5), fixed draw order per chunk.

    x = cumsum(Exp(1)) (non-decreasing float64 timestamps); y = float32 random
    walk (N(0,1) steps, sigma = 1) with 1% of points offset by +-50 sigma.
    """
    rng = np.random.Generator(np.random.PCG64(5))
    cx = 0.0
    cy = 0.0
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        gaps = rng.exponential(1.0, m)
        steps = rng.standard_normal(m)
        spike = rng.random(m) < 0.01
        sign = np.where(rng.random(m) < 0.5, -1.0, 1.0)
        gaps[0] += cx
        x = np.cumsum(gaps)
        steps[0] += cy
        walk = np.cumsum(steps)
        cx = float(x[-1])
        cy = float(walk[-1])
        y = (walk + np.where(spike, sign * 50.0, 0.0)).astype(np.float32)
        yield lo, x, y


def c5(n: int = 2_000_000_000, chunk: int = C5_CHUNK):
    x = np.empty(n, dtype=np.float64)
    y = np.empty(n, dtype=np.float32)
    for lo, xc, yc in c5_chunks(n, chunk):
        x[lo:lo + xc.shape[0]] = xc
        y[lo:lo + yc.shape[0]] = yc
    return x, y
