"""K1 over large closed-form sub-buckets (the flat split, and the tile mode of
the tuning build, csrc/k1_tiles.cuh), index-exact against the CPU oracle
(_kernels.py:28-78 first occurrence) on the shapes that stress the per-range
partial bookkeeping: misaligned rows
(odd N float32 batches: each row starts at a different 16-byte phase, so the
scalar head/tail extras move), constant and tied series whose first
occurrence lies in an earlier tile, sub-buckets just above the tile-mode
threshold (several edges per warp range / tile), one-tile series, bucket-range shards
(b0 > 0) and minmax / m4 with large buckets."""
import numpy as np
import pytest
import torch

import paper_2305_00332_b200 as mm
from paper_2305_00332_b200 import sharding as S
from oracle import oracle as O

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _walk(seed, shape, dt):
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.cumsum(rng.standard_normal(shape), axis=-1).astype(dt)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("B,n,n_out,r", [(1, 2_000_003, 60, 4), (3, 1_000_001, 40, 2), (5, 300_007, 12, 4),
                                         (1, 9_000, 3, 2), (2, 4_100 * 18 + 7, 20, 2)])
def test_k1_large_minmaxlttb(dt, B, n, n_out, r):
    x = np.arange(n, dtype=np.int64)
    y = _walk(B * 7 + n % 97, (B, n), dt)
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out,
                        minmax_ratio=r).cpu().numpy().reshape(B, -1)
    for i in range(B):
        assert np.array_equal(got[i], O.minmaxlttb(x, y[i].astype(np.float64), n_out, r)), i


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("kind", ["const", "ties", "plateau"])
def test_k1_large_first_occurrence(dt, kind):
    n, n_out, r = 1_500_001, 50, 4
    x = np.arange(n, dtype=np.int64)
    if kind == "const":
        y = np.full(n, 2.5, dtype=dt)
    elif kind == "ties":
        y = np.random.Generator(np.random.PCG64(3)).integers(-2, 3, n).astype(dt)
        y[::7] = -0.0
    else:  # long flat runs spanning whole tiles, extremes repeated far apart
        y = np.repeat(np.arange(n // 20_000 + 1, dtype=np.float64) % 5, 20_000)[:n].astype(dt)
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out, minmax_ratio=r)
    assert np.array_equal(got.cpu().numpy(), O.minmaxlttb(x, y.astype(np.float64), n_out, r))
    pre = mm.minmax_preselect(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out, r)
    assert np.array_equal(pre.cpu().numpy(), O.minmax_preselect(y.astype(np.float64), n_out, r))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_k1_large_minmax_m4(dt):
    n = 3_000_017
    x = np.arange(n, dtype=np.int64)
    y = _walk(11, n, dt)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    assert np.array_equal(mm.minmax(xd, yd, 100).cpu().numpy(), O.minmax(y.astype(np.float64), 100))
    assert np.array_equal(mm.m4(xd, yd, 200).cpu().numpy(), O.m4(y.astype(np.float64), 200))


@pytest.mark.parametrize("G", [2, 3, 8])
def test_k1_large_shards(G):
    n, n_out, r = 4_000_037, 200, 4
    rng = np.random.Generator(np.random.PCG64(G))
    x = np.cumsum(rng.exponential(1.0, n))
    y = _walk(G + 40, n, np.float32)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    plan = S.bucket_ranges(n, n_out, r, G)
    cap = plan[0].cap
    bufs = []
    for sh in plan:
        buf = torch.zeros((3 * cap + 1,), dtype=torch.int64, device=DEV)
        S.shard_preselect(xd[sh.lo:sh.hi], yd[sh.lo:sh.hi], n, n_out, r, sh, packed=buf)
        bufs.append(buf)
    got = S.lttb_merged(*S.merge_packed(torch.cat(bufs), G, cap), n_out, r)
    assert np.array_equal(got.cpu().numpy(), O.minmaxlttb(x, y.astype(np.float64), n_out, r))


def test_k1_large_repeatable():
    n = 20_000_000
    x = torch.arange(n, device=DEV)
    y = torch.randn(n, device=DEV).cumsum(0)
    first = mm.minmaxlttb(x, y, 2000, minmax_ratio=4)
    for _ in range(20):
        assert torch.equal(mm.minmaxlttb(x, y, 2000, minmax_ratio=4), first)
