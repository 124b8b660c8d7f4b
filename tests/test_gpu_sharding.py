"""Device kernels of the multi-GPU paths, exercised on one GPU.

G "virtual shards" run the real per-rank device code (mmlttb_shard_preselect,
pack) one after another on cuda:0; the all_gather is replaced by the
concatenation it produces, then the real device merge + LTTB runs.  (Running
G ranks that wait on each other on one GPU is not done -- see
B200_PROFILING.md; the collective itself is covered by the gloo test.)
"""
import numpy as np
import pytest
import torch

import paper_2305_00332_b200 as mm
from paper_2305_00332_b200 import sharding as S
from oracle import oracle as O

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.mark.parametrize("G,n,n_out,r", [(1, 100_000, 300, 4), (2, 1_000_003, 1000, 4), (8, 3_000_017, 2001, 2),
                                         (8, 500_000, 1500, 32), (8, 60, 12, 2)])
def test_virtual_shards_match_single_device(G, n, n_out, r):
    rng = np.random.Generator(np.random.PCG64(G * 1000 + r))
    x = np.cumsum(rng.exponential(1.0, n))
    y = np.cumsum(rng.standard_normal(n)).astype(np.float32)
    y[::997] = -0.0
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    plan = S.bucket_ranges(n, n_out, r, G)
    bufs = []
    for sh in plan:
        idx, xs, ys, cnt = S.shard_preselect(xd[sh.lo:sh.hi], yd[sh.lo:sh.hi], n, n_out, r, sh)
        bufs.append(S.pack(idx, xs, ys, cnt, sh.cap))
    gi, gx, gy, gc = S.unpack(torch.cat(bufs), G, plan[0].cap)
    out = S.merge_and_lttb(gi, gx, gy, gc, n_out, r).cpu().numpy()
    want = O.minmaxlttb(x, y.astype(np.float64), n_out, r)
    assert np.array_equal(out, want)
    single = mm.minmaxlttb(xd, yd, n_out, minmax_ratio=r).cpu().numpy()
    assert np.array_equal(single, want)


def test_series_sharded_world1():
    rng = np.random.Generator(np.random.PCG64(3))
    n = 400_000
    x = np.arange(n, dtype=np.int64)
    y = rng.standard_normal(n).astype(np.float32)
    out = S.minmaxlttb_series_sharded(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n, 800, 4)
    assert np.array_equal(out.cpu().numpy(), O.minmaxlttb(x, y.astype(np.float64), 800, 4))


def test_batch_sharded_local_rows():
    rng = np.random.Generator(np.random.PCG64(4))
    B, n = 12, 50_000
    y = np.cumsum(rng.standard_normal((B, n)), axis=1).astype(np.float32)
    x = np.arange(n, dtype=np.int64)
    lo, hi = S.batch_range(B, 1, 3)
    out = S.minmaxlttb_batch_sharded(torch.from_numpy(x).to(DEV), torch.from_numpy(y[lo:hi]).to(DEV), 200, 4)
    for i, row in enumerate(out.cpu().numpy()):
        assert np.array_equal(row, O.minmaxlttb(x, y[lo + i].astype(np.float64), 200, 4))
