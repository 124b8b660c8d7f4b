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


@pytest.mark.parametrize("G,n,n_out,r", [(1, 200_000, 500, 4), (4, 1_000_003, 1000, 4), (8, 3_000_017, 2001, 2)])
def test_p2p_exchange_kernels_virtual_ranks(G, n, n_out, r):
    """mmlttb_p2p_publish / mmlttb_p2p_merge with G virtual ranks on one GPU.

    Each virtual rank gets its own plain device buffer + flag pad; all
    publishes of an epoch are stream-ordered before all merges, so nothing
    waits on a kernel that has not been launched.  Four epochs exercise both
    buffer slots and the ack wait (epoch e waits for the acks of e-2).
    """
    rng = np.random.Generator(np.random.PCG64(G * 7 + r))
    x = np.cumsum(rng.exponential(1.0, n))
    y = np.cumsum(rng.standard_normal(n)).astype(np.float32)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    plan = S.bucket_ranges(n, n_out, r, G)
    cap, W = plan[0].cap, 3 * plan[0].cap + 1
    sets = [S.shard_preselect(xd[sh.lo:sh.hi], yd[sh.lo:sh.hi], n, n_out, r, sh) for sh in plan]
    bufs = [torch.full((2 * G * W,), -7, dtype=torch.int64, device=DEV) for _ in range(G)]
    pads = [torch.zeros(2 * G, dtype=torch.int32, device=DEV) for _ in range(G)]
    pb = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    pp = torch.tensor([p.data_ptr() for p in pads], dtype=torch.int64, device=DEV)
    L = mm._native.lib()
    st = mm._native.stream_ptr(DEV)
    want = O.minmaxlttb(x, y.astype(np.float64), n_out, r)
    for epoch in range(1, 5):
        for g in range(G):
            idx, xs, ys, cnt = sets[g]
            mm._native.check(L.mmlttb_p2p_publish(idx.data_ptr(), xs.data_ptr(), ys.data_ptr(), cnt.data_ptr(), cap,
                                                  pb.data_ptr(), pp.data_ptr(), pads[g].data_ptr(), G, g, epoch, st),
                             "p2p_publish")
        for g in range(G):
            oi = torch.empty(G * cap, dtype=torch.int64, device=DEV)
            ox = torch.empty(G * cap, dtype=torch.float64, device=DEV)
            oy = torch.empty(G * cap, dtype=torch.float64, device=DEV)
            om = torch.empty(1, dtype=torch.int64, device=DEV)
            mm._native.check(L.mmlttb_p2p_merge(bufs[g].data_ptr(), pads[g].data_ptr(), pp.data_ptr(), G, g, cap,
                                                epoch, oi.data_ptr(), ox.data_ptr(), oy.data_ptr(), om.data_ptr(), st),
                             "p2p_merge")
            out = S.lttb_merged(oi, ox, oy, om, n_out, r).cpu().numpy()
            assert np.array_equal(out, want), (epoch, g)
        torch.cuda.synchronize()
        for g in range(G):
            assert pads[g].cpu().tolist() == [epoch] * (2 * G)


P2P_WORLD1 = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2305_00332_b200 import sharding as S
from oracle import oracle as O
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
rng = np.random.Generator(np.random.PCG64(11))
n = 500_000
x = np.arange(n, dtype=np.int64)
y = rng.standard_normal(n).astype(np.float32)
want = O.minmaxlttb(x, y.astype(np.float64), 1000, 4)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
for it in range(5):
    out = S.minmaxlttb_series_sharded(xd, yd, n, 1000, 4, exchange_mode="p2p")
    assert np.array_equal(out.cpu().numpy(), want), it
dist.destroy_process_group()
print("P2P_OK")
'''


def test_series_sharded_p2p_world1():
    """The symmetric-memory exchange end to end through torch.distributed (world 1)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", P2P_WORLD1], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0 and "P2P_OK" in p.stdout, p.stdout[-2000:] + p.stderr[-4000:]


@pytest.mark.parametrize("G,n,n_out,r", [(1, 100_000, 300, 4), (3, 1_000_003, 1000, 4), (8, 3_000_017, 2001, 2)])
def test_virtual_shards_packed_merge(G, n, n_out, r):
    """K1 + K2 writing the exchange message in place (shard_preselect(packed=)),
    the concatenation an all_gather produces, then mmlttb_merge_packed."""
    rng = np.random.Generator(np.random.PCG64(G * 31 + r))
    x = np.cumsum(rng.exponential(1.0, n))
    y = np.cumsum(rng.standard_normal(n)).astype(np.float32)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    plan = S.bucket_ranges(n, n_out, r, G)
    cap = plan[0].cap
    bufs = []
    for sh in plan:
        buf = torch.full((3 * cap + 1,), -9, dtype=torch.int64, device=DEV)
        S.shard_preselect(xd[sh.lo:sh.hi], yd[sh.lo:sh.hi], n, n_out, r, sh, packed=buf)
        bufs.append(buf)
    out = S.lttb_merged(*S.merge_packed(torch.cat(bufs), G, cap), n_out, r).cpu().numpy()
    assert np.array_equal(out, O.minmaxlttb(x, y.astype(np.float64), n_out, r))
