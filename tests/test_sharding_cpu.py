"""Multi-rank host logic on CPU: world_size 2 over gloo.

The per-rank device kernels are stood in for by the CPU oracle here (tests
only, monkeypatched inside each worker); everything else -- the
bucket-range plan, the packed message layout, the host-staged gloo exchange
(``all_gather_flat``), and the calling sequence of the product functions
``minmaxlttb_series_sharded`` / ``minmaxlttb_batch_sharded(gather=True)``
themselves -- is the product's host code, and the result must equal the
single-process reference output.  tests/test_gpu_multirank.py runs the same
functions with the real kernels.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_00332_b200 import sharding as S
from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_batch_range_covers():
    for B in (1, 7, 4096, 4097):
        for G in (1, 2, 3, 8):
            r = [S.batch_range(B, i, G) for i in range(G)]
            assert r[0][0] == 0 and r[-1][1] == B
            assert all(r[i][1] == r[i + 1][0] for i in range(G - 1))
            assert max(h - l for l, h in r) - min(h - l for l, h in r) <= 1


def test_bucket_ranges_partition_the_series():
    for n, n_out, r, G in ((1000, 30, 4, 2), (10_007, 101, 6, 8), (2_000_000_000, 4000, 4, 8), (50, 10, 2, 8)):
        plan = S.bucket_ranges(n, n_out, r, G)
        k = (n_out - 2) * (r // 2)
        assert plan[0].b0 == 0 and plan[-1].b1 == k and plan[0].lo == 0 and plan[-1].hi == n
        for a, b in zip(plan, plan[1:]):
            assert a.b1 == b.b0 and a.hi == b.lo
        for sh in plan:  # every owned sub-bucket lies inside the owned elements
            if sh.b1 > sh.b0:
                assert 1 + (sh.b0 * (n - 2)) // k >= sh.lo and 1 + (sh.b1 * (n - 2)) // k <= sh.hi
            assert sh.cap >= 2 * (sh.b1 - sh.b0) + 2


def _local_oracle(x, y, n, n_out, r, sh):
    """Stand-in for mmlttb_shard_preselect (tests only)."""
    k = sh.k
    bounds = O.partition(1, n - 1, k)[sh.b0:sh.b1 + 1] - sh.lo
    ys = y[sh.lo:sh.hi].astype(np.float64)
    idx = []
    if sh.b1 > sh.b0:
        mn, mx = O.extrema_by_bucket(ys, bounds)
        for a, b in zip(mn + sh.lo, mx + sh.lo):
            lo, hi = min(a, b), max(a, b)
            idx.append(lo)
            if hi != lo:
                idx.append(hi)
    if sh.emit_first:
        idx = [0] + idx
    if sh.emit_last:
        idx = idx + [n - 1]
    idx = np.array(idx, dtype=np.int64)
    cap = sh.cap
    pi = torch.zeros(cap, dtype=torch.int64)
    px = torch.zeros(cap, dtype=torch.float64)
    py = torch.zeros(cap, dtype=torch.float64)
    pi[: idx.shape[0]] = torch.from_numpy(idx)
    px[: idx.shape[0]] = torch.from_numpy(x[idx].astype(np.float64))
    py[: idx.shape[0]] = torch.from_numpy(y[idx].astype(np.float64))
    return pi, px, py, torch.tensor([idx.shape[0]], dtype=torch.int64)


def _fake_shard_preselect(x_shard, y_shard, n, n_out, r_ps, shard, packed=None):
    """mmlttb_shard_preselect stand-in: writes the rank's set into the packed layout."""
    x = np.zeros(n)  # only [lo, hi) is read
    y = np.zeros(n, dtype=np.float32)
    x[shard.lo:shard.hi] = x_shard.numpy()
    y[shard.lo:shard.hi] = y_shard.numpy()
    pi, px, py, cnt = _local_oracle(x, y, n, n_out, r_ps, shard)
    cap = shard.cap
    packed[:cap] = pi
    packed[cap:2 * cap] = px.view(torch.int64)
    packed[2 * cap:3 * cap] = py.view(torch.int64)
    packed[3 * cap:] = cnt
    return pi, px, py, cnt


def _fake_merge_packed(allbuf, world, cap):
    """mmlttb_merge_packed stand-in: rank-order concatenation of the messages."""
    gi, gx, gy, gc = S.unpack(allbuf, world, cap)
    mi = torch.cat([gi[g, : gc[g]] for g in range(world)])
    mx = torch.cat([gx[g, : gc[g]] for g in range(world)])
    my = torch.cat([gy[g, : gc[g]] for g in range(world)])
    return mi, mx, my, torch.tensor([mi.shape[0]])


def _fake_lttb_merged(oi, ox, oy, om, n_out, r_ps):
    m = int(om[0])
    return torch.from_numpy(oi[:m].numpy()[O.lttb(ox[:m].numpy(), oy[:m].numpy(), n_out)])


def _fake_batch(b, n_out, r_ps):
    y = np.asarray(b._y_in)
    x = np.asarray(b._x_in)
    return torch.from_numpy(np.stack([O.minmaxlttb(x, row.astype(np.float64), n_out, r_ps) for row in y]))


def _product_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S.shard_preselect = _fake_shard_preselect
    S.merge_packed = _fake_merge_packed
    S.lttb_merged = _fake_lttb_merged
    S._minmaxlttb_batch = _fake_batch
    try:
        rng = np.random.Generator(np.random.PCG64(12))
        n, n_out, r = 100_003, 301, 4
        x = np.cumsum(rng.exponential(1.0, n))
        y = np.cumsum(rng.standard_normal(n)).astype(np.float32)
        sh = S.bucket_ranges(n, n_out, r, world)[rank]
        got = S.minmaxlttb_series_sharded(torch.from_numpy(x[sh.lo:sh.hi]), torch.from_numpy(y[sh.lo:sh.hi]),
                                          n, n_out, r).numpy()
        ok1 = bool(np.array_equal(got, O.minmaxlttb(x, y.astype(np.float64), n_out, r)))
        B, nb = 7, 3_000  # uneven split: rank 0 holds 3 rows, rank 1 holds 4
        yb = np.cumsum(rng.standard_normal((B, nb)), axis=1).astype(np.float32)
        xb = np.arange(nb, dtype=np.int64)
        lo, hi = S.batch_range(B, rank, world)
        allrows = S.minmaxlttb_batch_sharded(xb, yb[lo:hi], 100, 4, B=B, gather=True).numpy()
        want = np.stack([O.minmaxlttb(xb, row.astype(np.float64), 100, 4) for row in yb])
        ok2 = allrows.shape == want.shape and bool(np.array_equal(allrows, want))
        try:
            S.minmaxlttb_batch_sharded(xb, yb[lo:hi], 100, 4, gather=True)
            ok3 = False
        except ValueError:  # B is required with gather=True (rows may be split unevenly)
            ok3 = True
        q.put((rank, ok1, ok2, ok3))
    finally:
        dist.destroy_process_group()


def test_product_sharded_functions_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_product_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(a and b and c for _, a, b, c in res), res


def test_batch_sharded_checks_in_reference_order():
    """the batch-sharded entry raises the reference's classes before any compute."""
    from paper_2305_00332_b200 import errors

    x = np.arange(100, dtype=np.int64)
    y = np.zeros((2, 100), dtype=np.float32)
    with pytest.raises(errors.NOutOfRange):
        S.minmaxlttb_batch_sharded(x, y, 2, 4)
    with pytest.raises(errors.BadPreselectionRatio):
        S.minmaxlttb_batch_sharded(x, y, 10, 3)
    with pytest.raises(errors.RatioTooLargeForSeries):
        S.minmaxlttb_batch_sharded(x, y, 90, 4)
    with pytest.raises(errors.OddNOut):
        S.minmaxlttb_batch_sharded(x, y, 11, 1)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.Generator(np.random.PCG64(11))
        n, n_out, r = 200_003, 401, 4
        x = np.cumsum(rng.exponential(1.0, n))
        y = np.cumsum(rng.standard_normal(n)).astype(np.float32)
        y[::1013] = -0.0
        plan = S.bucket_ranges(n, n_out, r, world)
        sh = plan[rank]
        pi, px, py, cnt = _local_oracle(x, y, n, n_out, r, sh)
        buf = S.pack(pi, px, py, cnt, sh.cap)
        allbuf = S.exchange(buf, world)
        gi, gx, gy, gc = S.unpack(allbuf, world, sh.cap)
        parts = [(gi[g, : gc[g]], gx[g, : gc[g]], gy[g, : gc[g]]) for g in range(world)]
        mi = torch.cat([p[0] for p in parts]).numpy()
        mx_ = torch.cat([p[1] for p in parts]).numpy()
        my = torch.cat([p[2] for p in parts]).numpy()
        got = mi[O.lttb(mx_, my, n_out)]
        want = O.minmaxlttb(x, y.astype(np.float64), n_out, r)
        q.put((rank, bool(np.array_equal(got, want)), int(gc.sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_bucket_range_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert len({m for _, _, m in res}) == 1
