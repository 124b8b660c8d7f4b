"""Multi-rank host logic on CPU: world_size 2 over gloo.

The per-rank device compute (K1 + K2 on a shard) is stood in for by the CPU
oracle here (tests only); everything else -- the bucket-range plan, the
packed message layout, the all_gather exchange, unpacking and rank-order
merge -- is the product's host code, and the result must equal the
single-process reference output.
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
