"""The multi-GPU product functions at world size 2: two processes, one gloo group.

Both ranks run on cuda:0 (this pool leases one GPU per call).  Their kernels
never wait on each other -- the only cross-rank step is the host-staged gloo
all_gather inside ``sharding.all_gather_flat`` -- so this is the real product
path (``minmaxlttb_series_sharded`` / ``minmaxlttb_batch_sharded``: plan,
per-rank K1+K2 into the packed message, exchange, device merge, LTTB), not a
stand-in.  Under NCCL on an 8-GPU box the same functions run with the
in-place all_gather_into_tensor.  The reference contract is identical output
for every worker count (downsamplers.py:224-244, _kernels.py:71-78).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _series(case):
    n, xk, yk, seed = case["n"], case["x"], case["y"], case["seed"]
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.cumsum(rng.exponential(1.0, n)) if xk == "f64" else np.arange(n, dtype=np.int64) * 3
    y = np.cumsum(rng.standard_normal(n))
    y[::997] = -0.0
    y = y.astype(np.float32 if yk == "f32" else np.float64)
    return x, y


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_00332_b200 import sharding as S

        dev = torch.device("cuda", 0)
        res = []
        for case in cases:
            if case["kind"] == "series":
                x, y = _series(case)
                n, n_out, r = case["n"], case["n_out"], case["r"]
                sh = S.bucket_ranges(n, n_out, r, world)[rank]
                xs = torch.from_numpy(x[sh.lo:sh.hi]).to(dev)
                ys = torch.from_numpy(y[sh.lo:sh.hi]).to(dev)
                out = S.minmaxlttb_series_sharded(xs, ys, n, n_out, r)
                res.append(out.cpu().numpy())
            else:  # batch rows sharded, result all-gathered
                B, n, n_out, r = case["B"], case["n"], case["n_out"], case["r"]
                rng = np.random.Generator(np.random.PCG64(case["seed"]))
                y = np.cumsum(rng.standard_normal((B, n)), axis=1).astype(np.float32)
                x = np.arange(n, dtype=np.int64)
                lo, hi = S.batch_range(B, rank, world)
                out = S.minmaxlttb_batch_sharded(torch.from_numpy(x).to(dev), torch.from_numpy(y[lo:hi]).to(dev),
                                                 n_out, r, B=B, gather=True)
                if isinstance(out, list):
                    res.append([o.cpu().numpy() for o in out])
                else:
                    res.append(out.cpu().numpy())
        q.put((rank, res))
    except Exception as e:  # surface the worker's failure in the parent
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


CASES = [
    dict(kind="series", n=1_000_003, n_out=1000, r=4, x="i64", y="f32", seed=1),
    dict(kind="series", n=3_000_017, n_out=2001, r=2, x="f64", y="f32", seed=2),
    dict(kind="series", n=500_000, n_out=1500, r=32, x="f64", y="f64", seed=3),
    dict(kind="series", n=60, n_out=12, r=2, x="i64", y="f64", seed=4),
    dict(kind="batch", B=37, n=50_000, n_out=300, r=4, seed=5),
    dict(kind="batch", B=5, n=20_000, n_out=200, r=1, seed=6),
]


def test_world2_product_paths_match_single_device():
    import paper_2305_00332_b200 as mm
    from oracle import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert all(not isinstance(v, str) for v in got.values()), got
    assert all(p.exitcode == 0 for p in procs)
    dev = torch.device("cuda", 0)
    for ci, case in enumerate(CASES):
        if case["kind"] == "series":
            x, y = _series(case)
            want = O.minmaxlttb(x, y.astype(np.float64), case["n_out"], case["r"])
            single = mm.minmaxlttb(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev), case["n_out"],
                                   minmax_ratio=case["r"]).cpu().numpy()
            assert np.array_equal(single, want), ci
            for rank in range(world):  # every rank holds the full result
                assert np.array_equal(got[rank][ci], want), (ci, rank)
        else:
            rng = np.random.Generator(np.random.PCG64(case["seed"]))
            y = np.cumsum(rng.standard_normal((case["B"], case["n"])), axis=1).astype(np.float32)
            x = np.arange(case["n"], dtype=np.int64)
            for rank in range(world):
                rows = got[rank][ci]
                assert len(rows) == case["B"], (ci, rank)
                for i in range(case["B"]):
                    want = O.minmaxlttb(x, y[i].astype(np.float64), case["n_out"], case["r"])
                    assert np.array_equal(np.asarray(rows[i]).reshape(-1), want), (ci, rank, i)
