"""Small cases over every cross-CTA protocol of libmmlttb.so, for compute-sanitizer.

Run under `tools/sanitize.sh` (memcheck / racecheck / synccheck / initcheck).
Each case runs the product path on cuda:0 at a size the sanitizers finish in
seconds and checks the result index-exactly against the CPU oracle (test
infrastructure only), so a protocol that misbehaves under the sanitizer's
changed scheduling also shows up as a parity failure.

Protocols covered:
  k1_flat      K1 flat split, per-(bucket, warp) partials combined by the
               bucket's last-arriving warp (threadfence reduction)
  k1_chunked   K1 chunked buckets (explicit bounds / batches), last-arriver combine
  post_smem    K2+K3a in one CTA per series, state in shared memory (C1 shape)
  c3_multi     K2 k_compact_pairs (multi-CTA offsets) + K3a tables + block scan
  jump         k_lttb_jump (33-64-point LTTB buckets, shared-memory pointer jumping)
  k3c_flat     full LTTB, K3c flat passes: means/verify last-arriver partials,
               fix-up, verify2, repair_smem
  k3c_repair   same with the candidate sets cut to one point (forces the
               sequential repair walk and its exact re-scans)
  k3c_cert     same with every certification failing (in-order exact means)
  k3c_batch    K3c per-bucket CTAs (B = 2)
  fused        k_mmlttb_fused (one CTA per series, B >= 148)
  minmax_m4    k_compact (single CTA), m4 first/last
  validate     k_validate (batched TimeSeries invariants)
  shards       bucket-range shards + k_merge_packed (virtual ranks)
  p2p          k_p2p_publish / k_p2p_merge epoch flags with 4 virtual ranks
  raster       k_raster
"""
from __future__ import annotations

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2305_00332_b200 as mm  # noqa: E402
from paper_2305_00332_b200 import sharding as S  # noqa: E402
from oracle import oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)


def _rw(n, seed, dt=np.float32):
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.cumsum(rng.standard_normal(n)).astype(dt)


def _eq(got, want, what):
    got = got.cpu().numpy() if isinstance(got, torch.Tensor) else np.asarray(got)
    assert np.array_equal(got, want), f"{what}: differs from the oracle"


def case_k1_flat():
    n = 3_000_000
    x = np.arange(n, dtype=np.int64)
    y = _rw(n, 1)
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 100, minmax_ratio=4)
    _eq(got, O.minmaxlttb(x, y.astype(np.float64), 100, 4), "k1_flat")


def case_k1_chunked():
    B, n = 3, 400_000
    x = np.arange(n, dtype=np.int64)
    ys = np.stack([_rw(n, 10 + i) for i in range(B)])
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(ys).to(DEV), 40, minmax_ratio=2)
    for i in range(B):
        _eq(got[i], O.minmaxlttb(x, ys[i].astype(np.float64), 40, 2), f"k1_chunked row {i}")


def case_post_smem():
    n = 200_000
    x = np.arange(n, dtype=np.int64)
    y = _rw(n, 2, np.float64)
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 1000, minmax_ratio=4)
    _eq(got, O.minmaxlttb(x, y, 1000, 4), "post_smem")


def case_c3_multi():
    n = 1_000_000
    x = np.arange(n, dtype=np.int64)
    y = _rw(n, 3)
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 2000, minmax_ratio=4)
    _eq(got, O.minmaxlttb(x, y.astype(np.float64), 2000, 4), "c3_multi")


def case_jump():
    n = 100_000
    x = np.arange(n, dtype=np.int64)
    y = _rw(n, 4, np.float64)
    got = mm.lttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), 2500)  # ~40-point buckets
    _eq(got, O.lttb(x, y, 2500), "jump")


def _k3c(seed, B=1):
    n = 300_000
    x = np.arange(n, dtype=np.int64)
    ys = np.stack([_rw(n, seed + i, np.float64) for i in range(B)])
    got = mm.lttb(torch.from_numpy(x).to(DEV), torch.from_numpy(ys if B > 1 else ys[0]).to(DEV), 50)
    got = got.reshape(B, -1)
    for i in range(B):
        _eq(got[i], O.lttb(x, ys[i], 50), f"k3c row {i}")


def case_k3c_flat():
    _k3c(5)


def case_k3c_repair():
    os.environ["MMLTTB_K3C_CAND_CAP"] = "1"  # read once per process: run this case in its own process
    _k3c(6)


def case_k3c_cert():
    os.environ["MMLTTB_K3C_CERT_FORCE"] = "1"  # read once per process
    _k3c(7)


def case_k3c_batch():
    _k3c(8, B=2)


def case_fused():
    B, n = 148, 20_000
    x = np.arange(n, dtype=np.int64)
    ys = np.stack([_rw(n, 100 + i) for i in range(B)])
    got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(ys).to(DEV), 100, minmax_ratio=4).cpu().numpy()
    for i in (0, 1, 73, B - 1):
        _eq(got[i], O.minmaxlttb(x, ys[i].astype(np.float64), 100, 4), f"fused row {i}")


def case_minmax_m4():
    n = 123_457
    x = np.arange(n, dtype=np.int64)
    y = _rw(n, 9, np.float64)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    _eq(mm.minmax(xd, yd, 500), O.minmax(y, 500), "minmax")
    _eq(mm.m4(xd, yd, 500), O.m4(y, 500), "m4")
    _eq(mm.minmaxlttb(xd, yd, 500, minmax_ratio=1), O.minmaxlttb(x, y, 500, 1), "minmax_with_endpoints")


def case_validate():
    n = 50_000
    x = np.arange(n, dtype=np.float64)
    y = _rw(n, 12, np.float64)
    ts = mm.TimeSeries(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV))
    _eq(mm.minmaxlttb(ts, 300, 4), O.minmaxlttb(x, y, 300, 4), "validate ok")
    bad = y.copy()
    bad[777] = np.nan
    try:
        mm.TimeSeries(torch.from_numpy(x).to(DEV), torch.from_numpy(bad).to(DEV))
    except mm.errors.NonFiniteValue:
        pass
    else:
        raise AssertionError("NaN not rejected")


def case_shards():
    n, n_out, r = 1_000_003, 1000, 4
    rng = np.random.Generator(np.random.PCG64(13))
    x = np.cumsum(rng.exponential(1.0, n))
    y = _rw(n, 13)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    plan = S.bucket_ranges(n, n_out, r, 4)
    cap = plan[0].cap
    bufs = []
    for sh in plan:
        buf = torch.zeros((3 * cap + 1,), dtype=torch.int64, device=DEV)
        S.shard_preselect(xd[sh.lo:sh.hi], yd[sh.lo:sh.hi], n, n_out, r, sh, packed=buf)
        bufs.append(buf)
    got = S.lttb_merged(*S.merge_packed(torch.cat(bufs), 4, cap), n_out, r)
    _eq(got, O.minmaxlttb(x, y.astype(np.float64), n_out, r), "shards")


def case_p2p():
    G, n, n_out, r = 4, 400_000, 1000, 4
    rng = np.random.Generator(np.random.PCG64(14))
    x = np.cumsum(rng.exponential(1.0, n))
    y = _rw(n, 14)
    xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
    plan = S.bucket_ranges(n, n_out, r, G)
    cap, W = plan[0].cap, 3 * plan[0].cap + 1
    sets = [S.shard_preselect(xd[sh.lo:sh.hi], yd[sh.lo:sh.hi], n, n_out, r, sh) for sh in plan]
    bufs = [torch.zeros((2 * G * W,), dtype=torch.int64, device=DEV) for _ in range(G)]
    pads = [torch.zeros(2 * G, dtype=torch.int32, device=DEV) for _ in range(G)]
    pb = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=DEV)
    pp = torch.tensor([p.data_ptr() for p in pads], dtype=torch.int64, device=DEV)
    L = mm._native.lib()
    st = mm._native.stream_ptr(DEV)
    want = O.minmaxlttb(x, y.astype(np.float64), n_out, r)
    for epoch in range(1, 4):
        for g in range(G):
            idx, xs, ys, cnt = sets[g]
            mm._native.check(L.mmlttb_p2p_publish(idx.data_ptr(), xs.data_ptr(), ys.data_ptr(), cnt.data_ptr(), cap,
                                                  pb.data_ptr(), pp.data_ptr(), pads[g].data_ptr(), G, g, epoch, st),
                             "p2p_publish")
        for g in range(G):
            oi = torch.zeros(G * cap, dtype=torch.int64, device=DEV)
            ox = torch.zeros(G * cap, dtype=torch.float64, device=DEV)
            oy = torch.zeros(G * cap, dtype=torch.float64, device=DEV)
            om = torch.zeros(1, dtype=torch.int64, device=DEV)
            mm._native.check(L.mmlttb_p2p_merge(bufs[g].data_ptr(), pads[g].data_ptr(), pp.data_ptr(), G, g, cap,
                                                epoch, oi.data_ptr(), ox.data_ptr(), oy.data_ptr(), om.data_ptr(), st),
                             "p2p_merge")
            _eq(S.lttb_merged(oi, ox, oy, om, n_out, r), want, f"p2p epoch {epoch} rank {g}")


def _k3s(seed, n=1_600_000, n_out=1400):
    # >= 8 x SMs large buckets: the one-launch K3s path (grid barrier, neighbour flags,
    # aggregate maps, deviation walks)
    x = np.arange(n, dtype=np.int64)
    y = _rw(n, seed, np.float64)
    got = mm.lttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out)
    _eq(got, O.lttb(x, y, n_out), "k3s")


def case_k3s():
    _k3s(16)


def case_k3s_miss():
    os.environ["MMLTTB_K3C_CAND_CAP"] = "1"  # every candidate set misses: 4a/4b walks + repair walk
    _k3s(17)


def case_k23():
    # one series, cooperative K2+K3a (grid barriers, per-CTA status slots), C1 and C3 shapes
    for n, n_out, r, dt in ((1_000_000, 1000, 4, np.float64), (4_000_000, 2000, 4, np.float32),
                            (4_000_000, 2000, 32, np.float32)):
        x = np.arange(n, dtype=np.int64)
        y = _rw(n, 18, dt)
        got = mm.minmaxlttb(torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV), n_out, minmax_ratio=r)
        _eq(got, O.minmaxlttb(x, y.astype(np.float64), n_out, r), f"k23 n={n} r={r}")


def case_raster():
    n = 5_000
    x = np.arange(n, dtype=np.float64)
    y = _rw(n, 15, np.float64)
    ts = mm.TimeSeries(x, y)
    sel = O.minmaxlttb(x, y, 200, 4)
    cv = mm.fit_canvas(ts, 120, 60)
    full = mm.rasterize(ts, cv, device=DEV)
    part = mm.rasterize(ts, cv, sel, device=DEV)
    assert full is not None and part is not None


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        torch.cuda.synchronize()
        print(f"case {nm}: ok", flush=True)
