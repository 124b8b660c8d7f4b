"""Multi-GPU MinMaxLTTB: one process per GPU over ``torch.distributed``.

Two decompositions; the reference has no multi-device code,
its only parallelism is numba ``prange`` over disjoint buckets
(``_kernels.py:71-78``), and both paths below keep its output byte-identical.

* **Batch sharding** (BASELINE.json C4): independent series, rank r owns rows
  ``batch_range(B, r, G)``; no collective on the data path (an optional
  ``all_gather`` assembles the [B, n_out] result).
* **Bucket-range sharding of one series** (C5): rank r owns MinMax
  sub-buckets ``[b0, b1)`` of ``partition(1, N-1, k)`` and exactly the y/x
  elements they cover (rank 0 also element 0, rank G-1 also element N-1), so
  no sub-bucket straddles ranks.  Each rank runs K1 + K2 on its shard
  (``mmlttb_shard_preselect``), the small preselected sets (global index, x,
  y as f64; <= 2*(b1-b0)+2 entries) are packed into one int64 buffer and
  exchanged with ONE ``all_gather`` (NCCL over NVLink), every rank merges
  them in rank order on the device (``mmlttb_merge_packed``, straight from
  the gathered messages) and runs the LTTB stage on the merged set
  (``mmlttb_lttb_preselected``).  The exchanged
  bytes are O(k), independent of N.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _native as N
from .downsamplers import Batch, _check_n_out, _check_preselect, _minmax_like, _minmaxlttb_batch
from .errors import OddNOut


# ------------------------------------------------------------ batch path ----
def batch_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) of a B-series batch owned by `rank` (balanced, contiguous)."""
    return (B * rank) // world, (B * (rank + 1)) // world


def minmaxlttb_batch_sharded(x, y_local, n_out: int, r_ps: int = 4, *, B: int | None = None,
                             gather: bool = False, group=None):
    """MinMaxLTTB over this rank's rows of a batch (no collective on the data path).

    ``y_local``: this rank's [b, N] rows (see :func:`batch_range`).  The
    reference's checks run first, in its order (downsamplers.py:182-209 with
    :37-41, :146-153; r_ps == 1 diverts to MinMax with endpoints, :164-179).
    With ``gather=True`` the [B, n_out] result is all-gathered to every rank;
    ``B`` (the global series count) is then required, since rows may be split
    unevenly.  r_ps == 1 rows can be shorter than n_out: they come back (and
    are gathered) as a list of per-series index tensors.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if gather and world > 1 and B is None:
        raise ValueError("gather=True needs the global series count B")
    b = _prepared(x, y_local)
    if r_ps == 1:
        _check_n_out(b.n, n_out)
        if n_out % 2:
            raise OddNOut(f"minmax needs an even n_out, got {n_out}")
        rows = _minmax_like(b, n_out, "minmax", force=True)
        rows = rows if isinstance(rows, list) else [rows]
        if not gather or world == 1:
            return rows
        got = [None] * world
        dist.all_gather_object(got, [r.cpu() for r in rows], group=group)
        dev = b.device
        return [r.to(dev) for part in got for r in part]
    _check_preselect(b.n, n_out, r_ps)
    out = _minmaxlttb_batch(b, n_out, r_ps)
    if not gather or world == 1:
        return out
    rank = dist.get_rank(group)
    lo, hi = batch_range(B, rank, world)
    if out.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} must hold rows [{lo}, {hi}) of the {B}-series batch, got {out.shape[0]}")
    per = -(-B // world)
    buf = torch.full((per, n_out), -1, dtype=torch.int64, device=out.device)
    buf[: out.shape[0]] = out
    allb = all_gather_flat(buf.reshape(-1), world, group).view(world * per, n_out)
    rows = [allb[r * per: r * per + (batch_range(B, r, world)[1] - batch_range(B, r, world)[0])] for r in range(world)]
    return torch.cat(rows, 0)


def all_gather_flat(buf: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[world * buf.numel()] concatenation of every rank's `buf`, on buf's device.

    NCCL gathers in place over NVLink; any other backend (gloo: the CPU test
    groups, or several ranks sharing one GPU) is staged through host memory."""
    backend = dist.get_backend(group)
    if backend == "nccl":
        allbuf = torch.empty(world * buf.numel(), dtype=buf.dtype, device=buf.device)
        dist.all_gather_into_tensor(allbuf, buf, group=group)
        return allbuf
    host = buf.detach().cpu()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    return torch.cat(parts).to(buf.device)


def _prepared(x, y):
    b = Batch(x, y)
    b.squeeze = False
    return b


# ----------------------------------------------------- single-series path ---
@dataclass(frozen=True)
class Shard:
    """What rank `rank` of `world` owns of one N-point series."""

    rank: int
    world: int
    b0: int   # first MinMax sub-bucket (of k)
    b1: int   # one past the last
    lo: int   # first element index held by the rank
    hi: int   # one past the last element index
    k: int
    cap: int  # fixed per-rank capacity of the exchanged preselected set

    @property
    def emit_first(self) -> bool:
        return self.rank == 0

    @property
    def emit_last(self) -> bool:
        return self.rank == self.world - 1


def bucket_ranges(n: int, n_out: int, r_ps: int, world: int) -> list[Shard]:
    """Bucket-range sharding plan of partition(1, N-1, k) over `world` ranks.

    Rank r owns sub-buckets [floor(r*k/G), floor((r+1)*k/G)) and the elements
    they cover -- index arithmetic only (core.py:173 closed form), x is never
    consulted, so every rank's sub-buckets are exactly the reference's.
    """
    k = _check_preselect(n, n_out, r_ps)
    L = n - 2

    def bound(b):
        return 1 + (b * L) // k

    per = max((k * (r + 1)) // world - (k * r) // world for r in range(world))
    cap = 2 * per + 2
    out = []
    for r in range(world):
        b0, b1 = (k * r) // world, (k * (r + 1)) // world
        lo = 0 if r == 0 else bound(b0)
        hi = n if r == world - 1 else bound(b1)
        out.append(Shard(r, world, b0, b1, lo, hi, k, cap))
    return out


def pack(idx: torch.Tensor, xs: torch.Tensor, ys: torch.Tensor, count: torch.Tensor, cap: int) -> torch.Tensor:
    """One int64 message: [idx(cap) | x bits(cap) | y bits(cap) | count]."""
    buf = torch.empty(3 * cap + 1, dtype=torch.int64, device=idx.device)
    buf[:cap] = idx[:cap]
    buf[cap:2 * cap] = xs[:cap].view(torch.int64)
    buf[2 * cap:3 * cap] = ys[:cap].view(torch.int64)
    buf[3 * cap:] = count.reshape(1)
    return buf


def unpack(allbuf: torch.Tensor, world: int, cap: int):
    """Inverse of :func:`pack` over the all-gathered [world*(3cap+1)] buffer."""
    m = allbuf.view(world, 3 * cap + 1)
    idx = m[:, :cap].contiguous()
    xs = m[:, cap:2 * cap].contiguous().view(torch.float64)
    ys = m[:, 2 * cap:3 * cap].contiguous().view(torch.float64)
    counts = m[:, 3 * cap].contiguous()
    return idx, xs, ys, counts


def exchange(buf: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """The one collective of the path: all_gather of the packed shard sets."""
    return all_gather_flat(buf, world, group)


class PeerExchange:
    """Device-initiated replacement for :func:`exchange` + :func:`unpack` +
    ``mmlttb_merge_shards``: every rank stores its preselected set straight
    into each peer's symmetric buffer over NVLink (``mmlttb_p2p_publish``)
    and the peers concatenate the rows in rank order as soon as their epoch
    flags arrive (``mmlttb_p2p_merge``) -- no NCCL launch, no host sync, and
    the merged set lands directly in the LTTB stage's input.  Double-buffered
    by epoch parity with per-peer acks, so back-to-back calls never overwrite
    a row a peer has not consumed.  Opt-in (``exchange="p2p"``); built on
    ``torch.distributed._symmetric_memory`` for allocation + rendezvous only.
    """

    def __init__(self, cap: int, device, group=None):
        from torch.distributed import _symmetric_memory as symm
        self.cap, self.device = cap, torch.device(device)
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        W = 3 * cap + 1
        self.buf = symm.empty(2 * self.world * W, dtype=torch.int64, device=self.device)
        self.handle = symm.rendezvous(self.buf, dist.group.WORLD if group is None else group)
        # the flags live at the END of the signal pad, clear of the channel
        # slots torch's own barrier()/put_signal use at its start
        words = self.handle.signal_pad_size // 4
        if words < 2 * self.world + 64 * self.world:
            raise RuntimeError("symmetric-memory signal pad too small for the exchange flags")
        off = words - 2 * self.world
        pads = [self.handle.get_signal_pad(r, (2 * self.world,), dtype=torch.int32, storage_offset=off)
                for r in range(self.world)]
        bufs = [self.handle.get_remote_tensor(r, (2 * self.world * W,), torch.int64) for r in range(self.world)]
        self.own_pad = pads[self.rank]
        self.own_pad.zero_()
        self.peer_bufs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device=self.device)
        self.peer_pads = torch.tensor([p.data_ptr() for p in pads], dtype=torch.int64, device=self.device)
        self.epoch = 0
        self.handle.barrier()

    def __call__(self, idx, xs, ys, cnt):
        """Publish this rank's set, return the merged (idx, x, y, m) of all ranks."""
        self.epoch += 1
        G, cap = self.world, self.cap
        tot = G * cap
        oi = torch.empty(tot, dtype=torch.int64, device=self.device)
        ox = torch.empty(tot, dtype=torch.float64, device=self.device)
        oy = torch.empty(tot, dtype=torch.float64, device=self.device)
        om = torch.empty(1, dtype=torch.int64, device=self.device)
        L = N.lib()
        with torch.cuda.device(self.device):
            st = N.stream_ptr(self.device)
            N.check(L.mmlttb_p2p_publish(idx.data_ptr(), xs.data_ptr(), ys.data_ptr(), cnt.data_ptr(), cap,
                                         self.peer_bufs.data_ptr(), self.peer_pads.data_ptr(),
                                         self.own_pad.data_ptr(), G, self.rank, self.epoch, st), "p2p_publish")
            N.check(L.mmlttb_p2p_merge(self.buf.data_ptr(), self.own_pad.data_ptr(), self.peer_pads.data_ptr(), G,
                                       self.rank, cap, self.epoch, oi.data_ptr(), ox.data_ptr(), oy.data_ptr(),
                                       om.data_ptr(), st), "p2p_merge")
        return oi, ox, oy, om


_PEER_EXCHANGES: dict = {}


def _peer_exchange(cap: int, device, group) -> PeerExchange:
    key = (cap, str(device), id(group))
    ex = _PEER_EXCHANGES.get(key)
    if ex is None:
        ex = _PEER_EXCHANGES[key] = PeerExchange(cap, device, group)
    return ex


def shard_preselect(x_shard: torch.Tensor, y_shard: torch.Tensor, n: int, n_out: int, r_ps: int, shard: Shard,
                    packed: torch.Tensor | None = None):
    """K1 + K2 on this rank's elements -> (idx, x f64, y f64, count) on device.

    With ``packed`` (int64 [3*cap+1]) the results are written straight into
    the exchange message layout of :func:`pack` (views into ``packed``)."""
    dev = y_shard.device
    cap = shard.cap
    if packed is not None:
        idx = packed[:cap]
        xs = packed[cap:2 * cap].view(torch.float64)
        ys = packed[2 * cap:3 * cap].view(torch.float64)
        cnt = packed[3 * cap:]
    else:
        idx = torch.empty(cap, dtype=torch.int64, device=dev)
        xs = torch.empty(cap, dtype=torch.float64, device=dev)
        ys = torch.empty(cap, dtype=torch.float64, device=dev)
        cnt = torch.empty(1, dtype=torch.int64, device=dev)
    L = N.lib()
    with torch.cuda.device(dev):
        wsb = L.mmlttb_shard_workspace_bytes(n, n_out, r_ps, shard.b0, shard.b1)
        ws = N.workspace(wsb, dev, n)
        N.check(L.mmlttb_shard_preselect(x_shard.data_ptr(), N.DTYPE_CODE[x_shard.dtype], y_shard.data_ptr(),
                                         N.DTYPE_CODE[y_shard.dtype], shard.lo, n, n_out, r_ps, shard.b0, shard.b1,
                                         int(shard.emit_first), int(shard.emit_last), idx.data_ptr(), xs.data_ptr(),
                                         ys.data_ptr(), cnt.data_ptr(), ws.data_ptr(), wsb, N.stream_ptr(dev)),
                "shard_preselect", n)
    return idx, xs, ys, cnt


def merge_packed(allbuf: torch.Tensor, world: int, cap: int):
    """Device rank-order merge of the gathered packed messages (no unpack copies)."""
    dev = allbuf.device
    tot = world * cap
    oi = torch.empty(tot, dtype=torch.int64, device=dev)
    ox = torch.empty(tot, dtype=torch.float64, device=dev)
    oy = torch.empty(tot, dtype=torch.float64, device=dev)
    om = torch.empty(1, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        N.check(N.lib().mmlttb_merge_packed(allbuf.data_ptr(), world, cap, oi.data_ptr(), ox.data_ptr(),
                                            oy.data_ptr(), om.data_ptr(), N.stream_ptr(dev)), "merge_packed")
    return oi, ox, oy, om


def lttb_merged(oi, ox, oy, om, n_out: int, r_ps: int) -> torch.Tensor:
    """The LTTB stage over an already merged preselected set (m on device)."""
    dev = oi.device
    out = torch.empty(n_out, dtype=torch.int64, device=dev)
    L = N.lib()
    with torch.cuda.device(dev):
        wsb = L.mmlttb_lttb_preselected_workspace_bytes(1, n_out, r_ps)
        ws = N.workspace(wsb, dev)
        N.check(L.mmlttb_lttb_preselected(oi.data_ptr(), ox.data_ptr(), oy.data_ptr(), om.data_ptr(), 1, oi.numel(),
                                          n_out, r_ps, out.data_ptr(), ws.data_ptr(), wsb, N.stream_ptr(dev)),
                "lttb_preselected")
    return out


def merge_and_lttb(idx, xs, ys, counts, n_out: int, r_ps: int) -> torch.Tensor:
    """Device merge of the G shard sets in rank order, then the LTTB stage."""
    dev = idx.device
    G, cap = idx.shape
    tot = G * cap
    oi = torch.empty(tot, dtype=torch.int64, device=dev)
    ox = torch.empty(tot, dtype=torch.float64, device=dev)
    oy = torch.empty(tot, dtype=torch.float64, device=dev)
    om = torch.empty(1, dtype=torch.int64, device=dev)
    out = torch.empty(n_out, dtype=torch.int64, device=dev)
    L = N.lib()
    with torch.cuda.device(dev):
        st = N.stream_ptr(dev)
        N.check(L.mmlttb_merge_shards(idx.data_ptr(), xs.data_ptr(), ys.data_ptr(), counts.data_ptr(), G, cap,
                                      oi.data_ptr(), ox.data_ptr(), oy.data_ptr(), om.data_ptr(), st), "merge_shards")
        wsb = L.mmlttb_lttb_preselected_workspace_bytes(1, n_out, r_ps)
        ws = N.workspace(wsb, dev)
        N.check(L.mmlttb_lttb_preselected(oi.data_ptr(), ox.data_ptr(), oy.data_ptr(), om.data_ptr(), 1, tot, n_out,
                                          r_ps, out.data_ptr(), ws.data_ptr(), wsb, st), "lttb_preselected")
    return out


def minmaxlttb_series_sharded(x_shard: torch.Tensor, y_shard: torch.Tensor, n: int, n_out: int, r_ps: int = 4,
                              group=None, exchange_mode: str = "nccl") -> torch.Tensor:
    """minmaxlttb of ONE series split by bucket ranges across the ranks.

    ``x_shard``/``y_shard`` hold elements ``[shard.lo, shard.hi)`` of the
    series for this rank (see :func:`bucket_ranges`).  Returns the n_out
    indices (identical to the single-device result) on every rank.
    ``exchange_mode``: "nccl" (one all_gather, default) or "p2p" (device-
    initiated stores into the peers' symmetric buffers, :class:`PeerExchange`).
    """
    if exchange_mode not in ("nccl", "p2p"):
        raise ValueError(f"exchange_mode must be 'nccl' or 'p2p', got {exchange_mode!r}")
    _check_n_out(n, n_out)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    shard = bucket_ranges(n, n_out, r_ps, world)[rank]
    if y_shard.shape[0] != shard.hi - shard.lo or x_shard.shape[0] != y_shard.shape[0]:
        raise ValueError(f"rank {rank} must hold elements [{shard.lo}, {shard.hi}) of the series")
    if exchange_mode == "p2p":
        if not dist.is_initialized():
            raise RuntimeError("exchange_mode='p2p' needs an initialised process group")
        idx, xs, ys, cnt = shard_preselect(x_shard, y_shard, n, n_out, r_ps, shard)
        return lttb_merged(*_peer_exchange(shard.cap, y_shard.device, group)(idx, xs, ys, cnt), n_out, r_ps)
    # K1 + K2 write the exchange message in place (layout of pack()), one
    # all_gather, then the merge reads the gathered messages directly
    buf = torch.empty(3 * shard.cap + 1, dtype=torch.int64, device=y_shard.device)
    shard_preselect(x_shard, y_shard, n, n_out, r_ps, shard, packed=buf)
    allbuf = exchange(buf, world, group) if world > 1 else buf
    return lttb_merged(*merge_packed(allbuf, world, shard.cap), n_out, r_ps)
