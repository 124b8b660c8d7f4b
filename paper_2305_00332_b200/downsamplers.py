"""The selection algorithms on the B200 (reference ``tsdown/downsamplers.py``).

Same names, signatures, checks (in the reference's order) and outputs as
``/root/reference/pkg/src/tsdown/downsamplers.py``; the work is done by the
sm_100a kernels behind ``libmmlttb.so``:

* ``minmaxlttb``        -> ``mmlttb_minmaxlttb``   (K1 extrema -> K2 compact -> K3 LTTB)
* ``minmax_preselect``  -> ``mmlttb_minmax_preselect``
* ``lttb``              -> ``mmlttb_lttb``
* ``minmax`` / ``m4``   -> ``mmlttb_minmax`` / ``mmlttb_m4``
* ``every_nth``         -> ``mmlttb_every_nth``

Every function also accepts the flat form ``(x, y, n_out, ...)`` from the
north star (``minmaxlttb(x, y, n_out, minmax_ratio=4)``); ``y`` may then be
2-D ``[B, N]`` (one series per row, ``x`` shared ``[N]`` or per row) and the
result is ``[B, n_out]``.  Results follow the input's home: numpy in, numpy
out; CUDA tensors in, CUDA int64 tensor out (no host sync for fixed-size
outputs).  ``parallel``/``threads`` are accepted for parity; the device path
is always bucket-parallel and byte-identical to the sequential reference.
"""
from __future__ import annotations

import collections
import contextlib
import ctypes
import threading

import numpy as np
import torch

from . import _native as N
from .core import Algorithm, DownsampleConfig, TimeSeries, validate
from .errors import (
    BadPreselectionRatio,
    NonFiniteValue,
    NonMonotonicX,
    NotParallelizable,
    NOutNotDivisibleBy4,
    NOutOfRange,
    OddNOut,
    RatioTooLargeForSeries,
)

__all__ = [
    "every_nth", "minmax", "m4", "lttb", "minmax_preselect", "minmaxlttb", "run_parallel", "downsample",
    "Batch", "check_deferred",
]


# ----------------------------------------------- deferred status words ------
# Device-input calls (validate=None) do not sync: their status word (bit 0 =
# non-finite y) is stored by the device into a pinned host slot armed before
# the call (mmlttb_status_arm) and checked by later calls or check_deferred().
_DEFERRED: collections.deque = collections.deque()
_DEFERRED_LOCK = threading.Lock()
_DEFERRED_MAX = 512  # the C ring holds 1024 outstanding tickets


_RING = None  # numpy view of the library's pinned status ring (mmlttb_status_ring)
_RING_SLOTS = 1024


def _ring():
    global _RING
    if _RING is None:
        p = N.lib().mmlttb_status_ring()
        if not p:
            N.check(N.MM_ECUDA, "status_ring")
        _RING = np.ctypeslib.as_array((ctypes.c_uint64 * _RING_SLOTS).from_address(p))
    return _RING


def _poll_landed(block: bool) -> None:
    """Retire the deferred tickets whose slots the device has written, in order."""
    ring = _ring()
    with _DEFERRED_LOCK:
        while _DEFERRED:
            t, what = _DEFERRED[0]
            v = int(ring[t % _RING_SLOTS])
            if (v >> 3) != t + 1:
                if not block:
                    return
                rc = N.lib().mmlttb_status_poll(t, 1)  # synchronises the device
                if rc < 0:
                    _DEFERRED.popleft()
                    N.check(rc, "status_poll")
                v = rc
            _DEFERRED.popleft()
            if v & 1:
                raise NonFiniteValue(f"series contains NaN or infinite values (in an earlier {what} call on device "
                                     "inputs; pass validate=True to check before returning)")


def check_deferred(block: bool = True) -> None:
    """Raise ``NonFiniteValue`` if an earlier device-input call saw NaN/inf in ``y``.

    The reference rejects non-finite values when the series is built
    (core.py:80-94).  Calls on CUDA tensors with ``validate=None`` do not
    synchronise for that check; the device writes their status word into a
    pinned host slot, every later call polls the slots already written
    (non-blocking) and raises for the oldest failing call.
    ``check_deferred()`` synchronises the device for the outstanding slots
    (``block=True``) and raises the same way.
    """
    if _DEFERRED:
        _poll_landed(block)


# --------------------------------------------------------------- inputs ----
class Batch:
    """B series of N points for one CUDA device (the flat / batched form).

    ``y``: [B, N] (or [N]) float32/float64; ``x``: [N] shared or [B, N],
    int64/int32/float32/float64.  A pinned host ``x`` is read in place by the
    gather (zero-copy over PCIe: only the <= 2 + (n_out-2)*r_ps preselected
    x values are ever touched), so ``minmaxlttb`` moves just ``y`` to HBM.
    Shapes are known at construction; device transfers happen in
    ``ready()``, after the reference's O(1) checks have passed.
    """

    def __init__(self, x, y, device=None, validate=None):
        self._x_in, self._y_in, self._dev_in = x, y, device
        self.host = not (isinstance(y, torch.Tensor) and y.is_cuda)
        # None: host inputs get the free non-finite-y check (raised after the
        # call, which syncs anyway); True: full TimeSeries invariants first
        self.validate = validate
        self.numpy = not isinstance(y, torch.Tensor)
        shape = tuple(y.shape) if hasattr(y, "shape") else np.shape(y)
        if len(shape) not in (1, 2):
            raise ValueError("y must be [N] or [B, N]")
        self.squeeze = len(shape) == 1
        self.B, self.n = (1, int(shape[0])) if self.squeeze else (int(shape[0]), int(shape[1]))
        self._ready = False

    def ready(self):
        if self._ready:
            return self
        if _DEFERRED:
            _poll_landed(False)
        y, x = self._y_in, self._x_in
        dev = N.require_cuda(y.device if not self.host else self._dev_in)
        yt = torch.as_tensor(y) if not isinstance(y, torch.Tensor) else y
        if yt.dtype not in (torch.float32, torch.float64):
            yt = yt.to(torch.float64)
        if yt.dim() == 1:
            yt = yt.unsqueeze(0)
        self.y = yt.to(dev, non_blocking=True).contiguous() if yt.device != dev else yt.contiguous()
        self.device = dev
        self.x = None
        self.x_ld = 0
        if x is not None:
            xt = torch.as_tensor(x) if not isinstance(x, torch.Tensor) else x
            if xt.dtype not in (torch.float32, torch.float64, torch.int64, torch.int32):
                xt = xt.to(torch.float64)
            if xt.dim() == 2 and xt.shape[0] == 1:
                xt = xt[0]
            if xt.shape[-1] != self.n or xt.dim() > 2 or (xt.dim() == 2 and xt.shape[0] != self.B):
                raise ValueError("x must be [N] or [B, N] matching y")
            xt = xt.contiguous()
            if not xt.is_cuda and not xt.is_pinned():
                xt = xt.to(dev, non_blocking=True)
            self.x = xt
            self.x_ld = self.n if xt.dim() == 2 else 0
        self._ready = True
        if self.validate:
            self._full_validate()
        return self

    def _full_validate(self):
        """TimeSeries invariants (core.py:80-94) for every row: one batched launch, one sync.

        The rows are B series built in order, so the first failing row decides,
        and within it non-finite values are reported before a decreasing x."""
        if self.x is None:
            return
        xs = self.x if self.x.is_cuda else self.x.to(self.device)
        flags = torch.empty(self.B, dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            N.check(N.lib().mmlttb_validate_batch(xs.data_ptr(), N.DTYPE_CODE[xs.dtype], self.n if xs.dim() == 2 else 0,
                                                  self.y.data_ptr(), N.DTYPE_CODE[self.y.dtype], self.n, self.B, self.n,
                                                  flags.data_ptr(), N.stream_ptr(self.device)), "validate", self.n)
        fl = flags.cpu().numpy()
        bad = np.flatnonzero(fl)
        if bad.shape[0] == 0:
            return
        f = int(fl[bad[0]])
        if f & 1:
            raise NonFiniteValue("series contains NaN or infinite values")
        raise NonMonotonicX("xs must be sorted in non-decreasing order")

    def arm(self) -> int | None:
        """Device inputs with validate=None: arm a deferred status slot for the
        next library call (mmlttb_status_arm); None when the check is synchronous
        (host inputs, validate=True) or skipped (validate=False).  A call under
        graph capture delivers no status (the library checks)."""
        if self.validate is not None or self.host:
            return None
        t = N.lib().mmlttb_status_arm()
        if t < 0:
            N.check(t, "status_arm")
        return t

    def post_check(self, ws: torch.Tensor, what: str, ticket: int | None) -> None:
        """Raise the reference's NonFiniteValue from the kernels' status word.

        Host inputs (and validate=True) read it now; device inputs with
        validate=None get it back through the armed slot (``check_deferred``),
        so the call stays free of host syncs; validate=False skips it."""
        if ticket is not None:
            _DEFERRED.append((ticket, what))  # (deque.append is atomic)
            if len(_DEFERRED) > _DEFERRED_MAX:
                check_deferred(block=True)
            return
        if self.validate is False or not (self.host or self.validate):
            return
        if int(ws[:4].view(torch.int32)[0].item()) & 1:
            raise NonFiniteValue("series contains NaN or infinite values")

    def ret(self, t: torch.Tensor):
        if self.squeeze:
            t = t[0]
        return t.cpu().numpy() if self.numpy else (t.cpu() if self.host else t)


class _Series(Batch):
    """Adapter: a TimeSeries seen as a 1-series Batch (already validated)."""

    def __init__(self, series: TimeSeries, device=None):
        self._series, self._dev_in = series, device
        self.validate = False
        self.host = self.numpy = series.is_host
        self.squeeze = True
        self.B, self.n = 1, len(series)
        self._ready = False

    def ready(self):
        if not self._ready:
            x, y = self._series.device_arrays(self._dev_in)
            self.y, self.x, self.x_ld, self.device = y.unsqueeze(0), x, 0, y.device
            self._ready = True
        return self


def _input(series, y=None, device=None):
    return _Series(series, device) if isinstance(series, TimeSeries) else Batch(series, y, device)


def _codes(b):
    return (N.DTYPE_CODE[b.x.dtype] if b.x is not None else 0), N.DTYPE_CODE[b.y.dtype]


def _ctx(b):
    # switching devices costs two driver calls; skip it when already there
    if torch.cuda.current_device() == b.device.index:
        return contextlib.nullcontext()
    return torch.cuda.device(b.device)


def _is_flat(first) -> bool:
    return not isinstance(first, TimeSeries)


def _int_arg(v, what: str) -> int:
    """Strict integer argument: a bool or an array in an integer slot means the
    reference form and the flat form were mixed up -- raise, never rebind."""
    if isinstance(v, (bool, np.bool_)) or not isinstance(v, (int, np.integer)):
        raise TypeError(f"{what} must be an integer, got {type(v).__name__}")
    return int(v)


def _no_extra(fn: str, args) -> None:
    if args:
        raise TypeError(f"{fn}() got {len(args)} unexpected positional argument(s)")


# ------------------------------------------------------------- checks -------
def _check_n_out(n: int, n_out: int) -> int:
    if not 3 <= n_out <= n:  # downsamplers.py:37-41
        raise NOutOfRange(f"n_out must be in [3, {n}], got {n_out}")
    return n


def _check_preselect(n: int, n_out: int, r_ps: int) -> int:
    _check_n_out(n, n_out)
    if r_ps < 2 or r_ps % 2:  # downsamplers.py:147-148
        raise BadPreselectionRatio(f"preselection needs an even r_ps >= 2, got {r_ps}")
    sub_buckets = (n_out - 2) * (r_ps // 2)
    if sub_buckets > n - 2:  # :149-153
        raise RatioTooLargeForSeries(f"{sub_buckets} sub-buckets exceed the {n - 2} interior samples")
    return sub_buckets


def _counted(b, out, cnt):
    """Trim variable-length rows (minmax/m4/preselect) -- one host sync."""
    counts = cnt.cpu().tolist()
    if b.B == 1:
        return b.ret(out[:, : counts[0]])
    rows = [out[i, : counts[i]] for i in range(b.B)]
    if b.numpy:
        return [r.cpu().numpy() for r in rows]
    return rows


# ------------------------------------------------------------ algorithms ----
def every_nth(series, n_out, *args):
    """Select floor(i * N / n_out), i in [0, n_out) (downsamplers.py:44-47)."""
    if _is_flat(series):  # every_nth(x, y, n_out)
        if len(args) != 1:
            raise TypeError("flat form: every_nth(x, y, n_out)")
        b, n_out = Batch(series, n_out, None), _int_arg(args[0], "n_out")
    else:
        _no_extra("every_nth", args)
        b, n_out = _Series(series), _int_arg(n_out, "n_out")
    _check_n_out(b.n, n_out)
    b.ready()
    out = torch.empty((1, n_out), dtype=torch.int64, device=b.device)
    with _ctx(b):
        N.check(N.lib().mmlttb_every_nth(b.n, n_out, out.data_ptr(), N.stream_ptr(b.device)), "every_nth")
    if b.B > 1:
        out = out.expand(b.B, n_out).contiguous()
    return b.ret(out)


def _minmax_like(b, n_out, op: str, force: bool = False):
    b.ready()
    fn = N.lib().mmlttb_m4 if op == "m4" else N.lib().mmlttb_minmax
    code = N.OP_M4 if op == "m4" else N.OP_MINMAX
    xdt, ydt = _codes(b)
    out = torch.empty((b.B, n_out), dtype=torch.int64, device=b.device)
    cnt = torch.empty(b.B, dtype=torch.int64, device=b.device)
    with _ctx(b):
        st = N.stream_ptr(b.device)
        ticket = b.arm()
        if force:  # r_ps == 1 through the fused entry (downsamplers.py:164-179)
            wsb = N.lib().mmlttb_workspace_bytes(N.OP_MINMAXLTTB, b.B, b.n, n_out, 1, ydt)
            ws = N.workspace(wsb, b.device, b.n)
            N.check(N.lib().mmlttb_minmaxlttb(N.ptr(b.x), xdt, b.x_ld, b.y.data_ptr(), ydt, b.n, b.B, b.n,
                                              n_out, 1, out.data_ptr(), cnt.data_ptr(), ws.data_ptr(), wsb, st),
                    "minmaxlttb(r_ps=1)", b.n)
        else:
            wsb = N.lib().mmlttb_workspace_bytes(code, b.B, b.n, n_out, 0, ydt)
            ws = N.workspace(wsb, b.device, b.n)
            N.check(fn(b.y.data_ptr(), ydt, b.n, b.B, b.n, n_out, out.data_ptr(), cnt.data_ptr(), ws.data_ptr(),
                       wsb, st), op, b.n)
    b.post_check(ws, "minmaxlttb" if force else op, ticket)
    return _counted(b, out, cnt)


def minmax(series, n_out, parallel=False, *args, **kw):
    """Vertical extrema per bucket (downsamplers.py:72-92).

    Flat form: ``minmax(x, y, n_out)``.
    """
    if _is_flat(series):
        _no_extra("minmax", args)
        b, n_out = Batch(series, n_out, kw.get("device"), kw.get("validate")), _int_arg(parallel, "n_out")
    else:
        _no_extra("minmax", args)
        b, n_out = _Series(series), _int_arg(n_out, "n_out")
    _check_n_out(b.n, n_out)
    if n_out % 2:
        raise OddNOut(f"minmax needs an even n_out, got {n_out}")
    return _minmax_like(b, n_out, "minmax")


def m4(series, n_out, parallel=False, *args, **kw):
    """First, min, max and last sample per bucket (downsamplers.py:95-112).

    Flat form: ``m4(x, y, n_out)``.
    """
    _no_extra("m4", args)
    if _is_flat(series):
        b, n_out = Batch(series, n_out, kw.get("device"), kw.get("validate")), _int_arg(parallel, "n_out")
    else:
        b, n_out = _Series(series), _int_arg(n_out, "n_out")
    _check_n_out(b.n, n_out)
    if n_out % 4:
        raise NOutNotDivisibleBy4(f"m4 needs n_out divisible by 4, got {n_out}")
    return _minmax_like(b, n_out, "m4")


def lttb(series, n_out, *args, **kw):
    """Largest-Triangle-Three-Buckets (downsamplers.py:115-132): exactly n_out indices.

    Flat form: ``lttb(x, y, n_out)``.
    """
    if _is_flat(series):
        if len(args) != 1:
            raise TypeError("flat form: lttb(x, y, n_out)")
        b, n_out = Batch(series, n_out, kw.get("device"), kw.get("validate")), _int_arg(args[0], "n_out")
    else:
        _no_extra("lttb", args)
        b, n_out = _Series(series), _int_arg(n_out, "n_out")
    _check_n_out(b.n, n_out)
    b.ready()
    xdt, ydt = _codes(b)
    out = torch.empty((b.B, n_out), dtype=torch.int64, device=b.device)
    x = b.x
    if x is not None and not x.is_cuda:
        x = x.to(b.device)  # full LTTB reads every x
    with _ctx(b):
        st = N.stream_ptr(b.device)
        wsb = N.workspace_bytes(N.OP_LTTB, b.B, b.n, n_out, 0, ydt)
        ws = N.stream_workspace(wsb, b.device, st, b.n)
        N.check(N.lib().mmlttb_lttb(x.data_ptr(), xdt, b.x_ld, b.y.data_ptr(), ydt, b.n, b.B, b.n, n_out,
                                    out.data_ptr(), ws.data_ptr(), wsb, st), "lttb", b.n)
    return b.ret(out)


def minmax_preselect(series, n_out, r_ps, parallel=False, *args, **kw):
    """MinMax candidate preselection for MinMaxLTTB (downsamplers.py:135-161).

    Flat form: ``minmax_preselect(x, y, n_out, r_ps)``.
    """
    _no_extra("minmax_preselect", args)
    if _is_flat(series):
        b = Batch(series, n_out, kw.get("device"), kw.get("validate"))
        n_out, r_ps = _int_arg(r_ps, "n_out"), _int_arg(parallel, "r_ps")
    else:
        b, n_out, r_ps = _Series(series), _int_arg(n_out, "n_out"), _int_arg(r_ps, "r_ps")
    k = _check_preselect(b.n, n_out, r_ps)
    b.ready()
    _, ydt = _codes(b)
    cap = 2 + 2 * k
    out = torch.empty((b.B, cap), dtype=torch.int64, device=b.device)
    cnt = torch.empty(b.B, dtype=torch.int64, device=b.device)
    with _ctx(b):
        wsb = N.lib().mmlttb_workspace_bytes(N.OP_PRESELECT, b.B, b.n, n_out, r_ps, ydt)
        ws = N.workspace(wsb, b.device, b.n)
        ticket = b.arm()
        N.check(N.lib().mmlttb_minmax_preselect(b.y.data_ptr(), ydt, b.n, b.B, b.n, n_out, r_ps, out.data_ptr(),
                                                cap, cnt.data_ptr(), ws.data_ptr(), wsb, N.stream_ptr(b.device)),
                "minmax_preselect", b.n)
    b.post_check(ws, "minmax_preselect", ticket)
    return _counted(b, out, cnt)


def _minmaxlttb_batch(b, n_out: int, r_ps: int):
    b.ready()
    xdt, ydt = _codes(b)
    out = torch.empty((b.B, n_out), dtype=torch.int64, device=b.device)
    with _ctx(b):
        st = N.stream_ptr(b.device)
        wsb = N.workspace_bytes(N.OP_MINMAXLTTB, b.B, b.n, n_out, r_ps, ydt)
        ws = N.stream_workspace(wsb, b.device, st, b.n)
        ticket = b.arm()
        N.check(N.lib().mmlttb_minmaxlttb(N.ptr(b.x), xdt, b.x_ld, b.y.data_ptr(), ydt, b.n, b.B, b.n, n_out,
                                          r_ps, out.data_ptr(), None, ws.data_ptr(), wsb, st),
                "minmaxlttb", b.n)
    b.post_check(ws, "minmaxlttb", ticket)
    return b.ret(out)


def minmaxlttb(series, n_out, r_ps=4, parallel=False, *args, minmax_ratio=None, device=None, validate=None):
    """MinMax preselection, then LTTB on the candidates (downsamplers.py:182-209).

    Reference form: ``minmaxlttb(series, n_out, r_ps=4, parallel=False)``.
    Flat form (north star): ``minmaxlttb(x, y, n_out, minmax_ratio=4)`` with
    ``y`` of shape [N] or [B, N]; returns [n_out] or [B, n_out].
    """
    _no_extra("minmaxlttb", args)
    if _is_flat(series):  # minmaxlttb(x, y, n_out[, minmax_ratio])
        x, y = series, n_out
        n_out = _int_arg(r_ps, "n_out")
        if minmax_ratio is not None and parallel is not False:
            raise TypeError("minmax_ratio given both positionally and by keyword")
        r_ps = _int_arg(minmax_ratio if minmax_ratio is not None else (4 if parallel is False else parallel),
                        "minmax_ratio")
        b = Batch(x, y, device, validate)
    else:
        n_out = _int_arg(n_out, "n_out")
        if minmax_ratio is not None:
            r_ps = minmax_ratio
        r_ps = _int_arg(r_ps, "r_ps")
        b = _Series(series, device)
    if r_ps == 1:
        _check_n_out(b.n, n_out)
        if n_out % 2:
            raise OddNOut(f"minmax needs an even n_out, got {n_out}")
        return _minmax_like(b, n_out, "minmax", force=True)
    _check_preselect(b.n, n_out, r_ps)
    return _minmaxlttb_batch(b, n_out, r_ps)


# ------------------------------------------------------------ dispatch ------
def run_parallel(series: TimeSeries, config: DownsampleConfig):
    """Parallel dispatch (downsamplers.py:224-244); identical output to sequential."""
    if not config.parallel:
        raise ValueError("run_parallel needs a config with parallel=True")
    validate(series, config)
    if config.algorithm is Algorithm.LTTB:
        raise NotParallelizable("LTTB is not parallelizable")
    return _dispatch(series, config)


def _dispatch(series, config):
    algo = config.algorithm
    if algo is Algorithm.EVERY_NTH:
        return every_nth(series, config.n_out)
    if algo is Algorithm.MINMAX:
        return minmax(series, config.n_out)
    if algo is Algorithm.M4:
        return m4(series, config.n_out)
    if algo is Algorithm.LTTB:
        return lttb(series, config.n_out)
    return minmaxlttb(series, config.n_out, config.r_ps)


def downsample(series: TimeSeries, config: DownsampleConfig):
    """Dispatch a config to the matching algorithm (downsamplers.py:247-260)."""
    validate(series, config)
    if config.parallel:
        return run_parallel(series, config)
    return _dispatch(series, config)
