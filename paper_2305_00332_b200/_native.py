"""ctypes binding of ``libmmlttb.so`` (the C ABI declared in include/mmlttb.h).

This is the ONLY compute path of the package: there is no CPU fallback.  If
the shared library is missing or CUDA is unavailable, every downsampling call
raises instead of silently computing somewhere else.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import torch

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "libmmlttb.so"

MM_F32, MM_F64, MM_I64, MM_I32 = 0, 1, 2, 3
OP_MINMAXLTTB, OP_PRESELECT, OP_LTTB, OP_MINMAX, OP_M4 = 0, 1, 2, 3, 4
MM_OK, MM_EINVAL, MM_ECUDA, MM_EWORKSPACE, MM_ERANGE = 0, -1, -2, -3, -4

DTYPE_CODE = {
    torch.float32: MM_F32,
    torch.float64: MM_F64,
    torch.int64: MM_I64,
    torch.int32: MM_I32,
}

_lock = threading.Lock()
_lib = None

_i64, _i32, _p = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
_SIGS = {
    "mmlttb_version": (_i32, []),
    "mmlttb_last_error": (ctypes.c_char_p, []),
    "mmlttb_launch_count": (_i64, []),
    "mmlttb_repair_scans": (_i64, []),
    "mmlttb_stage_timer": (_i32, [_i32]),
    "mmlttb_stage_timer_read": (_i32, [_p, _p]),
    "mmlttb_trace": (_i32, [_i32]),
    "mmlttb_trace_read": (_i64, [_p, _i64]),
    "mmlttb_status_arm": (_i64, []),
    "mmlttb_status_ring": (_p, []),
    "mmlttb_status_poll": (_i32, [_i64, _i32]),
    "mmlttb_workspace_bytes": (_i64, [_i32, _i64, _i64, _i64, _i64, _i32]),
    "mmlttb_minmaxlttb": (_i32, [_p, _i32, _i64, _p, _i32, _i64, _i64, _i64, _i64, _i64, _p, _p, _p, _i64, _p]),
    "mmlttb_minmax_preselect": (_i32, [_p, _i32, _i64, _i64, _i64, _i64, _i64, _p, _i64, _p, _p, _i64, _p]),
    "mmlttb_lttb": (_i32, [_p, _i32, _i64, _p, _i32, _i64, _i64, _i64, _i64, _p, _p, _i64, _p]),
    "mmlttb_minmax": (_i32, [_p, _i32, _i64, _i64, _i64, _i64, _p, _p, _p, _i64, _p]),
    "mmlttb_m4": (_i32, [_p, _i32, _i64, _i64, _i64, _i64, _p, _p, _p, _i64, _p]),
    "mmlttb_every_nth": (_i32, [_i64, _i64, _p, _p]),
    "mmlttb_extrema_workspace_bytes": (_i64, [_i64, _i64]),
    "mmlttb_extrema_by_bucket": (_i32, [_p, _i32, _p, _i64, _i64, _p, _p, _p, _i64, _p]),
    "mmlttb_lttb_select_workspace_bytes": (_i64, [_i64, _i64]),
    "mmlttb_lttb_select": (_i32, [_p, _i32, _p, _i32, _i64, _p, _i64, _p, _p, _i64, _p]),
    "mmlttb_shard_workspace_bytes": (_i64, [_i64, _i64, _i64, _i64, _i64]),
    "mmlttb_shard_preselect": (_i32, [_p, _i32, _p, _i32, _i64, _i64, _i64, _i64, _i64, _i64, _i32, _i32,
                                      _p, _p, _p, _p, _p, _i64, _p]),
    "mmlttb_merge_shards": (_i32, [_p, _p, _p, _p, _i64, _i64, _p, _p, _p, _p, _p]),
    "mmlttb_merge_packed": (_i32, [_p, _i64, _i64, _p, _p, _p, _p, _p]),
    "mmlttb_p2p_publish": (_i32, [_p, _p, _p, _p, _i64, _p, _p, _p, _i64, _i64, ctypes.c_uint32, _p]),
    "mmlttb_p2p_merge": (_i32, [_p, _p, _p, _i64, _i64, _i64, ctypes.c_uint32, _p, _p, _p, _p, _p]),
    "mmlttb_lttb_preselected_workspace_bytes": (_i64, [_i64, _i64, _i64]),
    "mmlttb_lttb_preselected": (_i32, [_p, _p, _p, _p, _i64, _i64, _i64, _i64, _p, _p, _i64, _p]),
    "mmlttb_validate": (_i32, [_p, _i32, _p, _i32, _i64, _p, _p]),
    "mmlttb_validate_batch": (_i32, [_p, _i32, _i64, _p, _i32, _i64, _i64, _i64, _p, _p]),
    "mmlttb_deinterleave_f64": (_i32, [_p, _i64, _p, _p, _p]),
    "mmlttb_raster_workspace_bytes": (_i64, [_i64, _i64, _i64]),
    "mmlttb_rasterize": (_i32, [_p, _i32, _p, _i32, _p, _i64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                ctypes.c_double, _i64, _i64, _p, _p, _i64, _p]),
    "mmlttb_conv_mask": (_i32, [_p, _p, _i64, _i64, _i32, _p, _p]),
    "mmlttb_pixel_metrics": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p, _p, _i64, _p]),
}
EXPORTED = tuple(_SIGS)


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load the library and declare every entry point (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # MMLTTB_LIB: an alternative in-tree build (A/B tuning builds under tools/)
        p = Path(path) if path else Path(os.environ.get("MMLTTB_LIB", LIB_PATH))
        if not p.exists():
            raise ImportError(
                f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the device path has no CPU fallback)")
        L = ctypes.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if path is None:
            _lib = L
        return L


def lib() -> ctypes.CDLL:
    return _lib if _lib is not None else load()


_cuda_ok = False


def require_cuda(device=None) -> torch.device:
    global _cuda_ok
    if not _cuda_ok:  # availability cannot change once the driver has initialised
        if not torch.cuda.is_available():
            raise errors.CudaError("no CUDA device: the MinMaxLTTB device path has no CPU fallback")
        lib()
        _cuda_ok = True
    if isinstance(device, torch.device) and device.type == "cuda" and device.index is not None:
        return device
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise errors.CudaError(f"device {d} is not a CUDA device")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device: torch.device) -> int:
    """Raw cudaStream_t of the device's current torch stream (per-call hot path)."""
    try:
        return torch._C._cuda_getCurrentRawStream(device.index)
    except (AttributeError, TypeError):  # pragma: no cover - older torch
        return torch.cuda.current_stream(device).cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def check(rc: int, what: str, n: int | None = None) -> None:
    if rc == MM_OK:
        return
    msg = lib().mmlttb_last_error().decode(errors="replace")
    if rc == MM_ECUDA and "out of memory" in msg:
        raise errors.OutOfMemory(f"out of memory at N={n} in {what}: {msg}")
    if rc in (MM_EINVAL, MM_ERANGE):
        raise errors.ValidationError(f"{what}: {msg}")
    raise errors.CudaError(f"{what} failed ({rc}): {msg}")


_wsb_cache: dict = {}


def workspace_bytes(op: int, B: int, n: int, n_out: int, r_ps: int, ydt: int) -> int:
    """mmlttb_workspace_bytes, memoised (a pure function of its arguments)."""
    key = (op, B, n, n_out, r_ps, ydt)
    v = _wsb_cache.get(key)
    if v is None:
        v = _wsb_cache[key] = int(lib().mmlttb_workspace_bytes(op, B, n, n_out, r_ps, ydt))
    return v


_ws_local = threading.local()
WS_CACHE_MAX = 64 << 20  # larger workspaces are allocated per call


def stream_workspace(nbytes: int, device: torch.device, stream: int, n: int | None = None) -> torch.Tensor:
    """Workspace reused across calls on the same (thread, device, stream).

    Calls on one stream are ordered, so a later call's kernels only start after
    the earlier call's are done with the buffer; the cache is thread-local so two
    host threads sharing a stream never interleave their use of one buffer.
    """
    if nbytes > WS_CACHE_MAX:
        return workspace(nbytes, device, n)
    d = getattr(_ws_local, "d", None)
    if d is None:
        d = _ws_local.d = {}
    key = (device.index, stream)
    t = d.get(key)
    if t is None or t.numel() < nbytes:
        t = d[key] = workspace(max(int(nbytes), 1 << 20), device, n)
    return t


def workspace(nbytes: int, device: torch.device, n: int | None = None) -> torch.Tensor:
    try:
        return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
    except torch.cuda.OutOfMemoryError as exc:  # pragma: no cover - needs a GPU
        raise errors.OutOfMemory(f"failed to allocate the N={n} workspace ({nbytes} bytes)") from exc
