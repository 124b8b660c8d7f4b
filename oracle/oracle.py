"""ctypes front-end of the CPU oracle (tsdown_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker and the CPU baseline arm.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product package never does.

Each wrapper mirrors one reference entry point of package ``tsdown``
(``/root/reference/pkg/src/tsdown/downsamplers.py``), takes numpy arrays and
returns a fresh ``np.ndarray[int64]``.  Float inputs are handed to the C code
as float64 exactly as ``TimeSeries`` would hold them (``core.py:48-53``); the
``*_typed`` variants convert per sub-bucket instead (the chunked oracle of
SURVEY §8(c)), so very large float32 series never need an f64 copy.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

# return codes of tsdown_oracle.c -> reference exception class names
_ERRORS = {
    -1: "NOutOfRange",
    -2: "MemoryError",
    -3: "OddNOut",
    -4: "BadPreselectionRatio",
    -5: "RatioTooLargeForSeries",
    -6: "NOutNotDivisibleBy4",
}
_DT = {np.dtype(np.float32): 0, np.dtype(np.float64): 1, np.dtype(np.int64): 2, np.dtype(np.int32): 3}


class OracleError(ValueError):
    """Raised with the reference exception name as ``.name``."""

    def __init__(self, code: int):
        self.name = _ERRORS.get(code, f"code{code}")
        super().__init__(self.name)


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return all(t in flags for t in ("avx512f", "avx512bw", "avx512vl", "avx512dq"))
    except OSError:
        return False


def build() -> None:
    """Compile both ISA variants (gcc; no reference build system involved)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


_LIB = None


def lib() -> ctypes.CDLL:
    global _LIB
    if _LIB is not None:
        return _LIB
    name = "liboracle_v4.so" if _cpu_has_avx512() else "liboracle_v3.so"
    path = HERE / name
    if not path.exists():
        build()
    L = ctypes.CDLL(str(path))
    i64, p = ctypes.c_int64, ctypes.c_void_p
    sig = {
        "or_partition": (ctypes.c_int, [i64, i64, i64, p]),
        "or_extrema_by_bucket": (None, [p, p, i64, p, p, ctypes.c_int]),
        "or_lttb_select": (None, [p, p, i64, p, i64, p]),
        "or_lttb": (ctypes.c_int, [p, p, i64, i64, p]),
        "or_minmax": (i64, [p, i64, i64, p, ctypes.c_int]),
        "or_minmax_preselect": (i64, [p, i64, i64, i64, p, ctypes.c_int]),
        "or_minmax_with_endpoints": (i64, [p, i64, i64, p, ctypes.c_int]),
        "or_minmaxlttb": (i64, [p, p, i64, i64, i64, p, ctypes.c_int]),
        "or_m4": (i64, [p, i64, i64, p, ctypes.c_int]),
        "or_minmax_preselect_typed": (i64, [p, ctypes.c_int, i64, i64, i64, p, ctypes.c_int]),
        "or_minmaxlttb_typed": (i64, [p, ctypes.c_int, p, ctypes.c_int, i64, i64, i64, p, ctypes.c_int]),
        "or_shard_preselect_typed": (i64, [p, ctypes.c_int, i64, i64, i64, i64, i64, i64, i64, ctypes.c_int,
                                           ctypes.c_int, p, ctypes.c_int]),
        "or_max_threads": (ctypes.c_int, []),
    }
    for fn, (res, args) in sig.items():
        f = getattr(L, fn)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


def max_threads() -> int:
    return int(lib().or_max_threads())


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _check(rc: int) -> int:
    if rc < 0:
        if rc == -2:
            raise MemoryError("oracle allocation failed")
        raise OracleError(rc)
    return rc


def partition(start: int, end: int, k: int) -> np.ndarray:
    """core.py:161-175."""
    out = np.empty(max(k, 0) + 1, dtype=np.int64)
    _check(lib().or_partition(start, end, k, _ptr(out)))
    return out


def extrema_by_bucket(ys, bounds, threads: int = 1):
    """_kernels.py:63-78 (threads > 1 = the prange variant)."""
    ys = _f64(ys)
    bounds = np.ascontiguousarray(bounds, dtype=np.int64)
    k = bounds.shape[0] - 1
    mn = np.empty(k, dtype=np.int64)
    mx = np.empty(k, dtype=np.int64)
    lib().or_extrema_by_bucket(_ptr(ys), _ptr(bounds), k, _ptr(mn), _ptr(mx), threads)
    return mn, mx


def lttb(xs, ys, n_out: int) -> np.ndarray:
    """downsamplers.py:115-132."""
    xs, ys = _f64(xs), _f64(ys)
    out = np.empty(max(n_out, 0), dtype=np.int64)
    _check(lib().or_lttb(_ptr(xs), _ptr(ys), xs.shape[0], n_out, _ptr(out)))
    return out


def minmax(ys, n_out: int, threads: int = 1) -> np.ndarray:
    """downsamplers.py:72-92."""
    ys = _f64(ys)
    out = np.empty(max(n_out, 0), dtype=np.int64)
    m = _check(lib().or_minmax(_ptr(ys), ys.shape[0], n_out, _ptr(out), threads))
    return out[:m].copy()


def m4(ys, n_out: int, threads: int = 1) -> np.ndarray:
    """downsamplers.py:95-112."""
    ys = _f64(ys)
    out = np.empty(max(n_out, 0), dtype=np.int64)
    m = _check(lib().or_m4(_ptr(ys), ys.shape[0], n_out, _ptr(out), threads))
    return out[:m].copy()


def minmax_preselect(ys, n_out: int, r_ps: int, threads: int = 1) -> np.ndarray:
    """downsamplers.py:135-161."""
    ys = _f64(ys)
    k = max((n_out - 2) * (r_ps // 2), 0)
    out = np.empty(2 + 2 * k, dtype=np.int64)
    m = _check(lib().or_minmax_preselect(_ptr(ys), ys.shape[0], n_out, r_ps, _ptr(out), threads))
    return out[:m].copy()


def minmaxlttb(xs, ys, n_out: int, r_ps: int = 4, threads: int = 1) -> np.ndarray:
    """downsamplers.py:182-209 (r_ps == 1 -> downsamplers.py:164-179)."""
    xs, ys = _f64(xs), _f64(ys)
    out = np.empty(max(n_out, 0), dtype=np.int64)
    m = _check(lib().or_minmaxlttb(_ptr(xs), _ptr(ys), ys.shape[0], n_out, r_ps, _ptr(out), threads))
    return out[:m].copy()


def _typed(a):
    a = np.ascontiguousarray(a)
    if a.dtype not in _DT:
        a = a.astype(np.float64)
    return a, _DT[a.dtype]


def minmax_preselect_typed(ys, n_out: int, r_ps: int, threads: int = 0) -> np.ndarray:
    """Chunked minmax_preselect over f32/f64 storage."""
    ys, ydt = _typed(ys)
    threads = threads or max_threads()
    k = max((n_out - 2) * (r_ps // 2), 0)
    out = np.empty(2 + 2 * k, dtype=np.int64)
    m = _check(lib().or_minmax_preselect_typed(_ptr(ys), ydt, ys.shape[0], n_out, r_ps, _ptr(out), threads))
    return out[:m].copy()


def minmaxlttb_typed(xs, ys, n_out: int, r_ps: int = 4, threads: int = 0) -> np.ndarray:
    """Chunked minmaxlttb (r_ps >= 2) over typed storage."""
    xs, xdt = _typed(xs)
    ys, ydt = _typed(ys)
    threads = threads or max_threads()
    out = np.empty(max(n_out, 0), dtype=np.int64)
    m = _check(lib().or_minmaxlttb_typed(_ptr(xs), xdt, _ptr(ys), ydt, ys.shape[0], n_out, r_ps,
                                         _ptr(out), threads))
    return out[:m].copy()


def shard_preselect_typed(ys_shard, lo: int, n: int, n_out: int, r_ps: int, b0: int, b1: int, emit_first: bool,
                          emit_last: bool, threads: int = 0) -> np.ndarray:
    """One rank's bucket-range share of minmax_preselect (global indices)."""
    ys, ydt = _typed(ys_shard)
    threads = threads or max_threads()
    out = np.empty(2 * (b1 - b0) + 2, dtype=np.int64)
    m = _check(lib().or_shard_preselect_typed(_ptr(ys), ydt, lo, ys.shape[0], n, n_out, r_ps, b0, b1,
                                              int(emit_first), int(emit_last), _ptr(out), threads))
    return out[:m].copy()


def minmaxlttb_batch_typed(xs, ys2d, n_out: int, r_ps: int = 4, threads: int = 0) -> np.ndarray:
    """Per-row minmaxlttb over a [B, N] matrix sharing x (C4)."""
    return np.stack([minmaxlttb_typed(xs, ys2d[i], n_out, r_ps, threads) for i in range(ys2d.shape[0])])


if __name__ == "__main__":  # pragma: no cover
    build()
    print("oracle built:", sorted(p.name for p in HERE.glob("liboracle_*.so")))
    os.sys.exit(0)
