"""CPU arm of bench.py: the REFERENCE's own implementation timed on host cores.

TEST / MEASUREMENT INFRASTRUCTURE ONLY (bench.py's ``--impl reference`` and
its ``cpu_baseline`` leg).  It times package ``tsdown`` -- the reference
itself, installed unmodified into the git-ignored ``oracle/_ref`` by
``make -C oracle ref`` (pip --target from a /tmp copy of
/root/reference/pkg; the directory travels to the GPU box with the snapshot)
-- through its public API and its stock numba kernels:

* ``tsdown.minmaxlttb(series, n_out, r_ps, parallel=False)`` (sequential,
  ``downsamplers.py:182-209``), and
* ``tsdown.run_parallel(series, DownsampleConfig(..., parallel=True,
  threads=cores))`` (``downsamplers.py:224-244``: numba ``prange`` over
  buckets, ``_kernels.py:71-78``), for ``lttb`` (C2) the sequential
  ``tsdown.lttb`` only (LTTB is not parallelizable, ``:238-239``),

with the reference's own timing boundary (``bench.py:120-134``: the series is
built as a ``TimeSeries`` -- its float64 copies -- outside the timed region;
one discarded warm-up, then the median of the timed repetitions).  If the
reference cannot be imported (no ``oracle/_ref``, no numba), the C
restatement ``oracle/tsdown_oracle.c`` (OpenMP) is timed instead and the
line says ``kind: "port"``.

Thread count and pinning are fixed BEFORE numba / OpenMP initialise:
``NUMBA_NUM_THREADS`` = all cores this process may run on,
``OMP_PROC_BIND=close``, ``OMP_PLACES=cores`` -- so call ``configure_threads``
before anything imports numba or loads an OpenMP runtime (bench.py runs this
arm in a fresh interpreter for exactly that reason).
"""
from __future__ import annotations

import os
import statistics
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"


def configure_threads() -> int:
    cores = len(os.sched_getaffinity(0))
    os.environ["NUMBA_NUM_THREADS"] = str(cores)
    os.environ["OMP_NUM_THREADS"] = str(cores)
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(REF_DIR / ".numba_cache"))
    return cores


def import_reference():
    """The unmodified reference package from oracle/_ref, or None (and why)."""
    if not (REF_DIR / "tsdown" / "__init__.py").exists():
        return None, "oracle/_ref not built (make -C oracle ref)"
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import tsdown  # noqa: F401
        import numba  # noqa: F401
    except Exception as e:  # pragma: no cover - depends on the host image
        return None, f"reference import failed: {e!r}"
    return tsdown, None


# -------------------------------------------------------------- workloads --
def _par_chunks(n, fn, chunk=1 << 24, threads=None):
    threads = threads or len(os.sched_getaffinity(0))
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda c: fn(c * chunk, min(n, (c + 1) * chunk), c), range((n + chunk - 1) // chunk)))


def make_series(name: str, n: int, seed: int):
    """Host arrays with the workload's recipe (bench.py WORKLOADS), generated
    chunk-parallel (independent PCG64 streams per 16M-point chunk, spawned
    from `seed`): values differ from the device Philox stream, shapes, dtypes
    and distributions do not -- the CPU kernels' speed does not depend on them."""
    y = np.empty(n, dtype=np.float32 if name.startswith(("c3", "c4", "c5")) else np.float64)
    nch = (n + (1 << 24) - 1) >> 24
    seqs = np.random.SeedSequence(seed).spawn(nch)
    if name.startswith("c3"):
        def fill(lo, hi, c):
            i = np.arange(lo, hi, dtype=np.float64)
            v = np.sin(2 * np.pi * i / 1e3)
            v += np.sin(2 * np.pi * i / 1e5)
            v += np.sin(2 * np.pi * i / 1e7)
            v += np.random.Generator(np.random.PCG64(seqs[c])).standard_normal(hi - lo)
            y[lo:hi] = v
        _par_chunks(n, fill)
    else:  # random walks (+ noise and spikes for c2 / c5): steps per chunk, then one cumsum
        steps = np.empty(n, dtype=np.float64)

        def fill(lo, hi, c):
            steps[lo:hi] = np.random.Generator(np.random.PCG64(seqs[c])).standard_normal(hi - lo)
        _par_chunks(n, fill)
        w = np.cumsum(steps, out=steps)
        if name in ("c2", "c5"):
            rng = np.random.Generator(np.random.PCG64(seed + 1))
            frac, sig = (0.001, 0.5) if name == "c2" else (0.01, 1.0)
            if name == "c2":
                w += rng.normal(0.0, 0.5, n)
            spike = rng.random(n) < frac
            w += np.where(spike, np.where(rng.random(n) < 0.5, -1.0, 1.0) * 50.0 * sig, 0.0)
        y[:] = w
        del steps
    if name == "c5":
        x = np.cumsum(np.random.Generator(np.random.PCG64(seed + 2)).exponential(1.0, n))
    else:
        x = np.arange(n, dtype=np.int64)
    return x, y


def _median_run(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        fn()
        times.append(time.perf_counter() - t0)
    return statistics.median(times), times


def time_reference(name: str, n: int, n_out: int, r_ps: int, op: str, steps: int, warmup: int,
                   seq_steps: int = 3, max_points: int | None = None, seed: int = 3) -> dict:
    """Time the CPU arm on the workload (or its first `max_points` points).

    Returns a dict with value (points/s of the all-cores run: the reference's
    parallel path; LTTB: sequential), the sequential figure, and a description.
    """
    cores = configure_threads()
    m = n if max_points is None else min(n, max_points)
    n_out_s = n_out if m == n else max(3, int(round((n_out - 2) * m / n)) + 2)
    ref, why = import_reference()
    x, y = make_series(name, m, seed)
    out = {"cores": cores, "points": m, "n_out": n_out_s}
    if ref is not None:
        import numba

        t0 = time.perf_counter()
        ts = ref.TimeSeries(x, y)  # the reference's f64 copies + checks: outside the timed region
        out["timeseries_build_s"] = time.perf_counter() - t0
        del x, y
        if op == "lttb":
            fpar = fseq = lambda: ref.lttb(ts, n_out_s)  # noqa: E731  (not parallelizable)
        else:
            cfg = ref.DownsampleConfig(ref.Algorithm.MINMAXLTTB, n_out_s, r_ps=r_ps, parallel=True, threads=cores)
            fpar = lambda: ref.run_parallel(ts, cfg)  # noqa: E731
            fseq = lambda: ref.minmaxlttb(ts, n_out_s, r_ps, parallel=False)  # noqa: E731
        kind = "reference"
        layer = None
        impl = (f"tsdown {getattr(ref, '__version__', '0.1.0')} (unmodified, oracle/_ref) + numba "
                f"{numba.__version__}")
    else:
        sys.path.insert(0, str(HERE.parent))
        from oracle import oracle as O

        yf = y.astype(np.float64)
        xf = x.astype(np.float64)
        del x, y
        if op == "lttb":
            fpar = fseq = lambda: O.lttb(xf, yf, n_out_s)  # noqa: E731
        else:
            fpar = lambda: O.minmaxlttb(xf, yf, n_out_s, r_ps, cores)  # noqa: E731
            fseq = lambda: O.minmaxlttb(xf, yf, n_out_s, r_ps, 1)  # noqa: E731
        kind = "port"
        layer = None
        impl = f"oracle/tsdown_oracle.c (OpenMP) -- reference unavailable: {why}"
    med, times = _median_run(fpar, steps, max(1, warmup))
    if ref is not None:
        try:
            layer = numba.threading_layer()
        except Exception:  # pragma: no cover
            layer = None
    out.update(value=m / med, ms_per_step=med * 1e3, times_ms=[t * 1e3 for t in times], kind=kind, impl=impl,
               threading_layer=layer, par_cores=cores if op != "lttb" else 1)
    if op != "lttb" and seq_steps > 0:
        smed, _ = _median_run(fseq, seq_steps, 1)
        out["sequential"] = {"value": m / smed, "ms_per_step": smed * 1e3, "cores": 1, "runs": seq_steps}
    par = f"{cores} threads (numba prange, layer {layer})" if kind == "reference" and op != "lttb" else (
        "1 thread (sequential by contract)" if op == "lttb" else f"{cores} OpenMP threads")
    out["sample"] = (f"{name}: {'full workload' if m == n else f'first {m:.3g} points'} of one series "
                     f"(n={m}, n_out={n_out_s}, r_ps={r_ps}, {op}); {impl}; {par}; "
                     f"OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')}; median of {steps} after {max(1, warmup)} "
                     "warm-up; TimeSeries (f64 copies) built outside the timed region as in the reference's "
                     "bench.py:124-127")
    return out
