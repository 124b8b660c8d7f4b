"""Generate the golden fixtures from the REFERENCE itself (package ``tsdown``).

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py [--skip-c4] [--skip-c5]

Writes, next to this script:
  kats.json       SPEC known-answer examples evaluated by the reference
  fuzz.json.gz    outputs (or exception class) of tests/fuzzgen.py cases
  configs.json    BASELINE.json C1, C2, C3 (r=2..32), C5 outputs + sha256
  c4.json         sha256 of every C4 series' output (+ 8 full outputs)
  config_errors.json  DownsampleConfig / validate / downsample error parity

C5 (2e9 points) uses the chunked reference procedure of SURVEY §8(c): the
global partition(1, N-1, k), sub-bucket-aligned slices converted to float64,
the reference's own ``_extrema_by_bucket`` and ``_interleave_minmax``, then
the reference ``lttb`` over ``TimeSeries(x[pre], y[pre])``.  It is checked
against the unchunked reference at 1e7 before being trusted.
"""
from __future__ import annotations

import argparse
import gzip
import hashlib
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

import numpy as np  # noqa: E402

import tsdown  # noqa: E402
from tsdown import _kernels as K  # noqa: E402
from tsdown import downsamplers as D  # noqa: E402

import fuzzgen  # noqa: E402
import recipes  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def ref_call(op, x, y, n_out, r_ps):
    try:
        ts = tsdown.TimeSeries(x, y)
        if op == "minmaxlttb":
            out = tsdown.minmaxlttb(ts, n_out, r_ps)
        elif op == "lttb":
            out = tsdown.lttb(ts, n_out)
        elif op == "minmax":
            out = tsdown.minmax(ts, n_out)
        elif op == "minmax_preselect":
            out = tsdown.minmax_preselect(ts, n_out, r_ps)
        elif op == "m4":
            out = tsdown.m4(ts, n_out)
        else:
            raise ValueError(op)
        return {"out": [int(v) for v in out]}
    except tsdown.errors.TsdownError as e:
        return {"error": type(e).__name__}


def make_kats():
    ts = tsdown.TimeSeries
    a = [1, 3, 2, 0, 5, 4, 9, 8]
    xa = list(range(8))
    kats = {
        "partition": {
            "0,10,2": tsdown.partition(0, 10, 2).boundaries.tolist(),
            "1,9,4": tsdown.partition(1, 9, 4).boundaries.tolist(),
            "0,10,3": tsdown.partition(0, 10, 3).boundaries.tolist(),
        },
        "minmax": tsdown.minmax(ts(xa, a), 4).tolist(),
        "m4": tsdown.m4(ts(xa, a), 8).tolist(),
        "lttb_spike": tsdown.lttb(ts(list(range(6)), [0, 0, 10, 0, 0, 0]), 3).tolist(),
        "minmax_constant_n10": tsdown.minmax(ts(list(range(10)), [3.0] * 10), 4).tolist(),
        "lttb_collinear_n20": tsdown.lttb(ts(list(range(20)), list(range(20))), 6).tolist(),
        "preselect_sin10": tsdown.minmax_preselect(ts(list(range(10)), np.sin(np.arange(10.0))), 4, 2).tolist(),
        "minmaxlttb_r1": tsdown.minmaxlttb(ts(xa, a), 4, r_ps=1).tolist(),
        "every_nth_10_5": tsdown.every_nth(ts(list(range(10)), [0.0] * 10), 5).tolist(),
        "every_nth_7_3": tsdown.every_nth(ts(list(range(7)), [0.0] * 7), 3).tolist(),
        "signed_zero_minmax": tsdown.minmax(ts([0, 1, 2, 3], [0.0, -0.0, 0.0, -0.0]), 2 * 1 + 2).tolist(),
    }
    # SPEC.md's literal expectations
    kats["spec_literal"] = {
        "minmax": [1, 3, 5, 6],
        "m4": [0, 1, 3, 4, 5, 6, 7],
        "lttb_spike": [0, 2, 5],
        "preselect_sin10": [0, 2, 4, 5, 8, 9],
        "minmaxlttb_r1": [0, 3, 5, 7],
    }
    return kats


def make_fuzz():
    cases = []
    for i in range(fuzzgen.N_CASES):
        c = fuzzgen.make_case(i)
        r = ref_call(c["op"], c["x"], c["y"], c["n_out"], c["r_ps"])
        r.update(i=i, kind=c["kind"], op=c["op"], n=c["n"], n_out=c["n_out"], r_ps=c["r_ps"],
                 digest=fuzzgen.digest(c["x"], c["y"]))
        cases.append(r)
    return cases


def make_config_errors():
    """DownsampleConfig construction, validate() and downsample() outcomes."""
    rng = np.random.Generator(np.random.PCG64(77))
    out = []
    for n in (3, 4, 5, 10, 57):
        x = np.arange(n)
        y = rng.standard_normal(n)
        ts = tsdown.TimeSeries(x, y)
        for algo in ("everynth", "minmax", "m4", "lttb", "minmaxlttb"):
            for n_out in (0, 2, 3, 4, 5, 8, n, n + 1):
                for r_ps in (0, 1, 2, 3, 4, 8, 64):
                    for parallel in (False, True):
                        for threads in (0, 1, 3):
                            rec = dict(n=n, algo=algo, n_out=n_out, r_ps=r_ps, parallel=parallel,
                                       threads=threads)
                            try:
                                cfg = tsdown.DownsampleConfig(algo, n_out, r_ps, parallel, threads)
                            except (tsdown.errors.TsdownError, ValueError) as e:
                                rec["config_error"] = type(e).__name__
                                out.append(rec)
                                continue
                            try:
                                tsdown.validate(ts, cfg)
                                rec["validate"] = "ok"
                            except tsdown.errors.TsdownError as e:
                                rec["validate"] = type(e).__name__
                            try:
                                rec["out"] = [int(v) for v in tsdown.downsample(ts, cfg)]
                            except (tsdown.errors.TsdownError, ValueError) as e:
                                rec["downsample_error"] = type(e).__name__
                            out.append(rec)
    return out


def chunked_minmaxlttb(x, y, n_out, r_ps, group=64):
    """SURVEY §8(c) chunked reference: slices aligned to sub-bucket edges."""
    n = y.shape[0]
    k = (n_out - 2) * (r_ps // 2)
    bounds = tsdown.partition(1, n - 1, k).boundaries
    imin = np.empty(k, dtype=np.int64)
    imax = np.empty(k, dtype=np.int64)
    for b0 in range(0, k, group):
        b1 = min(k, b0 + group)
        lo, hi = int(bounds[b0]), int(bounds[b1])
        ys = y[lo:hi].astype(np.float64)
        lb = (bounds[b0:b1 + 1] - lo).astype(np.int64)
        mn = np.empty(b1 - b0, dtype=np.int64)
        mx = np.empty(b1 - b0, dtype=np.int64)
        K._extrema_by_bucket_parallel(ys.view(np.int64), lb, mn, mx)
        imin[b0:b1] = mn + lo
        imax[b0:b1] = mx + lo
    pairs = D._interleave_minmax(imin, imax)
    pre = np.empty(pairs.shape[0] + 2, dtype=np.int64)
    pre[0] = 0
    pre[1:-1] = pairs
    pre[-1] = n - 1
    sub = tsdown.TimeSeries(x[pre], y[pre])
    return pre[tsdown.lttb(sub, n_out)]


def make_configs(skip_c5: bool):
    res = {}
    t = time.time()
    x, y = recipes.c1()
    o = tsdown.minmaxlttb(tsdown.TimeSeries(x, y), 1000, 4)
    res["C1"] = {"r4": {"out": o.tolist(), "sha": sha(o)}}
    print(f"C1 done {time.time() - t:.1f}s", flush=True)
    x, y = recipes.c2()
    o = tsdown.lttb(tsdown.TimeSeries(x, y), 2000)
    res["C2"] = {"lttb": {"out": o.tolist(), "sha": sha(o)}}
    # chunked procedure self-check against the unchunked reference
    ts = tsdown.TimeSeries(x, y)
    for r in (2, 4, 32):
        full = tsdown.minmaxlttb(ts, 2000, r)
        assert np.array_equal(full, chunked_minmaxlttb(x, y, 2000, r)), r
    del ts
    print(f"C2 done {time.time() - t:.1f}s", flush=True)
    x, y = recipes.c3()
    ts = tsdown.TimeSeries(x, y)
    res["C3"] = {}
    for r in recipes.CONFIGS["C3"]["r_ps"]:
        o = tsdown.minmaxlttb(ts, 2000, r, parallel=True)
        res["C3"][f"r{r}"] = {"out": o.tolist(), "sha": sha(o)}
    del ts, x, y
    print(f"C3 done {time.time() - t:.1f}s", flush=True)
    if not skip_c5:
        x, y = recipes.c5()
        print(f"C5 generated {time.time() - t:.1f}s", flush=True)
        o = chunked_minmaxlttb(x, y, 4000, 4)
        res["C5"] = {"r4": {"out": o.tolist(), "sha": sha(o)}}
        del x, y
        print(f"C5 done {time.time() - t:.1f}s", flush=True)
    return res


def make_c4():
    n = recipes.CONFIGS["C4"]["n"]
    x = np.arange(n, dtype=np.int64)
    shas, full = [], {}
    for s in range(recipes.CONFIGS["C4"]["batch"]):
        y = recipes.c4_series(s, n)
        o = tsdown.minmaxlttb(tsdown.TimeSeries(x, y), 1000, 4, parallel=True)
        shas.append(sha(o))
        if s in (0, 1, 2, 3, 1000, 2047, 4094, 4095):
            full[str(s)] = o.tolist()
    return {"sha": shas, "full": full}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c4", action="store_true")
    ap.add_argument("--skip-c5", action="store_true")
    ap.add_argument("--only", default="kats,fuzz,errors,configs,c4")
    a = ap.parse_args()
    only = set(a.only.split(","))
    if "kats" in only:
        (HERE / "kats.json").write_text(json.dumps(make_kats(), indent=1))
        print("kats written", flush=True)
    if "fuzz" in only:
        with gzip.open(HERE / "fuzz.json.gz", "wt") as f:
            json.dump(make_fuzz(), f)
        print("fuzz written", flush=True)
    if "errors" in only:
        with gzip.open(HERE / "config_errors.json.gz", "wt") as f:
            json.dump(make_config_errors(), f)
        print("config errors written", flush=True)
    if "configs" in only:
        prev = {}
        p = HERE / "configs.json"
        if p.exists():
            prev = json.loads(p.read_text())
        cur = make_configs(a.skip_c5)
        prev.update(cur)
        p.write_text(json.dumps(prev))
        print("configs written", flush=True)
    if "c4" in only and not a.skip_c4:
        (HERE / "c4.json").write_text(json.dumps(make_c4()))
        print("c4 written", flush=True)


if __name__ == "__main__":
    main()
