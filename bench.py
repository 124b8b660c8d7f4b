#!/usr/bin/env python
"""MinMaxLTTB throughput on B200: input points/s, HBM GB/s and % of roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3_1e9|c1|c2|c3|c4|c5|...] [--impl ours|reference]

A step = one minmaxlttb call (K1 extrema -> K2 compact -> K3 LTTB) over the
workload's series.  Default workload "c3_1e9": BASELINE.json C3's recipe at
N = 1e9 points (float32 y = 3 sinusoids + N(0,1), int64 x, n_out = 2000,
minmax_ratio = 4) -- the north star's "10^9-point series".
Inputs are generated ON the device (torch Philox, seed 3; a 4 GB float32 y
is larger than the 126 MB L2, so consecutive steps never hit in L2) and the
warm-up output is checked index-exactly against the CPU oracle on the same
data (on every rank; rank 0 reports the AND).

--gpus N > 1 without torchrun: the script relaunches itself under
``torch.distributed.run`` with N ranks (and refuses, exit 2, when fewer than
N GPUs are visible or WORLD_SIZE disagrees with --gpus).  With N ranks the
default workload becomes ONE series of N x 1e9 points split by MinMax bucket
ranges (SURVEY 8(e) single-series path: K1 + K2 on each rank's 1e9-point
shard, one NCCL all_gather of the preselected sets, device merge, LTTB):
per-GPU work is fixed, "scaling": "weak".  c4 shards its 4096 series across
ranks (no collective, "strong"); c5s splits the 2e9-point C5 series.

--impl reference times the REFERENCE's own CPU implementation (package
tsdown, unmodified, installed into oracle/_ref; oracle/refbench.py) on the
box's host cores, rank 0 only; the same code supplies our line's
``cpu_baseline`` (run in a fresh interpreter so thread pinning applies).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (N per series, batch, n_out, r_ps, y dtype, x dtype, op)
    "c3_1e9": (1_000_000_000, 1, 2000, 4, "f32", "i64", "minmaxlttb"),
    "c1": (1_000_000, 1, 1000, 4, "f64", "i64", "minmaxlttb"),
    "c2": (10_000_000, 1, 2000, 0, "f64", "i64", "lttb"),
    "c3": (100_000_000, 1, 2000, 4, "f32", "i64", "minmaxlttb"),
    # C3's other preselection ratios (BASELINE.json: minmax_ratio in {2,4,8,16,32})
    "c3r2": (100_000_000, 1, 2000, 2, "f32", "i64", "minmaxlttb"),
    "c3r8": (100_000_000, 1, 2000, 8, "f32", "i64", "minmaxlttb"),
    "c3r16": (100_000_000, 1, 2000, 16, "f32", "i64", "minmaxlttb"),
    "c3r32": (100_000_000, 1, 2000, 32, "f32", "i64", "minmaxlttb"),
    "c4": (1_000_000, 4096, 1000, 4, "f32", "i64", "minmaxlttb"),
    "c5": (2_000_000_000, 1, 4000, 4, "f32", "f64", "minmaxlttb"),
    # one 2e9-point series split by MinMax bucket ranges over the ranks, one
    # all_gather of the preselected sets; strong scaling
    "c5s": (2_000_000_000, 1, 4000, 4, "f32", "i64", "minmaxlttb"),
}
METRIC = "MinMaxLTTB input points/sec and HBM GB/s (% roofline) at 1/2/4/8 B200"
UNIT = "points/s"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic():
    p = ROOT / "profiles" / "k1_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return None
    return None


class Clocks:
    """nvidia-smi sampling during a timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.rows = []

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
            out, _ = self.p.communicate()
        for line in out.splitlines():
            f = [t.strip() for t in line.split(",")]
            if len(f) >= 7:
                self.rows.append(f)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------- inputs ---
def make_shard(name, dev, seed, lo, hi):
    """Elements [lo, hi) of a C3-recipe series, generated on this rank's device."""
    import torch

    g = torch.Generator(device=dev).manual_seed(seed)
    y = torch.empty(hi - lo, dtype=torch.float32, device=dev)
    chunk = 1 << 26
    for a in range(lo, hi, chunk):
        b = min(hi, a + chunk)
        i = torch.arange(a, b, device=dev, dtype=torch.float64)
        v = torch.sin(2 * np.pi * i / 1e3) + torch.sin(2 * np.pi * i / 1e5) + torch.sin(2 * np.pi * i / 1e7)
        v += torch.randn(b - a, device=dev, dtype=torch.float64, generator=g)
        y[a - lo:b - lo] = v
    return torch.arange(lo, hi, dtype=torch.int64, device=dev), y


def make_inputs(name, dev, seed, batch=None):
    """Device-side generation of the workload (torch Philox streams)."""
    import torch

    n, nb, n_out, r_ps, ydt, xdt, op = WORKLOADS[name]
    batch = nb if batch is None else batch
    g = torch.Generator(device=dev).manual_seed(seed)
    ytype = torch.float32 if ydt == "f32" else torch.float64
    y = torch.empty((batch, n), dtype=ytype, device=dev)
    chunk = 1 << 26
    for b in range(batch):
        for lo in range(0, n, chunk):
            hi = min(n, lo + chunk)
            if name.startswith("c3"):
                i = torch.arange(lo, hi, device=dev, dtype=torch.float64)
                v = torch.sin(2 * np.pi * i / 1e3) + torch.sin(2 * np.pi * i / 1e5) + torch.sin(2 * np.pi * i / 1e7)
                v += torch.randn(hi - lo, device=dev, dtype=torch.float64, generator=g)
                y[b, lo:hi] = v
            else:  # random walks (+ spikes for c2/c5)
                v = torch.randn(hi - lo, device=dev, dtype=torch.float64, generator=g)
                y[b, lo:hi] = v
        if not name.startswith("c3"):
            w = torch.cumsum(y[b].to(torch.float64), 0)
            if name in ("c2", "c5"):
                frac = 0.001 if name == "c2" else 0.01
                sig = 0.5 if name == "c2" else 1.0
                spike = torch.rand(n, device=dev, generator=g) < frac
                sign = torch.where(torch.rand(n, device=dev, generator=g) < 0.5, -1.0, 1.0).to(torch.float64)
                w += torch.where(spike, sign * 50.0 * sig, torch.zeros((), dtype=torch.float64, device=dev))
            y[b] = w.to(ytype)
    if xdt == "i64":
        x = torch.arange(n, dtype=torch.int64, device=dev)
    else:
        x = torch.cumsum(torch.empty(n, dtype=torch.float64, device=dev).exponential_(1.0, generator=g), 0)
    return x, (y[0] if batch == 1 else y)


# ------------------------------------------------------------- CPU legs -----
# The reference arm times at most this many points of the workload per step
# (the full c3_1e9 series fits; N-GPU weak-scaled series and C5 use a prefix).
REF_MAX_POINTS = 1_000_000_000


def base_config(name, n, batch, n_out, r_ps, op, ydt, xdt):
    """The `config` dict shared verbatim by both arms (what was timed)."""
    return {"workload": name, "n": n, "batch": batch, "n_out": n_out, "minmax_ratio": r_ps, "op": op,
            "y_dtype": ydt, "x_dtype": xdt}


def reference_measure(name, n, batch, n_out, r_ps, op, steps, warmup):
    from oracle import refbench

    per_series = batch > 1  # C4: per-series calls, as the reference would loop
    r = refbench.time_reference(name, n, n_out, r_ps, op, steps, warmup, seq_steps=3,
                                max_points=REF_MAX_POINTS)
    if per_series:
        r["sample"] += f"; C4 = {batch} independent series: one series' call timed, points/s per series"
    return r


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    name = args.workload
    n, batch, n_out, r_ps, ydt, xdt, op = WORKLOADS[name]
    gpus = int(os.environ.get("WORLD_SIZE", args.gpus))
    if name == "c3_1e9" and gpus > 1:
        n = n * gpus  # our arm's weak-scaled series; the CPU times a 1e9-point prefix of it
    r = reference_measure(name, n, batch, n_out, r_ps, op, args.steps, args.warmup)
    value = r["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (numpy PCG64, BASELINE.json recipe; f64 TimeSeries as the reference holds it)",
        "config": base_config(name, n, batch, n_out, r_ps, op, ydt, xdt),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["par_cores"], "kind": r["kind"],
                         "sample": r["sample"], "sequential": r.get("sequential"),
                         "threading_layer": r.get("threading_layer"), "points_per_step": r["points"],
                         "timeseries_build_s": r.get("timeseries_build_s")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_subprocess(name, steps=5, timeout=900):
    """cpu_baseline = the reference arm's own measurement (same code, fresh
    interpreter so NUMBA/OMP thread settings apply), median of `steps`."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", name, "--steps", str(steps),
           "--warmup", "1", "--gpus", "1"]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "OMP_NUM_THREADS")}
    try:
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=str(ROOT))
    except subprocess.TimeoutExpired:
        return {"value": None, "unit": UNIT, "cores": None, "kind": None, "sample": "timed out"}
    for line in p.stdout.splitlines()[::-1]:
        if line.startswith("{"):
            d = json.loads(line)
            cb = d["cpu_baseline"]
            cb["config"] = d["config"]
            return cb
    return {"value": None, "unit": UNIT, "cores": None, "kind": None, "sample": "failed: " + p.stderr[-500:]}


# ------------------------------------------------------------- GPU leg ------
def _pinned_copy(t):
    """Device tensor -> pinned host copy, without a pageable intermediate (8 ranks x 12 GB of
    inputs must fit the host's memory once, not twice)."""
    import torch

    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    torch.cuda.synchronize()
    return h


def _e2e(step, x, y, e2e_steps, n_out, r_ps, batch, op, ws, dist):
    """Public API with pinned HOST buffers: H2D of y (+ zero-copy x gather)
    and the D2H of the indices are inside every timed step."""
    import torch

    yh, xh = _pinned_copy(y), _pinned_copy(x)
    res = step(xh, yh)  # warm the host path once
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_e2e = []
    for _ in range(e2e_steps):
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        res = step(xh, yh)
        f1.record()
        torch.cuda.synchronize()
        t_e2e.append(f0.elapsed_time(f1))
    h2d = yh.numel() * yh.element_size()
    h2d += (2 + (n_out - 2) * r_ps) * batch * 8 if op != "lttb" else xh.numel() * xh.element_size()
    d2h = res.numel() * res.element_size()
    return statistics.mean(t_e2e), h2d, d2h


def _e2e_sharded(x, y, e2e_steps, n, n_out, r_ps, ws, dist, dev):
    """Sharded single series through the public API with this rank's shard in
    pinned HOST memory: H2D of the shard's y, x gathered in place (zero-copy)
    at the preselected positions, D2H of the n_out indices, every step."""
    import torch

    from paper_2305_00332_b200 import sharding

    yh, xh = _pinned_copy(y), _pinned_copy(x)

    def host_step():
        yd = yh.to(dev, non_blocking=True)
        return sharding.minmaxlttb_series_sharded(xh, yd, n, n_out, r_ps).cpu()

    res = host_step()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_e2e = []
    for _ in range(e2e_steps):
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record()
        res = host_step()
        f1.record()
        torch.cuda.synchronize()
        t_e2e.append(f0.elapsed_time(f1))
    shard = sharding.bucket_ranges(n, n_out, r_ps, ws)[dist.get_rank() if ws > 1 else 0]
    h2d = yh.numel() * yh.element_size() + (2 + 2 * (shard.b1 - shard.b0)) * xh.element_size()
    return statistics.mean(t_e2e), h2d, res.numel() * res.element_size()


def _parity_rows(B):
    """Rows the warm-up parity check compares: 0, B-1 and >= 64 spread rows."""
    if B <= 66:
        return list(range(B))
    return sorted(set([0, B - 1] + [int(v) for v in np.linspace(0, B - 1, 64).round()]))


def _check_parity(out, x, y, n_out, r_ps, op, sharded, shard, n, dist, ws):
    """Index-exact check of the warm-up output against the CPU oracle, on EVERY rank.

    Batch / replica rows: rows 0, B-1 and >= 64 spread rows of this rank's
    batch.  Bucket-range sharded series: each rank checks its shard's
    preselected set (the product's own shard_preselect) against the oracle's
    shard preselection, then rank 0 checks the final LTTB over the gathered
    sets against the oracle's lttb on them.  Returns (ok, description)."""
    from oracle import oracle as O

    if sharded:
        from paper_2305_00332_b200 import sharding as S

        idx, xs, ys, cnt = S.shard_preselect(x, y, n, n_out, r_ps, shard)
        c = int(cnt.item())
        got = idx[:c].cpu().numpy()
        yh = y.cpu().numpy()
        want = O.shard_preselect_typed(yh, shard.lo, n, n_out, r_ps, shard.b0, shard.b1, shard.emit_first,
                                       shard.emit_last)
        del yh
        ok = bool(np.array_equal(got, want))
        mine = (got, xs[:c].cpu().numpy(), ys[:c].cpu().numpy())
        parts = [None] * ws
        if ws > 1:
            dist.all_gather_object(parts, mine)
        else:
            parts = [mine]
        if dist is not None and ws > 1 and dist.get_rank() != 0:
            return ok, "per-rank shard preselect vs oracle"
        pi = np.concatenate([p[0] for p in parts])
        px = np.concatenate([p[1] for p in parts])
        py = np.concatenate([p[2] for p in parts])
        final = pi[O.lttb(px, py, n_out)]
        ok = ok and bool(np.array_equal(out.cpu().numpy(), final))
        return ok, "every rank's shard preselect vs oracle + final LTTB over the gathered sets vs oracle"
    xh = x.cpu().numpy()
    o = out.cpu().numpy().reshape(-1, n_out)
    rows = _parity_rows(o.shape[0])
    ok = True
    for i in rows:
        yi = (y if y.dim() == 1 else y[i]).cpu().numpy()
        want = O.lttb(xh, yi, n_out) if op == "lttb" else O.minmaxlttb_typed(xh, yi, n_out, r_ps)
        ok = ok and bool(np.array_equal(o[i], want))
    return ok, f"{len(rows)} of {o.shape[0]} rows per rank vs oracle"


def _kernel_label(trace):
    names = [t for t in trace.split(",") if t]
    if not names:
        return "none", names
    if "k_mmlttb_fused" in names:
        return "fused", names
    if any(t.startswith("k_extrema") for t in names):
        return "k1", names
    return "lttb", names


def run_ours(args):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2305_00332_b200 as mm
    from paper_2305_00332_b200 import _native as NAT

    ws, rank, local = _dist()
    torch.cuda.set_device(local)  # before the process group: NCCL binds each rank to its device
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://", device_id=dev)
    name = args.workload
    n, batch, n_out, r_ps, ydt, xdt, op = WORKLOADS[name]
    scaling = "weak"
    sharded = name == "c5s" or (name == "c3_1e9" and ws > 1)
    if name == "c3_1e9" and ws > 1:  # one N x 1e9-point series, bucket-range sharded (weak)
        n = n * ws
    batch_total = batch
    if name == "c4" and ws > 1:  # C4: 4096 series sharded across ranks (strong)
        from paper_2305_00332_b200.sharding import batch_range

        lo, hi = batch_range(batch, rank, ws)
        batch = hi - lo
        scaling = "strong"
    shard = None
    if sharded:
        from paper_2305_00332_b200 import sharding

        shard = sharding.bucket_ranges(n, n_out, r_ps, ws)[rank]
        x, y = make_shard(name, dev, 3 + rank, shard.lo, shard.hi)
        scaling = "strong" if name == "c5s" else "weak"
    else:
        x, y = make_inputs(name, dev, seed=3 + rank, batch=batch)
    L = NAT.lib()
    torch.cuda.synchronize()

    plan = None
    if args.graph and op == "minmaxlttb" and not sharded:
        plan = mm.MinMaxLTTBPlan(n, n_out, r_ps, batch=batch, y_dtype=y.dtype, x_dtype=x.dtype, device=dev)

    def step(xx, yy):
        if plan is not None and xx.is_cuda:
            return plan(xx, yy)
        if sharded:
            return sharding.minmaxlttb_series_sharded(xx, yy, n, n_out, r_ps)
        if op == "lttb":
            return mm.lttb(xx, yy, n_out)
        return mm.minmaxlttb(xx, yy, n_out, minmax_ratio=r_ps)

    # warm-up (with the launch trace on: the kernels one step launches) + parity of
    # the warm-up output against the oracle, on every rank
    L.mmlttb_trace(1)
    out = step(x, y)
    torch.cuda.synchronize()
    tbuf = ctypes.create_string_buffer(1 << 16)
    L.mmlttb_trace_read(tbuf, len(tbuf))
    L.mmlttb_trace(0)
    kind, step_kernels = _kernel_label(tbuf.value.decode())
    parity = "unchecked"
    if not args.no_check:
        ok, how = _check_parity(out, x, y, n_out, r_ps, op, sharded, shard, n, dist if ws > 1 else None, ws)
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        if ws > 1:
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        parity = ("exact vs oracle" if int(flag.item()) else "MISMATCH vs oracle") + f" ({how}; {ws} rank(s))"
    for _ in range(max(0, args.warmup - 1)):
        step(x, y)
    torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.15)
    # ---- device-resident timed region (value) ----
    # (the library's per-stage event timer adds ~10 us of stream work per call on
    # C3, so it runs in a separate pass right after this region -- below)
    rep0 = L.mmlttb_repair_scans()
    l0 = L.mmlttb_launch_count()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step(x, y)
    e1.record()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches = L.mmlttb_launch_count() - l0
    repairs = (L.mmlttb_repair_scans() - rep0) / args.steps
    ms = e0.elapsed_time(e1)

    # ---- per-stage device times: CUDA events recorded by the library on the
    # call's stream around K1 / K2 / K3, over a live pass of the same steps
    stage_steps = min(args.steps, 50)
    L.mmlttb_stage_timer(1)
    for _ in range(stage_steps):
        step(x, y)
    torch.cuda.synchronize()
    st = (ctypes.c_double * 3)()
    calls = ctypes.c_int64()
    L.mmlttb_stage_timer_read(st, ctypes.byref(calls))
    L.mmlttb_stage_timer(0)
    stage_ms = [v / max(1, calls.value) for v in st]
    # ---- end-to-end through the public API with host buffers (e2e) ----
    e2e_steps = min(args.steps, args.e2e_steps)
    if e2e_steps <= 0:  # profiling runs (ncu) skip the host path
        clocks.stop()
        e2e_ms = float("nan")
        h2d = d2h = 0
    elif sharded:  # each rank: its shard's y from pinned host memory, x read in place
        e2e_ms, h2d, d2h = _e2e_sharded(x, y, e2e_steps, n, n_out, r_ps, ws, dist, dev)
        clocks.stop()
    else:
        e2e_ms, h2d, d2h = _e2e(step, x, y, e2e_steps, n_out, r_ps, batch, op, ws, dist)
        clocks.stop()
    pts = n * batch if not sharded else n / ws  # sharded: the one series is split across ranks

    # max over ranks of the device-timed region
    t = torch.tensor([ms, e2e_ms if e2e_steps > 0 else 0.0], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(t[0]), float(t[1])
    value = pts * ws * args.steps / (ms / 1e3)
    e2e_value = pts * ws / (e2e_ms / 1e3) if e2e_steps > 0 else None
    if rank == 0:
        peak, peak_src = _peaks()
        ysz = 4 if ydt == "f32" else 8
        step_ms = ms / args.steps
        kernel_timing = (f"CUDA events recorded by the library around the kernel on its stream, "
                         f"{stage_steps} live steps right after the timed region")
        if sharded:  # whole sharded step: K1+K2 on the shard, all_gather, merge, LTTB
            alg_bytes = pts * ysz
            k_ms = step_ms
            kname = "minmaxlttb_series_sharded (whole step: K1+K2 per shard, all_gather, merge, K3)"
            kernel_timing = "whole step (device-timed region / steps)"
        elif op == "lttb":
            alg_bytes = pts * (ysz + 8)
            k_ms = min(step_ms, sum(stage_ms) or step_ms)
            kname = "full LTTB, every launch of the step (" + "+".join(step_kernels) + ")"
        elif kind == "fused" or plan is not None or stage_ms[0] <= 0:
            # one kernel per step (fused per-series kernel) or a graph replay: the
            # step IS the kernel, so the roofline uses the device-timed step
            alg_bytes = pts * ysz
            k_ms = step_ms
            kname = ("k_mmlttb_fused (K1+K2+K3 per series, one launch)" if kind == "fused"
                     else "whole minmaxlttb step (CUDA graph replay)")
            kernel_timing = "whole step (device-timed region / steps)"
        else:
            alg_bytes = pts * ysz
            k_ms = min(stage_ms[0], step_ms)
            kname = [t for t in step_kernels if t.startswith("k_extrema")][0] + " (K1)"
        achieved = alg_bytes / (k_ms / 1e3) / 1e9
        tr = _traffic()
        traffic = None
        if tr and tr.get("workload") == name:
            traffic = tr.get("dram_bytes_per_launch")
        cpu = None
        if not args.no_cpu and ws == 1:
            cpu = cpu_baseline_subprocess(name, steps=args.cpu_steps)
        split = kind == "k1" and plan is None and stage_ms[2] > 0
        k23 = "k_k23" in step_kernels
        lstage = stage_ms[1] + stage_ms[2] if k23 else stage_ms[2]
        lk = "k_k23 (K2 + K3 in one launch)" if k23 else "K3 tables + scan"
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": step_ms,
            "higher_is_better": True,
            "scaling": scaling,
            "vs_baseline": None,
            "dtype": ydt,
            "data": "synthetic (device-generated, torch Philox; BASELINE.json recipe shapes)",
            "config": base_config(name, n, batch_total, n_out, r_ps, op, ydt, xdt),
            "details": {"parity": parity,
                        "sharding": ("bucket-range shards of one series + NCCL all_gather" if sharded
                                     else "batch rows per rank" if name == "c4" and ws > 1 else
                                     "independent replica per rank" if ws > 1 else "none"),
                        "graph": bool(plan is not None), "rows_this_rank": batch,
                        "l2": ("inputs larger than L2 (no flush needed)"
                               if pts * (4 if ydt == "f32" else 8) > 126e6
                               else "inputs smaller than L2: steady-state L2-resident repeat calls"),
                        "kernels_per_step": step_kernels},
            "hbm_gbs": alg_bytes * args.steps / (ms / 1e3) / 1e9,
            "pct_roofline_e2e_device": alg_bytes * args.steps / (ms / 1e3) / 1e9 / peak,
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel_ms": k_ms, "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel_timing": kernel_timing},
            "stage_ms": ({"k1_extrema": stage_ms[0], "k2_compact": stage_ms[1], "k3_lttb": stage_ms[2]}
                         if split else None),
            # LTTB stage latency per output bucket (the sequential chain the tables +
            # scan resolve), only where the stages are separate launches; with K23
            # (compaction + LTTB in one launch) the stage is K2+K3 together
            "lttb_stage": ({"ms": lstage, "buckets": (n_out - 2) * batch, "kernels": lk,
                            "ns_per_bucket": lstage * 1e6 / max(1, (n_out - 2) * batch)} if split else
                           {"ms": k_ms, "buckets": (n_out - 2) * batch,
                            "ns_per_bucket": k_ms * 1e6 / max(1, (n_out - 2) * batch)} if op == "lttb" else None),
            "cpu_baseline": cpu,
            "e2e": None if e2e_value is None else {
                "value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_ms, "steps": e2e_steps,
                "path": ("minmaxlttb_series_sharded(pinned host x shard read in place, y shard H2D) -> CPU "
                         "indices, per rank" if sharded else
                         "minmaxlttb(pinned host x, pinned host y) -> numpy-free CPU tensor result")},
            "gpu_launches": int(launches),
            "lttb_repair_scans_per_step": repairs,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def relaunch_torchrun(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}; refusing to run "
              "(no silent single-GPU fallback)", file=sys.stderr)
        return 2
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c3_1e9", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--cpu-steps", type=int, default=5, help="timed reference runs for cpu_baseline (median)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--graph", action="store_true", help="device loop through MinMaxLTTBPlan (CUDA graph replay)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        return relaunch_torchrun(args)
    if ws_env is not None and int(ws_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} disagrees with WORLD_SIZE={ws_env}; refusing to run", file=sys.stderr)
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
