"""Randomised parity sweep of the full-LTTB paths (K3s with pruned phases / fixed-point passes,
K3c, K3a) against the CPU oracle: random sizes, bucket widths, x kinds and y shapes.
python tools/lttb_fuzz.py [cases] [seed]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_00332_b200 as mm  # noqa: E402
from oracle import oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.Generator(np.random.PCG64(seed))
dev = torch.device("cuda", 0)
bad = 0
for it in range(cases):
    n = int(rng.integers(20_000, 4_000_000))
    width = float(np.exp(rng.uniform(np.log(8), np.log(30_000))))  # points per bucket
    n_out = int(min(max(3, n / width), n - 1))
    xk = rng.choice(["i64", "i64irr", "i32", "f64", "f64irr", "f32", "f64neg"])
    yk = rng.choice(["walk", "spikes", "sin", "steps", "const", "ramp", "noise", "dup"])
    ydt = rng.choice([np.float32, np.float64])
    if xk == "i64":
        x = np.arange(n, dtype=np.int64) * int(rng.integers(1, 1000)) - int(rng.integers(0, 10**9))
    elif xk == "i64irr":
        x = np.cumsum(rng.integers(0, 5, n)).astype(np.int64)
    elif xk == "i32":
        x = np.arange(n, dtype=np.int32)
    elif xk == "f64":
        x = np.arange(n, dtype=np.float64) * 0.125 + 3.0
    elif xk == "f64irr":
        x = np.cumsum(rng.exponential(1.0, n))
    elif xk == "f32":
        x = np.arange(n, dtype=np.float32)[: min(n, 1 << 24)]
        n = x.shape[0]
        n_out = min(n_out, n - 1)
    else:
        x = -0.5 * np.arange(n, dtype=np.float64)[::-1].copy() - 1.0
    i = np.arange(n, dtype=np.float64)
    if yk == "walk":
        y = np.cumsum(rng.standard_normal(n))
    elif yk == "spikes":
        y = np.cumsum(rng.standard_normal(n)) + np.where(rng.random(n) < 0.001, rng.choice([-25.0, 25.0], n), 0.0)
    elif yk == "sin":
        y = np.sin(i / rng.uniform(50, 5000)) * 100 + np.sin(i / 17.0)
    elif yk == "steps":
        y = np.repeat(rng.integers(-5, 5, n // 500 + 1), 500)[:n].astype(np.float64)
    elif yk == "const":
        y = np.full(n, -2.5)
    elif yk == "ramp":
        y = 0.25 * i - 1e5
    elif yk == "noise":
        y = rng.standard_normal(n) * 1e-3 + 1e6
    else:
        y = np.repeat(np.cumsum(rng.standard_normal(n // 2 + 1)), 2)[:n].copy()
    y = y.astype(ydt)
    only = os.environ.get("LTTB_FUZZ_ONLY")
    if only is not None and it != int(only):
        continue
    if only is not None and os.environ.get("LTTB_FUZZ_SAVE"):
        np.savez(os.environ["LTTB_FUZZ_SAVE"], x=x, y=y, n_out=n_out)
    want = O.lttb(x, y.astype(np.float64), n_out)
    got = mm.lttb(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev), n_out).cpu().numpy()
    ok = np.array_equal(got, want)
    if not ok:
        bad += 1
        d = np.nonzero(got != want)[0]
        print(f"MISMATCH case {it}: n={n} n_out={n_out} x={xk} y={yk}/{np.dtype(ydt).name}: {d.size} differ, first {d[:4].tolist()}", flush=True)
    elif it % 20 == 0:
        print(f"case {it}: n={n} n_out={n_out} x={xk} y={yk}/{np.dtype(ydt).name} ok", flush=True)
print(f"{cases} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
