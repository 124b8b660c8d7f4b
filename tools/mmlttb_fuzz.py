"""Randomised parity sweep of minmaxlttb / minmax / m4 (K1 variants, K23, K2 + K3a, the fused batch
kernel) against the CPU oracle: random sizes, n_out, ratios, dtypes, tie-heavy y shapes, batches.
python tools/mmlttb_fuzz.py [cases] [seed]"""
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
    r = int(rng.choice([2, 4, 6, 8, 16, 32]))
    n_out = int(np.exp(rng.uniform(np.log(8), np.log(6000))))
    lo_n = r * n_out + 10
    n = int(np.exp(rng.uniform(np.log(lo_n), np.log(max(lo_n * 2, 8_000_000)))))
    B = int(rng.choice([1, 1, 1, 3, 160])) if n < 300_000 else 1
    ydt = rng.choice([np.float32, np.float64])
    xk = rng.choice(["i64", "f64irr", "i64irr"])
    yk = rng.choice(["walk", "steps", "const", "dup", "sin", "noise", "spikes"])
    if xk == "i64":
        x = np.arange(n, dtype=np.int64)
    elif xk == "f64irr":
        x = np.cumsum(rng.exponential(1.0, n))
    else:
        x = np.cumsum(rng.integers(0, 5, n)).astype(np.int64)
    ys = []
    for b in range(B):
        i = np.arange(n, dtype=np.float64)
        if yk == "walk":
            y = np.cumsum(rng.standard_normal(n))
        elif yk == "steps":
            y = np.repeat(rng.integers(-5, 5, n // 37 + 1), 37)[:n].astype(np.float64)
        elif yk == "const":
            y = np.full(n, 1.5)
        elif yk == "dup":
            y = np.repeat(np.cumsum(rng.standard_normal(n // 2 + 1)), 2)[:n].copy()
        elif yk == "sin":
            y = np.sin(i / rng.uniform(5, 500)) * 10
        elif yk == "noise":
            y = rng.standard_normal(n)
        else:
            y = np.cumsum(rng.standard_normal(n)) + np.where(rng.random(n) < 0.01, rng.choice([-50.0, 50.0], n), 0.0)
        ys.append(y.astype(ydt))
    Y = np.stack(ys)
    xd = torch.from_numpy(x).to(dev)
    yd = torch.from_numpy(Y if B > 1 else Y[0]).to(dev)
    got = mm.minmaxlttb(xd, yd, n_out, minmax_ratio=r).cpu().numpy().reshape(B, -1)
    ok = True
    for b in range(B if B <= 3 else 4):
        bb = b if B <= 3 else int(rng.integers(0, B))
        want = O.minmaxlttb(x, Y[bb].astype(np.float64), n_out, r)
        if not np.array_equal(got[bb], want):
            ok = False
            d = np.nonzero(got[bb] != want)[0]
            print(f"MISMATCH case {it} row {bb}: n={n} n_out={n_out} r={r} B={B} x={xk} y={yk}/{np.dtype(ydt).name}: {d.size} differ, first {d[:4].tolist()}", flush=True)
    if n_out % 4 == 0 and B == 1:
        for name in ("minmax", "m4"):
            if name == "minmax" and n_out % 2:
                continue
            try:
                g = getattr(mm, name)(xd, yd, n_out).cpu().numpy()
                w = getattr(O, name)(Y[0].astype(np.float64), n_out)
            except Exception as e:  # noqa: BLE001
                print(f"case {it} {name}: {type(e).__name__}: {e}", flush=True)
                continue
            if not np.array_equal(g, w):
                ok = False
                print(f"MISMATCH case {it} {name}: n={n} n_out={n_out} y={yk}/{np.dtype(ydt).name}", flush=True)
    bad += 0 if ok else 1
    if ok and it % 20 == 0:
        print(f"case {it}: n={n} n_out={n_out} r={r} B={B} x={xk} y={yk}/{np.dtype(ydt).name} ok", flush=True)
print(f"{cases} cases, {bad} mismatches")
sys.exit(1 if bad else 0)
