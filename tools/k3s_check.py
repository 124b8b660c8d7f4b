"""Parity + timing of the full-LTTB large-bucket path (K3s single launch, or
the K3c kernels with MMLTTB_K3S=0) on C2-like shapes vs the CPU oracle.
Usage: python tools/k3s_check.py [--time]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2305_00332_b200 as mm  # noqa: E402
from oracle import oracle as O  # noqa: E402

DEV = torch.device("cuda", 0)


def c2_y(n, seed, dt=np.float64):
    rng = np.random.Generator(np.random.PCG64(seed))
    y = np.cumsum(rng.standard_normal(n)) + rng.normal(0, 0.5, n)
    sp = rng.random(n) < 0.001
    y[sp] += 50 * 0.5 * rng.choice([-1.0, 1.0], sp.sum())
    return y.astype(dt)


CASES = [
    # name, n, n_out, x kind, y dtype
    ("c2", 10_000_000, 2000, "i64", np.float64),
    ("c2_f32y", 10_000_000, 2000, "i64", np.float32),
    ("mid", 3_000_017, 701, "i64", np.float64),
    ("i32x", 2_000_000, 900, "i32", np.float64),
    ("f64x_irregular", 2_000_000, 600, "f64irr", np.float64),
    ("f64x_arange", 2_000_000, 600, "f64", np.float32),
    ("few_buckets", 500_000, 120, "i64", np.float64),
    ("ties", 1_000_000, 400, "i64tie", np.float64),
    # group pruning: 2^s warp-loads per group (s > 0), other data shapes
    ("big_buckets", 20_000_000, 1190, "i64", np.float64, "walk"),
    ("big_buckets_f32", 40_000_000, 1200, "i64", np.float32, "walk"),
    ("huge_buckets", 60_000_000, 1186, "i32", np.float32, "c2"),
    ("smooth", 6_000_000, 1500, "i64", np.float64, "sin"),
    ("const", 4_000_000, 1300, "i64", np.float64, "const"),
    ("steps", 6_000_000, 1400, "f64", np.float64, "steps"),
    ("neg_dx", 5_000_000, 1250, "f64neg", np.float64, "walk"),
    # few, wide buckets (K3s below 8 buckets per SM: one warp streams a whole bucket)
    ("wide_300", 10_000_000, 300, "i64", np.float64, "walk"),
    ("wide_1000", 10_000_000, 1000, "i64", np.float64, "walk"),
    ("wide_100", 10_000_000, 100, "i64", np.float32, "walk"),
    ("wide_30", 3_000_000, 30, "i64", np.float64, "walk"),
    ("tiny_k3", 200_000, 4, "i64", np.float64, "walk"),
    # many narrow buckets (several buckets per warp and phase)
    ("many_100pt", 1_000_000, 10_000, "i64", np.float64, "walk"),
    ("many_500pt", 4_000_000, 8_000, "i64", np.float64, "walk"),
    ("many_1500pt", 6_000_000, 4_000, "i64", np.float32, "walk"),
]


def make_y(kind, n, ydt):
    rng = np.random.Generator(np.random.PCG64(11))
    if kind == "c2":
        return c2_y(n, 2, ydt)
    if kind == "walk":
        return np.cumsum(rng.standard_normal(n)).astype(ydt)
    if kind == "sin":
        i = np.arange(n, dtype=np.float64)
        return (np.sin(i / 3000.0) * 100 + np.sin(i / 17.0)).astype(ydt)
    if kind == "const":
        return np.full(n, 3.25, dtype=ydt)
    if kind == "steps":  # long flat runs: whole groups tie
        return np.repeat(rng.integers(-5, 5, n // 1000 + 1), 1000)[:n].astype(ydt)
    raise ValueError(kind)


def make_x(kind, n, seed):
    if kind == "i64":
        return np.arange(n, dtype=np.int64)
    if kind == "i32":
        return np.arange(n, dtype=np.int32)
    if kind == "f64":
        return np.arange(n, dtype=np.float64)
    if kind == "f64irr":
        return np.cumsum(np.random.Generator(np.random.PCG64(seed)).exponential(1.0, n))
    if kind == "i64tie":
        return np.arange(n, dtype=np.int64)
    if kind == "f64neg":
        return -0.25 * np.arange(n, dtype=np.float64)[::-1].copy() - 7.0
    raise ValueError(kind)


def main():
    timing = "--time" in sys.argv
    only = [a for a in sys.argv[1:] if not a.startswith("--")]
    ok_all = True
    for name, n, n_out, xk, ydt, *yk in CASES:
        if only and name not in only:
            continue
        x = make_x(xk, n, 7)
        y = make_y(yk[0] if yk else "c2", n, ydt)
        if xk == "i64tie":  # duplicated values: exact area ties everywhere
            y = np.repeat(y[: n // 2], 2)[:n].copy()
        want = O.lttb(x, y.astype(np.float64), n_out)
        xd, yd = torch.from_numpy(x).to(DEV), torch.from_numpy(y).to(DEV)
        got = mm.lttb(xd, yd, n_out)
        torch.cuda.synchronize()
        ok = np.array_equal(got.cpu().numpy(), want)
        ok_all &= ok
        line = f"{name}: n={n} n_out={n_out} x={xk} y={np.dtype(ydt).name} {'OK' if ok else 'MISMATCH'}"
        if not ok:
            g = got.cpu().numpy()
            d = np.nonzero(g != want)[0]
            line += f" ({d.size} differ, first at {d[:5].tolist()})"
        if timing:
            for _ in range(3):
                mm.lttb(xd, yd, n_out)
            torch.cuda.synchronize()
            st = torch.cuda.Event(enable_timing=True)
            en = torch.cuda.Event(enable_timing=True)
            st.record()
            R = 20
            for _ in range(R):
                mm.lttb(xd, yd, n_out)
            en.record()
            torch.cuda.synchronize()
            line += f"  {st.elapsed_time(en) / R * 1000:.1f} us/call"
        print(line, flush=True)
        if "--prof" in sys.argv and os.environ.get("MMLTTB_K3S_PROF") == "1":
            import ctypes
            L = mm._native.lib()
            buf = (ctypes.c_ulonglong * (1024 * 8 + 64))()
            L.mmlttb_debug_k3s_prof.restype = ctypes.c_int64
            if L.mmlttb_debug_k3s_prof(buf, ctypes.c_int64(1024 * 8 + 64)) > 0:
                allv = np.array(buf, dtype=np.float64)
                cn = allv[1024 * 8:1024 * 8 + 8].astype(np.int64)
                print("   counters: verify calls %d, violations %d, shared-hi %d, cert fails %d, full picks %d, flagged %d, 4b picks %d, repair picks %d" % tuple(cn))
                pc = allv[1024 * 8 + 8:1024 * 8 + 16].astype(np.int64)
                print("   pruning: cand pruned %d (groups %d), cand plain %d; verify pruned %d (groups %d), verify plain %d; 4j re-verified %d in %d passes" % tuple(pc))
                tl = allv[1024 * 8 + 32:1024 * 8 + 64]
                if tl.max() > 0:
                    t00 = allv[70 * 8]
                    print("   CTA 70 warp 0 timeline (us):", " ".join(f"{i}:{(v - t00) / 1e3:.1f}" for i, v in enumerate(tl) if v > 0))
                dv = allv[1024 * 8 + 16:1024 * 8 + 32].reshape(4, 4)
                for st in dv:
                    if st[0] > 0:
                        print("   4b pick: guess %.2f us, pick %.2f us, guess right %d" % ((st[1] - st[0]) / 1e3, (st[2] - st[1]) / 1e3, st[3]))
                a = allv[:1024 * 8].reshape(1024, 8)
                a = a[a[:, 0] > 0]
                t0 = a[:, 0].min()
                if "--ctas" in sys.argv:  # per-CTA statistics-done times: buckets per CTA vs finish time
                    G = a.shape[0]
                    k3 = n_out - 2
                    nbk = np.array([(c + 1) * k3 // G - c * k3 // G for c in range(G)])
                    sd = (a[:, 1] - t0) / 1e3
                    order = np.argsort(sd)
                    print("   stats done by buckets/CTA:", {int(k): (round(float(sd[nbk == k].mean()), 1), round(float(sd[nbk == k].max()), 1)) for k in np.unique(nbk)})
                    print("   slowest CTAs (id, buckets, us):", [(int(c), int(nbk[c]), round(float(sd[c]), 1)) for c in order[-12:]])
                    print("   fastest CTAs (id, buckets, us):", [(int(c), int(nbk[c]), round(float(sd[c]), 1)) for c in order[:6]])
                    print("   start skew (us): max", round(float((a[:, 0].max() - t0) / 1e3), 2))
                names = ["start", "stats", "cand", "tab+agg", "chain", "verify", "verify2+", "repair"]
                for i in range(1, 8):
                    col = a[:, i]
                    col = col[col > 0]
                    if col.size:
                        print(f"   {names[i]:7s} done at us: min {(col.min()-t0)/1e3:7.1f}  mean {(col.mean()-t0)/1e3:7.1f}  max {(col.max()-t0)/1e3:7.1f}")
    print("ALL OK" if ok_all else "SOME MISMATCH")
    return 0 if ok_all else 1


if __name__ == "__main__":
    sys.exit(main())
