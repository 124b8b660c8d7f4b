"""A/B: device-timed cost of the deferred status copy (validate=None vs False)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2305_00332_b200 as mm

dev = torch.device("cuda", 0)
for n, B, n_out in ((1_000_000_000, 1, 2000), (100_000_000, 1, 2000), (200_000, 1, 1000), (10_000_000, 64, 1000)):
    y = torch.randn(B, n, device=dev) if B > 1 else torch.randn(n, device=dev)
    x = torch.arange(n, device=dev)
    res = {}
    for rep in range(2):
        for v in (None, False):
            for _ in range(5):
                mm.minmaxlttb(x, y, n_out, minmax_ratio=4, validate=v)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 200 if n < 1e9 else 100
            e0.record()
            h0 = time.perf_counter()
            for _ in range(K):
                mm.minmaxlttb(x, y, n_out, minmax_ratio=4, validate=v)
            h1 = time.perf_counter()
            e1.record()
            torch.cuda.synchronize()
            res.setdefault(v, []).append((round(e0.elapsed_time(e1) / K * 1e3, 2), round((h1 - h0) / K * 1e6, 2)))
    mm.check_deferred()
    print(f"n={n} B={B}: (device us, host us per call) validate=None {res[None]}, validate=False {res[False]}", flush=True)
    del x, y
    torch.cuda.empty_cache()
