import cProfile, pstats, time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2305_00332_b200 as mm
n = 1_000_000
x = torch.arange(n, device="cuda")
y = torch.cumsum(torch.randn(n, dtype=torch.float64, device="cuda"), 0)
for _ in range(20): mm.minmaxlttb(x, y, 1000, minmax_ratio=4)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N): out = mm.minmaxlttb(x, y, 1000, minmax_ratio=4)
torch.cuda.synchronize()
print("per call us", (time.perf_counter() - t0) / N * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(N): out = mm.minmaxlttb(x, y, 1000, minmax_ratio=4)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
