"""cProfile of the Python call path of minmaxlttb (C1 shape) and lttb: where the per-call host time goes.
python tools/py_call_profile.py"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_00332_b200 as mm  # noqa: E402

dev = torch.device("cuda", 0)
n = 1_000_000
x = torch.arange(n, dtype=torch.int64, device=dev)
y = torch.from_numpy(np.cumsum(np.random.default_rng(0).standard_normal(n))).to(dev)
for _ in range(50):
    mm.minmaxlttb(x, y, 1000, 4)
torch.cuda.synchronize()
R = 20000
t0 = time.perf_counter()
for _ in range(R):
    mm.minmaxlttb(x, y, 1000, 4)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e6 * (t1 - t0) / R:.1f} us/call, with drain {1e6 * (t2 - t0) / R:.1f} us/call")
pr = cProfile.Profile()
pr.enable()
for _ in range(R):
    mm.minmaxlttb(x, y, 1000, 4)
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)
