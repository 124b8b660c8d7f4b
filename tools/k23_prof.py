"""Phase timeline of the K23 kernel (minmaxlttb tail) on C1 / C3 shapes.
MMLTTB_K3S_PROF=1 python tools/k23_prof.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2305_00332_b200 as mm  # noqa: E402

DEV = torch.device("cuda", 0)
L = mm._native.lib()
L.mmlttb_debug_k3s_prof.restype = ctypes.c_int64
for name, n, n_out, r, dt in [("c1", 1_000_000, 1000, 4, torch.float64), ("c3", 100_000_000, 2000, 4, torch.float32),
                              ("c3r32", 100_000_000, 2000, 32, torch.float32)]:
    x = torch.arange(n, dtype=torch.int64, device=DEV)
    y = torch.randn(n, dtype=dt, device=DEV).cumsum(0)
    for _ in range(5):
        mm.minmaxlttb(x, y, n_out, minmax_ratio=r)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (1024 * 8 + 64))()
    L.mmlttb_debug_k3s_prof(buf, ctypes.c_int64(1024 * 8 + 64))
    a = np.array(buf, dtype=np.float64)[:1024 * 8].reshape(1024, 8)
    a = a[a[:, 0] > 0]
    t0 = a[:, 0].min()
    print(f"{name}: {a.shape[0]} CTAs, start spread {(a[:, 0].max() - t0) / 1e3:.2f} us")
    for i, nm in enumerate(["A done", "sync0", "B done", "sync1", "C done"], 1):
        col = a[:, i]
        print(f"   {nm:7s} min {(col.min() - t0) / 1e3:6.2f}  mean {(col.mean() - t0) / 1e3:6.2f}  max {(col.max() - t0) / 1e3:6.2f} us")
