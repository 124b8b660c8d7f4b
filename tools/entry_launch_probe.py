#!/usr/bin/env python
"""One call of every public entry point on 1e8 float32 points (for an ncu launch list)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_00332_b200 as mm  # noqa: E402

n = 100_000_000
x = torch.arange(n, device="cuda")
y = torch.randn(n, device="cuda")
for _ in range(2):
    mm.minmax(x, y, 4000)
    mm.m4(x, y, 4000)
    mm.minmax_preselect(x, y, 2000, 4)
    mm.minmaxlttb(x, y, 2000, minmax_ratio=4, validate=True)
    mm.every_nth(x, y, 2000)
    mm.minmaxlttb(x, y, 4000, minmax_ratio=1)
torch.cuda.synchronize()
print("ok")
