#!/usr/bin/env python
"""Per-call cost of the public API on C1/C3-sized inputs: device time per call with
and without the library's stage timer, and the host time to issue one call."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_00332_b200 as mm  # noqa: E402
from paper_2305_00332_b200 import _native as NAT  # noqa: E402


def run(n, n_out, r, dtype, calls=300):
    x = torch.arange(n, device="cuda")
    y = torch.randn(n, device="cuda", dtype=dtype)
    for _ in range(10):
        mm.minmaxlttb(x, y, n_out, minmax_ratio=r)
    torch.cuda.synchronize()
    for timer in (0, 1):
        NAT.lib().mmlttb_stage_timer(timer)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        for _ in range(calls):
            mm.minmaxlttb(x, y, n_out, minmax_ratio=r)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        print(f"n={n:.0e} timer={timer}: device {e0.elapsed_time(e1) * 1e3 / calls:.1f} us/call, "
              f"host issue {(t1 - t0) * 1e6 / calls:.1f} us/call", flush=True)
    NAT.lib().mmlttb_stage_timer(0)


if __name__ == "__main__":
    run(1_000_000, 1000, 4, torch.float64)
    run(100_000_000, 2000, 4, torch.float32)
