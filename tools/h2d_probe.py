#!/usr/bin/env python
"""Host->device copy bandwidth from pinned memory: one copy vs. chunks on several streams."""
import time

import torch


def run(n_bytes=4 << 30, reps=5):
    h = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(n_bytes, dtype=torch.uint8, device="cuda")
    for streams in (1, 2, 4):
        ss = [torch.cuda.Stream() for _ in range(streams)]
        for chunk in (n_bytes // streams, 64 << 20, 16 << 20):
            best = 0.0
            for _ in range(reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for i, off in enumerate(range(0, n_bytes, chunk)):
                    with torch.cuda.stream(ss[i % streams]):
                        d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
                torch.cuda.synchronize()
                best = max(best, n_bytes / (time.perf_counter() - t0) / 1e9)
            print(f"streams={streams} chunk={chunk >> 20} MiB: {best:.1f} GB/s", flush=True)


if __name__ == "__main__":
    run()
