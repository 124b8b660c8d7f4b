"""Attainable HBM read bandwidth on this B200 with library reductions (context for K1's roofline)."""
import torch

n = 1_000_000_000
y = torch.randn(n, device="cuda", dtype=torch.float32)
for name, fn in (("sum", lambda: y.sum()), ("amax", lambda: y.amax()), ("aminmax", lambda: torch.aminmax(y))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    print(f"torch.{name}: {ms:.3f} ms -> {4e9 / ms / 1e6:.0f} GB/s")
