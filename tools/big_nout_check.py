import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2305_00332_b200 as mm
from oracle import oracle as O
rng = np.random.Generator(np.random.PCG64(3))
for n, k in [(5_000_000, 20_000), (3_000_000, 16_500), (3_000_000, 16_386), (2_000_000, 9_000)]:
    x = np.arange(n, dtype=np.int64); y = np.cumsum(rng.standard_normal(n))
    got = mm.lttb(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), k).cpu().numpy()
    print(n, k, 'OK' if np.array_equal(got, O.lttb(x, y, k)) else 'MISMATCH')
