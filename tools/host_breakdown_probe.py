#!/usr/bin/env python
"""Where the host time of one small minmaxlttb call goes (C1 size)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2305_00332_b200 as mm  # noqa: E402
from paper_2305_00332_b200 import _native as N  # noqa: E402
from paper_2305_00332_b200 import downsamplers as D  # noqa: E402


def t(label, fn, reps=2000):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    dt = (time.perf_counter() - t0) / reps * 1e6
    torch.cuda.synchronize()
    print(f"{label:40s} {dt:6.2f} us", flush=True)


n, n_out, r = 1_000_000, 1000, 4
x = torch.arange(n, device="cuda")
y = torch.randn(n, device="cuda", dtype=torch.float64)
dev = y.device
b = D.Batch(x, y)
b.ready()
out = torch.empty((1, n_out), dtype=torch.int64, device=dev)
st = N.stream_ptr(dev)
wsb = N.workspace_bytes(N.OP_MINMAXLTTB, 1, n, n_out, r, N.MM_F64)
ws = N.stream_workspace(wsb, dev, st, n)
L = N.lib()
t("full minmaxlttb(x, y, ...)", lambda: mm.minmaxlttb(x, y, n_out, minmax_ratio=r))
t("Batch(x, y)", lambda: D.Batch(x, y))
t("Batch(x, y).ready()", lambda: D.Batch(x, y).ready())
t("_check_preselect", lambda: D._check_preselect(n, n_out, r))
t("torch.empty(out)", lambda: torch.empty((1, n_out), dtype=torch.int64, device=dev))
t("stream_ptr", lambda: N.stream_ptr(dev))
t("workspace_bytes (memo)", lambda: N.workspace_bytes(N.OP_MINMAXLTTB, 1, n, n_out, r, N.MM_F64))
t("stream_workspace (cached)", lambda: N.stream_workspace(wsb, dev, st, n))
t("_ctx(b)", lambda: D._ctx(b))
xp, yp, op, wp = x.data_ptr(), y.data_ptr(), out.data_ptr(), ws.data_ptr()
t("ctypes mmlttb_minmaxlttb (launches)", lambda: L.mmlttb_minmaxlttb(xp, N.MM_I64, 0, yp, N.MM_F64, n, 1, n, n_out, r,
                                                                     op, None, wp, wsb, st))
t("b.ret(out)", lambda: b.ret(out))
t("post_check", lambda: b.post_check(ws))
