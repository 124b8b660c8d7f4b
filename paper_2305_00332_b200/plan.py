"""Pre-planned, graph-captured minmaxlttb for repeated calls of one shape.

Small series (BASELINE C1: 1e6 points, a 1.2 us roofline) are bound by the
per-call host work (argument checks, allocations, 4-6 launches), not by the
device.  A plan does the reference's O(1) checks and the allocations once,
and records the stream-ordered launch sequence of ``mmlttb_minmaxlttb`` into
a CUDA graph per (x, y) buffer pair, so a call is one ``graph.replay()``.

    plan = MinMaxLTTBPlan(n=1_000_000, n_out=1000, r_ps=4, y_dtype=torch.float64)
    idx = plan(x_dev, y_dev)      # int64 [n_out] on the device (reused buffer)

The output tensor is owned by the plan and overwritten by the next call;
``.clone()`` it to keep it.  Inputs must stay alive and unchanged in place
while their graph is cached (rewriting their contents is fine).
"""
from __future__ import annotations

import torch

from . import _native as N
from .downsamplers import _check_preselect
from .errors import ValidationError

__all__ = ["MinMaxLTTBPlan"]


class MinMaxLTTBPlan:
    def __init__(self, n: int, n_out: int, r_ps: int = 4, batch: int = 1, y_dtype=torch.float32,
                 x_dtype=torch.int64, x_shared: bool = True, device=None, graph: bool = True, max_graphs: int = 8):
        _check_preselect(n, n_out, r_ps)  # reference order: NOutOfRange, BadPreselectionRatio, RatioTooLarge
        if y_dtype not in (torch.float32, torch.float64) or x_dtype not in N.DTYPE_CODE:
            raise ValidationError("unsupported dtype")
        self.device = N.require_cuda(device)
        self.n, self.n_out, self.r_ps, self.batch = n, n_out, r_ps, batch
        self.y_dtype, self.x_dtype, self.x_shared = y_dtype, x_dtype, x_shared
        self.ydt, self.xdt = N.DTYPE_CODE[y_dtype], N.DTYPE_CODE[x_dtype]
        self.x_ld = 0 if x_shared else n
        L = N.lib()
        self.wsb = L.mmlttb_workspace_bytes(N.OP_MINMAXLTTB, batch, n, n_out, r_ps, self.ydt)
        self.ws = N.workspace(self.wsb, self.device, n)
        self.out = torch.empty((batch, n_out), dtype=torch.int64, device=self.device)
        self.use_graph = graph
        self.max_graphs = max_graphs
        self._graphs: dict[tuple[int, int], torch.cuda.CUDAGraph] = {}

    def _check(self, x: torch.Tensor, y: torch.Tensor) -> None:
        want_y = (self.batch, self.n) if self.batch > 1 else None
        if y.dtype != self.y_dtype or x.dtype != self.x_dtype or not (y.is_cuda and x.is_cuda):
            raise ValidationError("inputs must be CUDA tensors of the planned dtypes")
        if (want_y and tuple(y.shape) != want_y) or (not want_y and y.shape[-1] != self.n):
            raise ValidationError(f"y must have shape {want_y or (self.n,)}")
        if x.shape[-1] != self.n or (not self.x_shared and x.dim() != 2):
            raise ValidationError("x does not match the plan")
        if not (x.is_contiguous() and y.is_contiguous()):
            raise ValidationError("inputs must be contiguous")

    def _launch(self, x: torch.Tensor, y: torch.Tensor) -> None:
        st = torch.cuda.current_stream(self.device).cuda_stream
        N.check(N.lib().mmlttb_minmaxlttb(x.data_ptr(), self.xdt, self.x_ld, y.data_ptr(), self.ydt, self.n,
                                          self.batch, self.n, self.n_out, self.r_ps, self.out.data_ptr(), None,
                                          self.ws.data_ptr(), self.wsb, st), "minmaxlttb", self.n)

    def __call__(self, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        self._check(x, y)
        if not self.use_graph:
            self._launch(x, y)
            return self.out if self.batch > 1 else self.out[0]
        key = (x.data_ptr(), y.data_ptr())
        g = self._graphs.get(key)
        if g is None:
            if len(self._graphs) >= self.max_graphs:
                self._graphs.pop(next(iter(self._graphs)))
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):
                self._launch(x, y)  # one-time kernel attributes before capture
            torch.cuda.current_stream(self.device).wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self._launch(x, y)
            self._graphs[key] = g
        g.replay()
        return self.out if self.batch > 1 else self.out[0]
