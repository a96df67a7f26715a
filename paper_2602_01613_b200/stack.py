"""A chain of TN layers (a decoder's projection stack) with CUDA-graph replay.

``TNStack(layers).forward(x)`` applies the layers in order (eager, one C-ABI
call per layer). ``capture(m)`` records one whole pass — optionally including
the host->device copy of x and the device->host copy of y from pinned
buffers — into a CUDA graph so small-M decode is not bound by host launch
overhead. All plans share one workspace (the steps of a stack are
stream-ordered, so reuse is safe).
"""

from __future__ import annotations

import torch

from . import _native as N
from .errors import ShapeError
from .layer import CompressedLayer


class TNStack:
    def __init__(self, layers: list[CompressedLayer], dtype=torch.bfloat16, device=None,
                 flags: int = N.PLAN_AUTO):
        if not layers:
            raise ShapeError("empty stack")
        self.layers = layers
        self.dtype = dtype
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.plans = [l.plan(dtype, self.device, flags) for l in layers]
        for a, b in zip(self.plans, self.plans[1:]):
            if a.rows_local != b.info["cols"]:
                raise ShapeError(f"stack link mismatch: {a.rows_local} outputs feed {b.info['cols']} inputs")
        self.cols = self.plans[0].info["cols"]
        self.rows = self.plans[-1].rows_local
        self._ws = None
        self.graph = None

    def workspace(self, m: int):
        need = max(p.workspace_bytes(m) for p in self.plans)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def forward(self, x, bufs=None):
        m = x.shape[0]
        ws = self.workspace(m)
        width = max(p.rows_local for p in self.plans)
        if bufs is None:
            bufs = [torch.empty((m, width), dtype=self.dtype, device=self.device) for _ in range(2)]
        cur = x
        for i, p in enumerate(self.plans):
            out = bufs[i % 2][:, : p.rows_local]
            p.forward(cur, out=out, ws=ws)
            cur = out
        return cur

    def capture(self, m: int, host_io: bool = True, warmup: int = 1):
        """Record one pass for M = m tokens into a CUDA graph (static buffers)."""
        self.m = m
        self.x_dev = torch.zeros((m, self.cols), dtype=self.dtype, device=self.device)
        width = max(p.rows_local for p in self.plans)
        self.bufs = [torch.empty((m, width), dtype=self.dtype, device=self.device) for _ in range(2)]
        self.workspace(m)
        self.host_io = host_io
        if host_io:
            self.x_host = torch.zeros((m, self.cols), dtype=self.dtype).pin_memory()
            self.y_host = torch.empty((m, self.rows), dtype=self.dtype).pin_memory()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for _ in range(warmup):  # plans build tensor maps / lazy state outside capture
                self.y_dev = self.forward(self.x_dev, self.bufs)
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        N.launch_count(reset=True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            if host_io:
                self.x_dev.copy_(self.x_host, non_blocking=True)
            self.y_dev = self.forward(self.x_dev, self.bufs)
            if host_io:
                self.y_host.copy_(self.y_dev, non_blocking=True)
        self.launches_per_pass = N.launch_count(reset=True)
        self.graph = g
        self.h2d_bytes = self.x_dev.numel() * self.x_dev.element_size() if host_io else 0
        self.d2h_bytes = self.y_dev.numel() * self.y_dev.element_size() if host_io else 0
        return g

    def replay(self):
        self.graph.replay()
