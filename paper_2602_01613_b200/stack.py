"""A chain of TN layers (a decoder's projection stack) with CUDA-graph replay.

``TNStack(layers).forward(x)`` applies the layers in order (eager, one C-ABI
call per layer). ``capture(m)`` records one whole pass — optionally including
the host->device copy of x and the device->host copy of y from pinned
buffers — into a CUDA graph so small-M decode is not bound by host launch
overhead.

Decode through a chain is latency-bound (every layer is two dependent
weight-streaming kernels), so ``capture(m, microbatches=k)`` splits the M
tokens into k groups that run the same chain concurrently on k forked
streams inside the graph: while one group waits on a kernel boundary the
others use the SMs, and layers run roughly in lockstep so their weight
streams share L2. Per-token results are unchanged (tokens are independent
through a linear layer). Every stream has its own zero-filled workspace
(the decode split-K accumulator lives at its head).
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N
from .errors import ShapeError
from .layer import CompressedLayer, check_out


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
        self.width = max(p.rows_local for p in self.plans)
        self._ws = []
        self.graph = None
        self._lib = N.load()
        self._handles = (ctypes.c_void_p * len(self.plans))(*[p.handle.value for p in self.plans])

    def workspace_bytes(self, m: int) -> int:
        n = ctypes.c_size_t()
        N.check(self._lib.tnl_stack_workspace_size(self._handles, len(self.plans), int(m), ctypes.byref(n)))
        return int(n.value)

    def workspace(self, m: int, slot: int = 0):
        """Zero-filled stack workspace for one concurrent token group (`slot`)."""
        need = self.workspace_bytes(m)
        while len(self._ws) <= slot:
            self._ws.append(None)
        if self._ws[slot] is None or self._ws[slot].numel() < need:
            self._ws[slot] = torch.zeros(max(need, 256), dtype=torch.uint8, device=self.device)
        return self._ws[slot]

    def forward(self, x, out=None, slot: int = 0):
        """y = L_{n-1}(...L_0(x)) through ``tnl_stack_forward`` (one fused kernel per layer
        boundary for decode-sized M, else one ``tnl_forward`` per layer)."""
        m = x.shape[0]
        if x.stride(1) != 1 or (m > 1 and x.stride(0) < self.cols):
            x = x.contiguous()
        if x.dim() != 2 or x.shape[1] != self.cols or x.dtype != self.dtype:
            raise ShapeError(f"x {tuple(x.shape)} {x.dtype} does not match the stack's {self.cols} {self.dtype} inputs")
        if out is None:
            out = torch.empty((m, self.rows), dtype=self.dtype, device=self.device)
        else:
            check_out(out, m, self.rows, self.dtype, x.device)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        ldx = x.stride(0) if m > 1 else self.cols
        ldy = out.stride(0) if m > 1 else self.rows
        ws = self.workspace(m, slot)
        N.check(self._lib.tnl_stack_forward(self._handles, len(self.plans), ctypes.c_void_p(x.data_ptr()), m, ldx,
                                            ctypes.c_void_p(out.data_ptr()), ldy, ctypes.c_void_p(ws.data_ptr()),
                                            ws.numel(), ctypes.c_void_p(stream)))
        return out

    def forward_host(self, x_host, y_host, slot: int = 0):
        """Zero-copy decode step (tnl_stack_forward_host): pinned host x -> the first kernel reads
        it over the bus, the last kernel writes y straight to pinned host y."""
        m = x_host.shape[0]
        ws = self.workspace(m, slot)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        N.check(self._lib.tnl_stack_forward_host(self._handles, len(self.plans), ctypes.c_void_p(x_host.data_ptr()), m,
                                                 x_host.stride(0) if m > 1 else self.cols,
                                                 ctypes.c_void_p(y_host.data_ptr()),
                                                 y_host.stride(0) if m > 1 else self.rows,
                                                 ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(stream)))
        return y_host

    def capture(self, m: int, host_io: bool = True, warmup: int = 1, microbatches: int = 1, zero_copy: bool = False):
        """Record one pass for M = m tokens into a CUDA graph (static buffers). host_io: the pass
        starts from pinned host x and ends in pinned host y — through SM-driven copies, or with
        zero_copy=True (decode stacks) read/written directly by the first/last kernel."""
        self.m = m
        k = max(1, min(microbatches, m))
        bounds = [(i * m // k, (i + 1) * m // k) for i in range(k)]
        self.x_dev = torch.zeros((m, self.cols), dtype=self.dtype, device=self.device)
        self.y_dev = torch.zeros((m, self.rows), dtype=self.dtype, device=self.device)
        for j, (lo, hi) in enumerate(bounds):
            self.workspace(hi - lo, slot=j)
        self.host_io = host_io
        if host_io:
            self.x_host = torch.zeros((m, self.cols), dtype=self.dtype).pin_memory()
            self.y_host = torch.empty((m, self.rows), dtype=self.dtype).pin_memory()
        main = torch.cuda.Stream(self.device)
        side = [torch.cuda.Stream(self.device) for _ in range(k)]

        def copy(dst, src):  # SM-driven copy (tnl_copy_async): PDL-chained, no memcpy node
            st = torch.cuda.current_stream(self.device).cuda_stream
            N.check(self._lib.tnl_copy_async(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                             dst.numel() * dst.element_size(), ctypes.c_void_p(st)))

        def one_pass():
            # host I/O per token group on the group's own stream: each group's chain starts when
            # its rows have arrived and its D2H leaves as soon as its chain ends
            fork = torch.cuda.Event()
            fork.record(main)
            joins = []
            for j, (lo, hi) in enumerate(bounds):
                s = side[j]
                s.wait_event(fork)
                with torch.cuda.stream(s):
                    if host_io and zero_copy:
                        self.forward_host(self.x_host[lo:hi], self.y_host[lo:hi], slot=j)
                    else:
                        if host_io:
                            copy(self.x_dev[lo:hi], self.x_host[lo:hi])
                        self.forward(self.x_dev[lo:hi], out=self.y_dev[lo:hi], slot=j)
                        if host_io:
                            copy(self.y_host[lo:hi], self.y_dev[lo:hi])
                    e = torch.cuda.Event()
                    e.record(s)
                    joins.append(e)
            for e in joins:
                main.wait_event(e)

        main.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(main):
            for _ in range(warmup):  # plans build tensor maps / lazy state outside capture
                one_pass()
        torch.cuda.current_stream(self.device).wait_stream(main)
        torch.cuda.synchronize(self.device)
        N.launch_count(reset=True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=main):
            one_pass()
        self.launches_per_pass = N.launch_count(reset=True)
        self.graph = g
        self.microbatches = k
        self.h2d_bytes = self.x_dev.numel() * self.x_dev.element_size() if host_io else 0
        self.d2h_bytes = self.y_dev.numel() * self.y_dev.element_size() if host_io else 0
        return g

    def replay(self):
        self.graph.replay()


class TNGroup:
    """Plans that read the same input — a decoder's q, k and v of one normalised hidden state
    (``tnl_group_*`` in include/tnl_stack.h). Prefill runs ONE first-step GEMM over the stacked
    B_in panels (x read once, the folded RMSNorm applied there), then each layer's output step;
    decode-sized M runs the layers one after another."""

    def __init__(self, layers: list[CompressedLayer], dtype=torch.bfloat16, device=None):
        if not layers:
            raise ShapeError("empty group")
        self.lib = N.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dtype = dtype
        self.plans = [l.plan(dtype, self.device) for l in layers]
        self.cols = self.plans[0].info["cols"]
        arr = (ctypes.c_void_p * len(self.plans))(*[p.handle.value for p in self.plans])
        h = ctypes.c_void_p()
        N.check(self.lib.tnl_group_create(arr, len(self.plans), ctypes.byref(h)))
        self.handle = h
        self._ws = None

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.tnl_group_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def workspace_bytes(self, m: int) -> int:
        n = ctypes.c_size_t()
        N.check(self.lib.tnl_group_workspace_size(self.handle, int(m), ctypes.byref(n)))
        return int(n.value)

    def workspace(self, m: int):
        n = self.workspace_bytes(m)
        if self._ws is None or self._ws.numel() < n:
            self._ws = torch.zeros(max(n, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def forward(self, x: torch.Tensor, outs=None, ws=None, opts=None):
        """ys[i] = layers[i](x); opts: an ``N.FwdOpts`` (folded RMSNorm of x via ss_in)."""
        m = x.shape[0]
        if x.dim() != 2 or x.shape[1] != self.cols or x.dtype != self.dtype or not x.is_cuda:
            raise ShapeError(f"x {tuple(x.shape)} {x.dtype} does not match the group's {self.cols} {self.dtype} inputs")
        if x.stride(1) != 1:
            x = x.contiguous()
        if outs is None:
            outs = [torch.empty((m, p.rows_local), dtype=self.dtype, device=x.device) for p in self.plans]
        for o, p in zip(outs, self.plans):
            check_out(o, m, p.rows_local, self.dtype, x.device)
        ws = ws if ws is not None and ws.numel() >= self.workspace_bytes(m) else self.workspace(m)
        ys = (ctypes.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        lds = (ctypes.c_int64 * len(outs))(*[o.stride(0) if m > 1 else o.shape[1] for o in outs])
        stream = torch.cuda.current_stream(x.device).cuda_stream
        N.check(self.lib.tnl_group_forward_ex(self.handle, ctypes.c_void_p(x.data_ptr()), m,
                                              x.stride(0) if m > 1 else self.cols, ys, lds,
                                              ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                              ctypes.byref(opts) if opts is not None else None,
                                              ctypes.c_void_p(stream)))
        return outs
