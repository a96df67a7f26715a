"""Qwen3 MLP block of TN layers: y = down(silu(gate(x)) * up(x)).

``TNMLP(gate, up, down).forward(x)`` runs ``tnl_mlp_forward``: for prefill-sized M and
merged-cut plans the SiLU*mul intermediate (M x 25600 for Qwen3-32B) stays on chip
(one fused kernel between the gate/up input GEMM and the down output GEMM); otherwise
the three layers run unfused around a SiLU*mul kernel.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as N
from .errors import DeviceError, ShapeError
from .layer import CompressedLayer


class TNMLP:
    def __init__(self, gate: CompressedLayer, up: CompressedLayer, down: CompressedLayer, dtype=torch.bfloat16,
                 device=None, fused: bool = True):
        self.lib = N.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dtype = dtype
        self.plans = [l.plan(dtype, self.device) for l in (gate, up, down)]
        self.hidden = self.plans[0].info["cols"]
        h = ctypes.c_void_p()
        N.check(self.lib.tnl_mlp_create(self.plans[0].handle, self.plans[1].handle, self.plans[2].handle,
                                        0 if fused else 1, ctypes.byref(h)))
        self.handle = h
        self.fused = bool(self.lib.tnl_mlp_is_fused(h))
        self._ws = None

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.tnl_mlp_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def workspace_bytes(self, m: int) -> int:
        n = ctypes.c_size_t()
        N.check(self.lib.tnl_mlp_workspace_size(self.handle, int(m), ctypes.byref(n)))
        return int(n.value)

    def workspace(self, m: int):
        n = self.workspace_bytes(m)
        if self._ws is None or self._ws.numel() < n:
            self._ws = torch.zeros(max(n, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None, ws: torch.Tensor | None = None) -> torch.Tensor:
        if not isinstance(x, torch.Tensor) or not x.is_cuda:
            raise DeviceError("forward needs a CUDA tensor (no CPU fallback)")
        if x.dim() != 2 or x.shape[1] != self.hidden:
            raise ShapeError(f"x inner dimension {tuple(x.shape)} does not match {self.hidden}")
        m = x.shape[0]
        if x.stride(1) != 1 or (m > 1 and x.stride(0) < self.hidden):
            x = x.contiguous()
        if out is None:
            out = torch.empty((m, self.hidden), dtype=self.dtype, device=self.device)
        if ws is None:
            ws = self.workspace(m)
        elif ws.numel() < self.workspace_bytes(m):
            raise ShapeError(f"MLP workspace {ws.numel()} < {self.workspace_bytes(m)} bytes")
        stream = torch.cuda.current_stream(self.device).cuda_stream
        N.check(self.lib.tnl_mlp_forward(self.handle, ctypes.c_void_p(x.data_ptr()), m,
                                         x.stride(0) if m > 1 else self.hidden, ctypes.c_void_p(out.data_ptr()),
                                         out.stride(0) if m > 1 else self.hidden, ctypes.c_void_p(ws.data_ptr()),
                                         ws.numel(), ctypes.c_void_p(stream)))
        return out

    __call__ = forward
