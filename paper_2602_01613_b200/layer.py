"""The TN-structured linear layer — drop-in for the reference layer API.

Reference: ``CompressedLayer`` and its module functions in
/root/reference/pkg/src/minima/tn_decompositions.py (:66-126, :346-401) and the
SPEC forward contract ``apply_compressed``. Same field
names, same families (``"dense","tucker","tt","tr"``, :41-42), same validation
messages (:97-126). What changes is where the arithmetic runs: every forward,
reconstruct and panel build executes in libtnl.so on the GPU (hand-written
sm_100a kernels); nothing here computes on the CPU.

Orientation: ``forward(x)`` takes torch-style ``x (M, cols)`` and returns
``(M, rows)``; ``apply_compressed(layer, x)`` takes the reference's
``x (cols, M)`` (sensitivity.py:154-160) and returns ``(rows, M)``.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _native as N
from .errors import DeviceError, ShapeError
from .modes import DENSE, FAMILIES, chain_flops_per_token, cut_rank, param_count_formula

try:  # torch is plumbing (device memory, streams); imported lazily-safe
    import torch
except Exception:  # pragma: no cover
    torch = None


def _as_host_array(a) -> np.ndarray:
    """Contiguous host float64/float32 copy of a numpy array or torch tensor."""
    if torch is not None and isinstance(a, torch.Tensor):
        t = a.detach().cpu()
        if t.dtype not in (torch.float64, torch.float32):
            t = t.to(torch.float32)
        return np.ascontiguousarray(t.numpy())
    arr = np.asarray(a)
    if arr.dtype not in (np.float64, np.float32):
        arr = arr.astype(np.float64)
    return np.ascontiguousarray(arr)


def _shape(a) -> tuple[int, ...]:
    return tuple(int(s) for s in a.shape)


def _array_token(a) -> tuple:
    """Cheap identity of one payload array: object id, data pointer, shape, dtype and (torch) the
    in-place version counter — changes whenever the array is replaced or a torch tensor is
    written in place."""
    if torch is not None and isinstance(a, torch.Tensor):
        return (id(a), a.data_ptr(), tuple(a.shape), str(a.dtype), a._version)
    arr = np.asarray(a)
    return (id(a), arr.__array_interface__["data"][0], arr.shape, arr.dtype.str)


def _array_digest(a) -> int:
    """Content checksum (crc32 of the bytes) of one payload array — detects in-place writes to
    numpy arrays, which carry no version counter."""
    import zlib

    if torch is not None and isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    arr = np.ascontiguousarray(np.asarray(a))
    return zlib.crc32(memoryview(arr).cast("B"))


@dataclass(eq=False)
class CompressedLayer:
    """Tagged union over Dense / Tucker / TT / TR storage (tn_decompositions.py:66-126).

    Arrays are stored by reference, as in the reference, and the reference re-reads them on
    every ``reconstruct`` (:346-361). Device plans are packed snapshots, so they are cached under
    a key that includes every payload array's identity (object, data pointer, shape, dtype, and a
    torch tensor's in-place version): replacing a core, swapping the factor list or writing a
    torch core in place re-plans on the next call. numpy arrays have no version counter, so the
    reference-API functions (``reconstruct``, ``layer_to_matrix``, ``apply_compressed``) also
    compare a crc32 of the payload bytes; ``forward(x, check_cores=True)`` does the same on the
    hot path. ``invalidate()`` drops every cached plan explicitly.
    """

    family: str
    mode_shape: tuple
    row_mode_count: int
    matrix: Any = None
    core: Any = None
    factors: list = field(default_factory=list)
    cores: list = field(default_factory=list)

    def __post_init__(self):
        self.mode_shape = tuple(int(s) for s in self.mode_shape)
        self._plans: dict = {}
        self.validate()

    # --- reference properties (:82-95) --------------------------------------
    @property
    def matrix_shape(self) -> tuple[int, int]:
        rows = math.prod(self.mode_shape[: self.row_mode_count])
        return rows, math.prod(self.mode_shape) // rows

    @property
    def ranks(self) -> tuple[int, ...] | None:
        if self.family == "tucker":
            return _shape(self.core)
        if self.family == "tt":
            return tuple(_shape(c)[2] for c in self.cores[:-1])
        if self.family == "tr":
            return tuple(_shape(c)[0] for c in self.cores)
        return None

    def validate(self) -> None:
        """Same checks and messages as tn_decompositions.py:97-126."""
        d = len(self.mode_shape)
        if not 1 <= self.row_mode_count < d:
            raise ShapeError(f"row_mode_count {self.row_mode_count} invalid for {d} modes")
        if self.family == DENSE:
            if self.matrix is None or _shape(self.matrix) != self.matrix_shape:
                raise ShapeError("dense layer must hold its matricized payload")
        elif self.family == "tucker":
            if self.core is None or len(self.factors) != d:
                raise ShapeError("tucker layer needs a core and one factor per mode")
            cs = _shape(self.core)
            for k, f in enumerate(self.factors):
                if _shape(f) != (self.mode_shape[k], cs[k] if k < len(cs) else -1):
                    raise ShapeError(f"tucker factor {k} has shape {_shape(f)}")
        elif self.family in ("tt", "tr"):
            if len(self.cores) != d:
                raise ShapeError(f"{self.family} layer needs {d} cores")
            for k, c in enumerate(self.cores):
                s = _shape(c)
                if len(s) != 3 or s[1] != self.mode_shape[k]:
                    raise ShapeError(f"core {k} has shape {s}")
                nxt = _shape(self.cores[(k + 1) % d])
                if k + 1 < d and s[2] != nxt[0]:
                    raise ShapeError("chain bond mismatch")
            if self.family == "tt":
                if _shape(self.cores[0])[0] != 1 or _shape(self.cores[-1])[2] != 1:
                    raise ShapeError("tt boundary ranks must be 1")
            else:
                if _shape(self.cores[-1])[2] != _shape(self.cores[0])[0]:
                    raise ShapeError("tr closing bond mismatch")
        else:
            raise ShapeError(f"unknown family {self.family!r}")

    # --- bookkeeping ------------------------------------------------------------
    @property
    def bonds(self) -> tuple[int, ...]:
        """TT/TR bonds b_0..b_d (core k = (b_k, n_k, b_{k+1})); Tucker ranks."""
        if self.family in ("tt", "tr"):
            return tuple(_shape(c)[0] for c in self.cores) + (_shape(self.cores[-1])[2],)
        if self.family == "tucker":
            return _shape(self.core)
        return ()

    @property
    def cut_rank(self) -> int:
        return cut_rank(self.family, self.mode_shape, self.row_mode_count, self.bonds)

    def chain_flops_per_token(self) -> int:
        return chain_flops_per_token(self.family, self.mode_shape, self.row_mode_count, self.bonds)

    def invalidate(self) -> None:
        for p in self._plans.values():
            p.close()
        self._plans.clear()
        self._digest = None

    def _payload(self) -> list:
        if self.family == "tucker":
            return [self.core] + list(self.factors)
        if self.family in ("tt", "tr"):
            return list(self.cores)
        return [self.matrix]

    def _identity(self) -> tuple:
        return (self.family, self.mode_shape, self.row_mode_count,
                tuple(_array_token(a) for a in self._payload()))

    def check_cores(self) -> None:
        """Re-plan if any payload array changed content since the plans were built (crc32)."""
        dg = tuple(_array_digest(a) for a in self._payload())
        prev = getattr(self, "_digest", None)
        if self._plans and (prev is None or dg != prev):  # plans of unknown / different content
            self.invalidate()
        self._digest = dg

    # --- device plans -------------------------------------------------------
    def plan(self, dtype=None, device=None, flags: int = N.PLAN_AUTO, max_m: int = 0,
             row_range: tuple[int, int] | None = None) -> "NativePlan":
        if torch is None:
            raise DeviceError("torch is required for device plans")
        dtype = dtype or torch.bfloat16
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        if device is None:
            raise DeviceError("no CUDA device: the TN layer has no CPU fallback")
        device = torch.device(device)
        ident = self._identity()
        if getattr(self, "_ident", None) != ident:  # a core was replaced / written (torch) in place
            if self._plans:
                self.validate()
                for p in self._plans.values():
                    p.close()
                self._plans.clear()
            self._ident = ident
        key = (dtype, device.index, flags, max_m, row_range)
        p = self._plans.get(key)
        if p is None:
            p = NativePlan(self, dtype, device, flags, max_m, row_range)
            self._plans[key] = p
        return p

    def forward(self, x, out=None, flags: int = N.PLAN_AUTO, check_cores: bool = False):
        """y (M, rows) = x (M, cols) @ W^T on the GPU (x: CUDA bf16 or fp32 tensor)."""
        if torch is None or not isinstance(x, torch.Tensor) or not x.is_cuda:
            raise DeviceError("forward needs a CUDA tensor (no CPU fallback)")
        if check_cores:
            self.check_cores()
        return self.plan(x.dtype, x.device, flags).forward(x, out=out)

    __call__ = forward


class NativePlan:
    """Owns a ``tnl_plan*``: packed cores, panels, and a reusable workspace."""

    def __init__(self, layer: CompressedLayer, dtype, device, flags: int, max_m: int,
                 row_range: tuple[int, int] | None = None):
        if dtype not in (torch.bfloat16, torch.float32):
            raise ValueError(f"compute dtype must be bfloat16 or float32, got {dtype}")
        self.lib = N.load()
        self.dtype = dtype
        self.device = device
        self.layer = layer
        desc = N.LayerDesc()
        desc.family = N.FAMILY_CODE.get(layer.family, -1)
        d = len(layer.mode_shape)
        desc.ndim = d
        desc.row_mode_count = layer.row_mode_count
        if d > N.MAX_MODES:
            raise ShapeError(f"mode shape length must be in [2, {N.MAX_MODES}], got {d}")
        for k, s in enumerate(layer.mode_shape):
            desc.mode_shape[k] = s
        if layer.family == "tucker":
            arrays = [layer.core] + list(layer.factors)
            for k, r in enumerate(_shape(layer.core)):
                desc.ranks[k] = r
        elif layer.family in ("tt", "tr"):
            arrays = list(layer.cores)
            for k, b in enumerate(layer.bonds):
                desc.ranks[k] = b
        else:
            arrays = [layer.matrix]
        host = [_as_host_array(a) for a in arrays]
        src = N.TNL_F64 if all(h.dtype == np.float64 for h in host) else N.TNL_F32
        host = [h.astype(np.float64 if src == N.TNL_F64 else np.float32, copy=False) for h in host]
        for h in host:
            if not np.all(np.isfinite(h)):
                from .errors import NumericsError

                raise NumericsError("tensor entries must be finite")
        desc.src_dtype = src
        for k, h in enumerate(host):
            desc.arrays[k] = h.ctypes.data_as(ctypes.c_void_p)
        self._keep = host
        cdt = N.TNL_BF16 if dtype == torch.bfloat16 else N.TNL_F32
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            if row_range is None:
                st = self.lib.tnl_plan_create(ctypes.byref(desc), cdt, max_m, flags, ctypes.byref(handle))
            else:
                st = self.lib.tnl_plan_create_rows(ctypes.byref(desc), cdt, max_m, flags, int(row_range[0]),
                                                   int(row_range[1]), ctypes.byref(handle))
        N.check(st)
        self.handle = handle
        self._keep = None
        info = N.PlanInfo()
        N.check(self.lib.tnl_plan_query(self.handle, ctypes.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in N.PlanInfo._fields_}
        self.info["plan_large_name"] = N.PLAN_NAMES.get(info.plan_large, str(info.plan_large))
        self.info["plan_small_name"] = N.PLAN_NAMES.get(info.plan_small, str(info.plan_small))
        self.rows_local = info.row_end - info.row_begin
        self._ws = None

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.tnl_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def workspace_bytes(self, m: int) -> int:
        n = ctypes.c_size_t()
        N.check(self.lib.tnl_workspace_size(self.handle, int(m), ctypes.byref(n)))
        return int(n.value)

    def workspace(self, m: int):
        """Zero-filled workspace (the decode accumulator at its head is kept zero at rest)."""
        need = self.workspace_bytes(m)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.zeros(max(need, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def forward(self, x, out=None, stream=None, ws=None):
        if not isinstance(x, torch.Tensor) or not x.is_cuda:
            raise DeviceError("forward needs a CUDA tensor (no CPU fallback)")
        cols = self.info["cols"]
        if x.dim() != 2 or x.shape[1] != cols:
            raise ShapeError(f"x inner dimension {tuple(x.shape)} does not match {cols} columns")
        if x.dtype != self.dtype:
            raise ValueError(f"x dtype {x.dtype} != plan dtype {self.dtype}")
        m = x.shape[0]
        if x.stride(1) != 1 or (m > 1 and x.stride(0) < cols):
            x = x.contiguous()
        ldx = x.stride(0) if m > 1 else cols
        if out is None:
            out = torch.empty((m, self.rows_local), dtype=self.dtype, device=x.device)
        else:
            check_out(out, m, self.rows_local, self.dtype, x.device)
        if ws is None or ws.numel() < self.workspace_bytes(m):
            ws = self.workspace(m)
        if stream is None:
            stream = torch.cuda.current_stream(x.device).cuda_stream
        ldy = out.stride(0) if m > 1 else self.rows_local
        st = self.lib.tnl_forward(self.handle, ctypes.c_void_p(x.data_ptr()), m, ldx,
                                  ctypes.c_void_p(out.data_ptr()), ldy,
                                  ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(stream))
        N.check(st)
        return out

    def forward_host(self, x_host, y_host, stream=None):
        """End-to-end call: pinned host x -> device -> forward -> pinned host y (async)."""
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        st = self.lib.tnl_forward_host(self.handle, ctypes.c_void_p(x_host.data_ptr()), x_host.shape[0],
                                       ctypes.c_void_p(y_host.data_ptr()), ctypes.c_void_p(stream))
        N.check(st)
        return y_host

    def reconstruct(self, out_dtype=torch.float32):
        rows, cols = self.rows_local, self.info["cols"]
        w = torch.empty((rows, cols), dtype=out_dtype, device=self.device)
        odt = N.TNL_BF16 if out_dtype == torch.bfloat16 else N.TNL_F32
        stream = torch.cuda.current_stream(self.device).cuda_stream
        N.check(self.lib.tnl_reconstruct(self.handle, ctypes.c_void_p(w.data_ptr()), cols, odt,
                                         ctypes.c_void_p(stream)))
        return w


def check_out(out, m: int, rows: int, dtype, device) -> None:
    """A caller-supplied output must be exactly what the kernels write: (m, rows), the plan's
    compute dtype, on the input's device, unit stride along rows, row pitch >= rows."""
    if not isinstance(out, torch.Tensor):
        raise ShapeError("out must be a torch tensor")
    if tuple(out.shape) != (m, rows):
        raise ShapeError(f"out has shape {tuple(out.shape)}, expected {(m, rows)}")
    if out.dtype != dtype:
        raise ShapeError(f"out dtype {out.dtype} != compute dtype {dtype}")
    if out.device != torch.device(device):
        raise ShapeError(f"out is on {out.device}, x on {device}")
    if m > 0 and (out.stride(1) != 1 or (m > 1 and out.stride(0) < rows)):
        raise ShapeError(f"out strides {tuple(out.stride())} are not row-major with unit column stride")


# --- module functions (reference API) ------------------------------------------


def from_compressed_layer(ref_layer) -> CompressedLayer:
    """Adapter from a reference ``minima.tn_decompositions.CompressedLayer`` (`:66-80`), or any
    object with the same fields, to this package's layer. Arrays are taken by
    reference, as the reference does; validation runs with the reference's messages."""
    return CompressedLayer(
        str(ref_layer.family), tuple(int(s) for s in ref_layer.mode_shape), int(ref_layer.row_mode_count),
        matrix=getattr(ref_layer, "matrix", None), core=getattr(ref_layer, "core", None),
        factors=list(getattr(ref_layer, "factors", None) or []), cores=list(getattr(ref_layer, "cores", None) or []))


def reconstruct(layer: CompressedLayer, dtype=None, device=None):
    """Dense tensor of ``layer.mode_shape`` computed on the GPU (tn_decompositions.py:346-361).

    Uses fp32 cores (``dtype=torch.float32``, default) so the result is the
    layer itself; pass ``torch.bfloat16`` to reconstruct the bf16-rounded cores.
    """
    layer.validate()
    layer.check_cores()  # the reference re-reads the arrays on every call (:346-361)
    dtype = dtype or torch.float32
    p = layer.plan(dtype=dtype, device=device, flags=N.PLAN_GENERIC)
    return p.reconstruct(torch.float32).reshape(layer.mode_shape)


def layer_to_matrix(layer: CompressedLayer, dtype=None, device=None):
    """tn_decompositions.py:364-365 — reconstruct(...).reshape(rows, cols)."""
    return reconstruct(layer, dtype, device).reshape(layer.matrix_shape)


def apply_compressed(layer: CompressedLayer, x, flags: int = N.PLAN_AUTO):
    """W @ x for x (cols, M) without materialising W; returns (rows, M)."""
    rows, cols = layer.matrix_shape
    if x.dim() != 2 or x.shape[0] != cols:
        raise ShapeError(f"x inner dimension {tuple(x.shape)} does not match {cols} columns")
    return layer.forward(x.t().contiguous(), flags=flags, check_cores=True).t()


def param_count(layer: CompressedLayer) -> int:
    """tn_decompositions.py:368-374 — stored scalars in the payload."""
    if layer.family == DENSE:
        return int(math.prod(_shape(layer.matrix)))
    if layer.family == "tucker":
        return int(math.prod(_shape(layer.core)) + sum(math.prod(_shape(f)) for f in layer.factors))
    return int(sum(math.prod(_shape(c)) for c in layer.cores))


def compression_ratio(layer: CompressedLayer) -> float:
    """tn_decompositions.py:377-378."""
    return param_count(layer) / math.prod(layer.mode_shape)


__all__ = [
    "CompressedLayer",
    "NativePlan",
    "reconstruct",
    "layer_to_matrix",
    "apply_compressed",
    "param_count",
    "compression_ratio",
    "param_count_formula",
    "FAMILIES",
    "DENSE",
]
