"""One-sided Jacobi sweeps and the deterministic SVD built on them, on the GPU.

Drop-in for the reference's only native component and its caller:

* ``jacobi_sweeps(work, rot, tol, max_sweeps) -> int`` — same contract as
  ``minima._jacobi_cy.jacobi_sweeps`` (`_jacobi_cy.pyx:11-53`, selected by `_backend.py:5-25`):
  numpy float64 C-contiguous arrays, updated in place, returns the sweep count;
* ``jacobi_sweeps_batched(work, rot, tol, max_sweeps)`` — a batch of independent problems as
  CUDA float64 tensors ``(B, n, m)`` / ``(B, n, nv)`` (one warp per problem, `csrc/jacobi.cu`);
* ``full_svd`` / ``truncated_svd`` / ``svd_batched`` — `tensor_core._jacobi_svd`
  (`tensor_core.py:203-235`) with the sweeps AND the post-processing (stable sort by column norm,
  normalisation, zero-column completion `:185-200`, sign convention `:226-230`) on the GPU
  (``tnl_svd_finish``), and the reference's truncation policies (`:238-288`) applied to the
  returned spectrum;
* ``parallel=True`` — one large problem (a Qwen-shaped unfolding) swept in the round-robin
  parallel order (``tnl_jacobi_sweeps_parallel``, one warp per pair across all SMs) instead of the
  reference's cyclic order; equal up to rounding.

All numerics run in ``libtnl.so``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import DeviceError, InfeasibleBudgetError, RankError, ShapeError

JACOBI_TOL = 1e-12  # tensor_core.py:32
JACOBI_MAX_SWEEPS = 60  # tensor_core.py:33


# truncation policies (tensor_core.py:136-166) are shared with the rank planner
from .modes import FixedRank, ParamBudget, RelativeError  # noqa: E402


@dataclass(frozen=True)
class SvdResult:
    """``left @ diag(values) @ right.T`` approximates the input (tensor_core.py:169-182)."""

    left: np.ndarray
    values: np.ndarray
    right: np.ndarray

    @property
    def rank(self) -> int:
        return int(self.values.shape[0])

    def reconstruct(self) -> np.ndarray:
        return (self.left * self.values) @ self.right.T


# --- sweeps -----------------------------------------------------------------------------


def _device():
    if not torch.cuda.is_available():
        raise DeviceError("jacobi sweeps run on the GPU (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def jacobi_sweeps_batched(work: torch.Tensor, rot: torch.Tensor, tol: float = JACOBI_TOL,
                          max_sweeps: int = JACOBI_MAX_SWEEPS) -> torch.Tensor:
    """In-place sweeps over a batch: work (B, n, m), rot (B, n, nv) CUDA float64 contiguous.

    Returns the per-problem sweep counts (B,) int32 (on the device)."""
    if work.dim() != 3 or rot.dim() != 3 or work.shape[:2] != rot.shape[:2]:
        raise ShapeError(f"work {tuple(work.shape)} / rot {tuple(rot.shape)}: expected (B, n, m) / (B, n, nv)")
    for t in (work, rot):
        if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
            raise DeviceError("work / rot must be contiguous CUDA float64 tensors")
    b, n, m = work.shape
    nv = rot.shape[2]
    sweeps = torch.zeros(b, dtype=torch.int32, device=work.device)
    lib = N.load()
    stream = torch.cuda.current_stream(work.device).cuda_stream
    N.check(lib.tnl_jacobi_sweeps(ctypes.c_void_p(work.data_ptr()), ctypes.c_void_p(rot.data_ptr()), b, n, m, nv,
                                  float(tol), int(max_sweeps), ctypes.c_void_p(sweeps.data_ptr()),
                                  ctypes.c_void_p(stream)))
    return sweeps


def jacobi_sweeps(work: np.ndarray, rot: np.ndarray, tol: float, max_sweeps: int) -> int:
    """Reference contract (`_jacobi_cy.pyx:11`): orthogonalise the rows of ``work`` in place."""
    if not (isinstance(work, np.ndarray) and isinstance(rot, np.ndarray)) or work.dtype != np.float64 \
            or rot.dtype != np.float64 or work.ndim != 2 or rot.ndim != 2:
        raise ShapeError("work and rot must be 2-D float64 numpy arrays")
    if rot.shape[0] != work.shape[0]:
        raise ShapeError(f"rot has {rot.shape[0]} rows, work has {work.shape[0]}")
    dev = _device()
    w = torch.from_numpy(np.ascontiguousarray(work)).to(dev).unsqueeze(0).contiguous()
    r = torch.from_numpy(np.ascontiguousarray(rot)).to(dev).unsqueeze(0).contiguous()
    s = jacobi_sweeps_batched(w, r, tol, max_sweeps)
    work[...] = w[0].cpu().numpy()
    rot[...] = r[0].cpu().numpy()
    return int(s[0].item())


# --- SVD (tensor_core.py:185-288) --------------------------------------------------------


def svd_batched(mats, tol: float = JACOBI_TOL, max_sweeps: int = JACOBI_MAX_SWEEPS, parallel: bool = False) -> list:
    """Full deterministic SVDs of same-shape matrices (list or (B, m, n) array), all on the GPU:
    the sweeps (``tnl_jacobi_sweeps``, one launch for the batch — or, ``parallel=True``, the
    round-robin ``tnl_jacobi_sweeps_parallel`` per problem for large single unfoldings) and the
    post-processing of ``_jacobi_svd`` (tensor_core.py:214-235: ordering, normalisation, basis
    completion, sign convention) by ``tnl_svd_finish``. Only the results return to the host."""
    a = np.asarray(mats, dtype=np.float64)
    if a.ndim != 3:
        raise ShapeError(f"expected a batch of rank-2 arrays, got shape {a.shape}")
    if not np.all(np.isfinite(a)):
        from .errors import NumericsError

        raise NumericsError("non-finite values in SVD input")
    b, m, n = a.shape
    transposed = m < n
    if transposed:
        a = np.swapaxes(a, 1, 2)
        m, n = n, m
    dev = _device()
    work = torch.from_numpy(np.ascontiguousarray(np.swapaxes(a, 1, 2))).to(dev)  # (B, n, m): a.T per problem
    rot = torch.eye(n, dtype=torch.float64, device=dev).expand(b, n, n).contiguous()
    lib = N.load()
    stream = torch.cuda.current_stream(dev).cuda_stream
    if parallel:
        for i in range(b):
            N.check(lib.tnl_jacobi_sweeps_parallel(ctypes.c_void_p(work[i].data_ptr()), ctypes.c_void_p(rot[i].data_ptr()),
                                                   n, m, n, float(tol), int(max_sweeps), None, ctypes.c_void_p(stream)))
    else:
        jacobi_sweeps_batched(work, rot, tol, max_sweeps)
    left = torch.empty((b, m, n), dtype=torch.float64, device=dev)
    values = torch.empty((b, n), dtype=torch.float64, device=dev)
    right = torch.empty((b, n, n), dtype=torch.float64, device=dev)
    scratch = torch.empty((b, 2 * n + 2 * m), dtype=torch.float64, device=dev)
    N.check(lib.tnl_svd_finish(ctypes.c_void_p(work.data_ptr()), ctypes.c_void_p(rot.data_ptr()), b, n, m,
                               ctypes.c_void_p(left.data_ptr()), ctypes.c_void_p(values.data_ptr()),
                               ctypes.c_void_p(right.data_ptr()), ctypes.c_void_p(scratch.data_ptr()),
                               ctypes.c_void_p(stream)))
    lh, vh, rh = left.cpu().numpy(), values.cpu().numpy(), right.cpu().numpy()
    if transposed:
        lh, rh = rh, lh
    return [SvdResult(left=lh[i], values=vh[i], right=rh[i]) for i in range(b)]


def _select_rank(values: np.ndarray, shape, policy) -> int:
    """tensor_core.py:238-266."""
    m, n = shape
    kmax = min(m, n)
    if isinstance(policy, FixedRank):
        if policy.rank > kmax:
            raise RankError(f"fixed rank {policy.rank} exceeds min(m, n) = {kmax}")
        return policy.rank
    if isinstance(policy, RelativeError):
        energies = values**2
        total = float(energies.sum())
        if total == 0.0:
            return 1
        tail = total
        target = (policy.epsilon**2) * total
        for r in range(1, kmax + 1):
            tail -= float(energies[r - 1])
            if tail <= target:
                return r
        return kmax
    if isinstance(policy, ParamBudget):
        per_triplet = m + n + 1
        r = min(policy.budget // per_triplet, kmax)
        if r < 1:
            raise InfeasibleBudgetError(
                f"budget {policy.budget} below one (u, s, v) triplet of size {per_triplet}",
                best_achievable=per_triplet)
        return r
    raise TypeError(f"unknown truncation policy: {policy!r}")


def truncated_svd(matrix, policy, parallel: bool = False) -> SvdResult:
    """Deterministic truncated SVD (tensor_core.py:269-288), computed on the GPU."""
    m = np.asarray(matrix, dtype=np.float64)
    if m.ndim != 2:
        raise ShapeError(f"expected a rank-2 tensor, got rank {m.ndim}")
    full = svd_batched(m[None], parallel=parallel)[0]
    r = _select_rank(full.values, m.shape, policy)
    return SvdResult(left=np.ascontiguousarray(full.left[:, :r]), values=full.values[:r].copy(),
                     right=np.ascontiguousarray(full.right[:, :r]))


def full_svd(matrix, parallel: bool = False) -> SvdResult:
    """All ``min(m, n)`` singular triplets (tensor_core.py:291-296)."""
    m = np.asarray(matrix, dtype=np.float64)
    if m.ndim != 2:
        raise ShapeError(f"expected a rank-2 tensor, got rank {m.ndim}")
    return truncated_svd(m, FixedRank(min(m.shape)), parallel=parallel)
