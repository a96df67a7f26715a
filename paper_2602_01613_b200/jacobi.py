"""One-sided Jacobi sweeps and the deterministic SVD built on them, on the GPU.

Drop-in for the reference's only native component and its caller:

* ``jacobi_sweeps(work, rot, tol, max_sweeps) -> int`` — same contract as
  ``minima._jacobi_cy.jacobi_sweeps`` (`_jacobi_cy.pyx:11-53`, selected by `_backend.py:5-25`):
  numpy float64 C-contiguous arrays, updated in place, returns the sweep count;
* ``jacobi_sweeps_batched(work, rot, tol, max_sweeps)`` — a batch of independent problems as
  CUDA float64 tensors ``(B, n, m)`` / ``(B, n, nv)`` (one warp per problem, `csrc/jacobi.cu`);
* ``full_svd`` / ``truncated_svd`` / ``svd_batched`` — `tensor_core._jacobi_svd`
  (`tensor_core.py:203-235`) with the sweeps on the GPU and the reference's post-processing
  (stable sort by column norm, normalisation, zero-column completion `:185-200`, sign
  convention `:226-230`) and truncation policies (`:238-288`).

All sweeps run in ``libtnl.so`` (``tnl_jacobi_sweeps``); there is no CPU fallback.
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


def _complete_basis(u: np.ndarray, fixed: int) -> None:
    """Columns ``fixed:`` of ``u`` <- orthonormal filler, greedy canonical pick (tensor_core.py:185-200)."""
    m, k = u.shape
    for j in range(fixed, k):
        basis = u[:, :j]
        resid = np.eye(m) - basis @ basis.T
        pick = int(np.argmax(np.linalg.norm(resid, axis=0)))
        v = resid[:, pick]
        v = v - basis @ (basis.T @ v)
        u[:, j] = v / np.linalg.norm(v)


def _finish(work: np.ndarray, rot: np.ndarray, m: int, n: int, transposed: bool) -> SvdResult:
    """tensor_core.py:214-235: order by column norm, normalise, complete, sign-fix, un-transpose."""
    norms = np.linalg.norm(work, axis=1)
    order = np.argsort(-norms, kind="stable")
    values = norms[order]
    left = np.zeros((m, n))
    right = rot[order].T.copy()
    positive = int(np.count_nonzero(values > 0.0))
    for j in range(positive):
        left[:, j] = work[order[j]] / values[j]
    if positive < n:
        _complete_basis(left, positive)
    for j in range(n):
        pivot = int(np.argmax(np.abs(left[:, j])))
        if left[pivot, j] < 0.0:
            left[:, j] = -left[:, j]
            right[:, j] = -right[:, j]
    if transposed:
        left, right = right, left
    return SvdResult(left=left, values=values, right=right)


def svd_batched(mats, tol: float = JACOBI_TOL, max_sweeps: int = JACOBI_MAX_SWEEPS) -> list:
    """Full deterministic SVDs of same-shape matrices (list or (B, m, n) array), one GPU launch."""
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
    jacobi_sweeps_batched(work, rot, tol, max_sweeps)
    w, r = work.cpu().numpy(), rot.cpu().numpy()
    return [_finish(w[i], r[i], m, n, transposed) for i in range(b)]


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


def truncated_svd(matrix, policy) -> SvdResult:
    """Deterministic truncated SVD (tensor_core.py:269-288), sweeps on the GPU."""
    m = np.asarray(matrix, dtype=np.float64)
    if m.ndim != 2:
        raise ShapeError(f"expected a rank-2 tensor, got rank {m.ndim}")
    full = svd_batched(m[None])[0]
    r = _select_rank(full.values, m.shape, policy)
    return SvdResult(left=np.ascontiguousarray(full.left[:, :r]), values=full.values[:r].copy(),
                     right=np.ascontiguousarray(full.right[:, :r]))


def full_svd(matrix) -> SvdResult:
    """All ``min(m, n)`` singular triplets (tensor_core.py:291-296)."""
    m = np.asarray(matrix, dtype=np.float64)
    if m.ndim != 2:
        raise ShapeError(f"expected a rank-2 tensor, got rank {m.ndim}")
    return truncated_svd(m, FixedRank(min(m.shape)))
