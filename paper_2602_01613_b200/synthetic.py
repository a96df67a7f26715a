"""Synthetic layers and activations at the BASELINE shapes.

Random-init cores (there are no checkpoints offline) generated on the host
with the reference's generator ``np.random.Generator(np.random.Philox(seed))``
(sensitivity.py:179), variance-preserving so Var(y) ~ Var(x):
  TT  core k ~ N(0, 1/(r_{k+1} cols^{1/d})), last core N(0, cols^{-1/d})
  TR  core k ~ N(0, 1/(r_{k+1 mod d} cols^{1/d}))
  Tucker factors = orthonormal Q of QR(N(0,1)) (Cholesky QR); core ~ N(0, rows/prod R)
Seeds: 10_000*cfg + 100*layer + k for core k. Arrays are float32 (the GPU
plans round to bf16 themselves).
"""

from __future__ import annotations

import math

import numpy as np

from .layer import CompressedLayer


def philox(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed))


def orthonormal(a: np.ndarray) -> np.ndarray:
    """Q of the QR factorisation of a tall Gaussian matrix, with the positive-diagonal convention
    (Cholesky QR: R = chol(AᵀA)ᵀ, Q = A R⁻¹). For these well-conditioned matrices it equals
    Householder QR up to column signs to ~1e-16, at a quarter of the cost — the cfg4 stack draws
    ~400 factors of up to 25600 x 256, which dominated its construction time."""
    from scipy.linalg import solve_triangular

    if a.shape[1] > a.shape[0]:
        q, _ = np.linalg.qr(a)
        return np.ascontiguousarray(q)
    r = np.linalg.cholesky(a.T @ a).T  # upper triangular, positive diagonal
    return np.ascontiguousarray(solve_triangular(r, a.T, trans="T", lower=False).T)


def make_layer(family: str, mode_shape, row_mode_count: int, ranks, seed: int) -> CompressedLayer:
    ms = tuple(int(s) for s in mode_shape)
    d = len(ms)
    rows = math.prod(ms[:row_mode_count])
    cols = math.prod(ms) // rows
    f32 = np.float32
    if family == "tt":
        b = (1,) + tuple(ranks) + (1,)
        cores = []
        for k in range(d):
            var = 1.0 / (b[k + 1] * cols ** (1.0 / d)) if k < d - 1 else cols ** (-1.0 / d)
            cores.append((philox(seed + k).standard_normal((b[k], ms[k], b[k + 1])) * math.sqrt(var)).astype(f32))
        return CompressedLayer("tt", ms, row_mode_count, cores=cores)
    if family == "tr":
        r = tuple(ranks)
        cores = []
        for k in range(d):
            var = 1.0 / (r[(k + 1) % d] * cols ** (1.0 / d))
            cores.append((philox(seed + k).standard_normal((r[k], ms[k], r[(k + 1) % d])) * math.sqrt(var)).astype(f32))
        return CompressedLayer("tr", ms, row_mode_count, cores=cores)
    if family == "tucker":
        R = tuple(ranks)
        factors = []
        for k in range(d):
            factors.append(orthonormal(philox(seed + k).standard_normal((ms[k], R[k]))).astype(f32))
        core = (philox(seed + d).standard_normal(R) * math.sqrt(rows / math.prod(R))).astype(f32)
        return CompressedLayer("tucker", ms, row_mode_count, core=core, factors=factors)
    if family == "dense":
        w = (philox(seed).standard_normal((rows, cols)) / math.sqrt(cols)).astype(f32)
        return CompressedLayer("dense", ms, row_mode_count, matrix=w)
    raise ValueError(f"unknown family {family!r}")


def make_x(m: int, cols: int, seed: int) -> np.ndarray:
    return philox(seed).standard_normal((m, cols)).astype(np.float32)


# --- BASELINE config layer sets ------------------------------------------------

# cfg2: Qwen3-32B attention projection 5120 -> 5120, ranks 64-256 (cut), decode M=1..64
CFG2_VARIANTS = [
    ("tucker-2 R64", "tucker", (5120, 5120), 1, (64, 64)),
    ("tucker-2 R128", "tucker", (5120, 5120), 1, (128, 128)),
    ("tucker-2 R256", "tucker", (5120, 5120), 1, (256, 256)),
    ("tr2 (8,8)", "tr", (5120, 5120), 1, (8, 8)),
    ("tr2 (16,16)", "tr", (5120, 5120), 1, (16, 16)),
    ("tr4 r8", "tr", (64, 80, 64, 80), 2, (8, 8, 8, 8)),
    ("tr4 r16", "tr", (64, 80, 64, 80), 2, (16, 16, 16, 16)),
]

# cfg3: Qwen3-32B MLP gate/up (5120 -> 25600) and down (25600 -> 5120), TT r64
CFG3_GATE = ("tt", (160, 160, 64, 80), 2, (64, 64, 64))
CFG3_DOWN = ("tt", (64, 80, 160, 160), 2, (64, 64, 64))

# cfg1: TT 4096 -> 4096, (64,64|64,64) r32, M=16, fp32
CFG1 = ("tt", (64, 64, 64, 64), 2, (32, 32, 32))


def cfg2_bank(copies: int = 10):
    """copies x 7 distinct cfg2 layers, interleaved (weights > L2 at copies=10)."""
    out = []
    for c in range(copies):
        for v, (name, fam, ms, rm, ranks) in enumerate(CFG2_VARIANTS):
            layer = make_layer(fam, ms, rm, ranks, seed=20_000 + 100 * (c * len(CFG2_VARIANTS) + v))
            out.append((name, layer))
    return out
