"""Contraction planning and FLOP accounting of the layer-apply network.

Host-side mirror of the SPEC's `structured_inference` contracts (`SPEC.md:465-518`; absent from the
reference code) plus the two tensor helpers the reference forward path is built from
(`tensor_core.py:54-78`):

* ``relative_error(a, b)`` — ``‖a − b‖_F / ‖a‖_F`` in float64 with the reference's errors
  (`tensor_core.py:54-63`, `as_tensor` `:36-47`); accepts numpy arrays or torch tensors;
* ``reshape_to_modes(matrix, mode_shape)`` — the view `tensor_core.py:66-78` (numpy or torch);
* ``plan_contraction(layer, batch) -> ContractionPlan`` — exhaustive search (dynamic programming
  over operand subsets, i.e. every pairwise contraction tree) of the network
  {cores or core+factors or W, x (cols modes × batch)}, minimising
  Σ 2·Π(all mode sizes involved in a step) (`SPEC.md:465-473`), ties broken by the
  lexicographic step encoding; never worse than the left-to-right order (`SPEC.md:486-494`);
* (the float64 step-by-step executor of a plan, ``execute_plan``, is test infrastructure and lives
  in ``oracle/plan_exec.py``; this package never computes a layer on the CPU) — it counts the
  multiply-adds and the largest intermediate, for the SPEC's instrumentation invariants;
* ``flop_report(layers, batch) -> FlopReport`` (`SPEC.md:496-500`);
* ``micro_benchmark(layer, x, reps, warmup)`` (`SPEC.md:502-507`) — median / IQR of the GPU
  forward with CUDA events, warm-up discarded.

The device kernels do not consult these plans: their order is fixed per plan kind (cut or core
chain), and ``chain_flops_per_token`` reports what they execute. The planner here is
the reference-facing accounting (and shows how far each kernel order is from the optimum).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .errors import DegenerateReferenceError, NumericsError, ShapeError

# --- tensor helpers (tensor_core.py:36-78) ---------------------------------------------------


def _as_float64(t) -> np.ndarray:
    try:
        import torch

        if isinstance(t, torch.Tensor):
            t = t.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    a = np.asarray(t, dtype=np.float64)
    if not np.all(np.isfinite(a)):
        raise NumericsError("non-finite values")
    return a


def relative_error(a, b) -> float:
    """Frobenius-relative deviation ``‖a − b‖ / ‖a‖`` (tensor_core.py:54-63); a is the reference."""
    a = _as_float64(a)
    b = _as_float64(b)
    if a.shape != b.shape:
        raise ShapeError(f"shape mismatch: {a.shape} vs {b.shape}")
    ref = float(np.linalg.norm(a))
    if ref == 0.0:
        raise DegenerateReferenceError("relative error against a zero tensor")
    return float(np.linalg.norm(a - b)) / ref


def reshape_to_modes(matrix, mode_shape):
    """Reinterpret a matrix as a multi-mode tensor without moving data (tensor_core.py:66-78)."""
    shape = tuple(getattr(matrix, "shape", ()))
    if len(shape) != 2:
        raise ShapeError(f"expected a rank-2 tensor, got rank {len(shape)}")
    mode_shape = tuple(int(s) for s in mode_shape)
    if not 2 <= len(mode_shape) <= 6:
        raise ShapeError(f"mode shape length must be in [2, 6], got {len(mode_shape)}")
    if any(s < 1 for s in mode_shape):
        raise ShapeError(f"all mode sizes must be >= 1, got {mode_shape}")
    if math.prod(mode_shape) != shape[0] * shape[1]:
        raise ShapeError(f"mode shape {mode_shape} does not match {shape[0]}x{shape[1]} entries")
    return matrix.reshape(mode_shape)


# --- the layer-apply network ---------------------------------------------------------------


@dataclass(frozen=True)
class Network:
    """Operands as tuples of mode labels; `sizes` per label; `out` labels of y (rows modes, batch)."""

    names: tuple
    operands: tuple
    sizes: dict
    out: tuple


def layer_network(layer, batch: int) -> Network:
    """W·x of the reference orientation (`sensitivity.py:154-160`): x is (cols modes..., batch)."""
    ms, rm, fam = tuple(layer.mode_shape), int(layer.row_mode_count), layer.family
    d = len(ms)
    sizes = {f"n{k}": ms[k] for k in range(d)}
    sizes["m"] = int(batch)
    names, ops = [], []
    if fam == "dense":
        rows, cols = layer.matrix_shape
        sizes = {"i": rows, "j": cols, "m": int(batch)}
        return Network(("W", "x"), (("i", "j"), ("j", "m")), sizes, ("i", "m"))
    if fam == "tucker":
        rk = tuple(int(r) for r in np.shape(layer.core))
        for k in range(d):
            sizes[f"R{k}"] = rk[k]
        names.append("G")
        ops.append(tuple(f"R{k}" for k in range(d)))
        for k in range(d):
            names.append(f"U{k}")
            ops.append((f"n{k}", f"R{k}"))
    elif fam in ("tt", "tr"):
        shapes = [tuple(int(s) for s in np.shape(c)) for c in layer.cores]
        for k in range(d):
            sizes[f"b{k}"] = shapes[k][0]
        sizes[f"b{d}"] = shapes[-1][2]
        for k in range(d):
            right = f"b{k + 1}" if (fam == "tt" or k + 1 < d) else "b0"  # TR closes the ring
            names.append(f"C{k}")
            ops.append((f"b{k}", f"n{k}", right))
    else:
        raise ShapeError(f"unknown family {fam!r}")
    names.append("x")
    ops.append(tuple(f"n{k}" for k in range(rm, d)) + ("m",))
    return Network(tuple(names), tuple(ops), sizes, tuple(f"n{k}" for k in range(rm)) + ("m",))


@dataclass
class ContractionPlan:
    """Ordered pairwise steps ``(a, b)`` over operand ids (inputs 0..n-1, step results n, n+1, ...)."""

    network: Network
    steps: list = field(default_factory=list)
    step_modes: list = field(default_factory=list)  # (modes of a, modes of b, modes of result)
    predicted_flops: int = 0
    largest_intermediate: int = 0


def _step_cost(sizes, ma, mb) -> int:
    return 2 * math.prod(sizes[l] for l in sorted(set(ma) | set(mb)))


def _plan_from_order(net: Network, order) -> ContractionPlan:
    """Plan that contracts the operands sequentially in `order` (left-to-right baseline)."""
    alive = {i: tuple(m) for i, m in enumerate(net.operands)}
    plan = ContractionPlan(net)
    nxt = len(net.operands)
    cur = order[0]
    for j in order[1:]:
        plan_step(plan, alive, cur, j, nxt)
        cur, nxt = nxt, nxt + 1
    return plan


def plan_step(plan: ContractionPlan, alive: dict, a: int, b: int, new: int) -> None:
    net = plan.network
    ma, mb = alive.pop(a), alive.pop(b)
    others = set(net.out)
    for m in alive.values():
        others |= set(m)
    res = tuple(l for l in dict.fromkeys(ma + mb) if l in others)
    alive[new] = res
    plan.steps.append((a, b))
    plan.step_modes.append((ma, mb, res))
    plan.predicted_flops += _step_cost(net.sizes, ma, mb)
    plan.largest_intermediate = max(plan.largest_intermediate, math.prod(net.sizes[l] for l in res))


def plan_contraction(layer, batch: int) -> ContractionPlan:
    """Minimal-FLOP pairwise contraction order, exact over all trees."""
    net = layer_network(layer, batch)
    n = len(net.operands)
    full = (1 << n) - 1
    label_sets = [set(o) for o in net.operands]
    out = set(net.out)

    @lru_cache(maxsize=None)
    def modes(mask: int) -> tuple:
        inside, outside = set(), set(out)
        for i in range(n):
            (inside if mask >> i & 1 else outside).update(label_sets[i])
        return tuple(sorted(inside & outside))

    @lru_cache(maxsize=None)
    def best(mask: int):
        if mask & (mask - 1) == 0:  # single operand
            return 0, ()
        cand = None
        sub = (mask - 1) & mask
        while sub:
            other = mask ^ sub
            if sub < other:  # each unordered split once
                ca, ea = best(sub)
                cb, eb = best(other)
                c = ca + cb + _step_cost(net.sizes, modes(sub), modes(other))
                enc = ea + eb + ((sub, other),)
                if cand is None or (c, enc) < cand:
                    cand = (c, enc)
            sub = (sub - 1) & mask
        return cand

    cost, enc = best(full)
    # replay the tree (post-order) as numbered steps
    plan = ContractionPlan(net)
    alive = {i: tuple(m) for i, m in enumerate(net.operands)}
    ident = {1 << i: i for i in range(n)}
    nxt = n
    for sa, sb in enc:
        plan_step(plan, alive, ident[sa], ident[sb], nxt)
        ident[sa | sb] = nxt
        nxt += 1
    assert plan.predicted_flops == cost
    return plan


def left_to_right_plan(layer, batch: int) -> ContractionPlan:
    """The baseline: operands contracted in their listed order (cores / factors, then x)."""
    net = layer_network(layer, batch)
    return _plan_from_order(net, list(range(len(net.operands))))


# --- reports ---------------------------------------------------------------------------------


@dataclass
class FlopReport:
    dense_flops: int
    structured_flops: int
    speedup_ratio: float
    per_layer: dict


def flop_report(layers, batch: int) -> FlopReport:
    """dense = Σ 2·rows·cols·batch, structured = Σ optimal plan FLOPs."""
    items = layers.items() if isinstance(layers, dict) else enumerate(layers)
    per, dense, struct = {}, 0, 0
    for name, lay in items:
        rows, cols = lay.matrix_shape
        dn = 2 * rows * cols * int(batch)
        st = plan_contraction(lay, batch).predicted_flops
        per[name] = {"dense_flops": dn, "structured_flops": st, "ratio": dn / st}
        dense += dn
        struct += st
    return FlopReport(dense, struct, dense / struct if struct else 1.0, per)


def micro_benchmark(layer, x, reps: int = 20, warmup: int = 3) -> dict:
    """Median / IQR of the GPU forward (CUDA events, warm-up discarded); machine-dependent."""
    if reps < 10:
        raise ValueError("micro_benchmark needs reps >= 10 (SPEC.md:504)")
    import torch

    for _ in range(warmup):
        layer.forward(x)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        layer.forward(x)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    q1, med, q3 = np.percentile(ts, [25, 50, 75])
    return {"median_ms": float(med), "iqr_ms": float(q3 - q1), "reps": reps, "warmup": warmup,
            "note": "machine-dependent wall-clock (CUDA events); not an acceptance gate"}
