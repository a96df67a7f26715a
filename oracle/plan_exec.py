"""Step-by-step float64 executor of a SPEC contraction plan — TEST INFRASTRUCTURE ONLY.

Runs a ``paper_2602_01613_b200.contraction.ContractionPlan`` pairwise with numpy einsum, counting
multiply-adds and the largest intermediate, so the tests can check that the planner's predicted
FLOPs are what the plan executes and that every plan reproduces the
reference's ``layer_to_matrix(L) @ x`` (tn_decompositions.py:364-365, sensitivity.py:154-160).
Only ``tests/`` import it; the product package never computes a layer on the CPU.
"""

from __future__ import annotations

import math

import numpy as np


def _arrays(layer):
    if layer.family == "dense":
        return [np.asarray(layer.matrix, dtype=np.float64)]
    if layer.family == "tucker":
        return [np.asarray(layer.core, dtype=np.float64)] + [np.asarray(f, dtype=np.float64) for f in layer.factors]
    return [np.asarray(c, dtype=np.float64) for c in layer.cores]


def execute_plan(plan: ContractionPlan, layer, x) -> tuple[np.ndarray, dict]:
    """Apply a plan to x (cols, batch) in float64; returns (y (rows, batch), instrumentation)."""
    net = plan.network
    x = np.asarray(x, dtype=np.float64)
    rm = layer.row_mode_count
    ms = tuple(layer.mode_shape)
    if layer.family == "dense":
        xin = x
    else:
        xin = x.reshape(ms[rm:] + (x.shape[1],))
    tensors = {i: a for i, a in enumerate(_arrays(layer) + [xin])}
    labels = {i: m for i, m in enumerate(net.operands)}
    letters = {}
    for l in net.sizes:
        letters[l] = chr(ord("a") + len(letters)) if len(letters) < 26 else chr(ord("A") + len(letters) - 26)
    macs, largest = 0, 0
    nxt = len(net.operands)
    for (a, b), (ma, mb, res) in zip(plan.steps, plan.step_modes):
        spec = "".join(letters[l] for l in ma) + "," + "".join(letters[l] for l in mb) + "->" + \
            "".join(letters[l] for l in res)
        tensors[nxt] = np.einsum(spec, tensors.pop(a), tensors.pop(b), optimize=False)
        labels[nxt] = res
        macs += math.prod(net.sizes[l] for l in set(ma) | set(mb))
        largest = max(largest, tensors[nxt].size)
        nxt += 1
    (last,) = tensors.keys()
    y = tensors[last]
    order = [labels[last].index(l) for l in net.out]
    y = np.transpose(y, order)
    rows = math.prod(ms[:rm]) if layer.family != "dense" else layer.matrix_shape[0]
    return y.reshape(rows, x.shape[1]), {"multiply_adds": macs, "flops": 2 * macs, "largest_intermediate": largest}
