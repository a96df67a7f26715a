"""Contraction planning / FLOP accounting and the tensor helpers
(tensor_core.py:54-78) — CPU only; the oracle is the checker."""

import itertools
import math

import numpy as np
import pytest

from oracle import plan_exec as PE
from oracle import tn_oracle as O
from paper_2602_01613_b200 import CompressedLayer
from paper_2602_01613_b200 import contraction as C
from paper_2602_01613_b200.errors import DegenerateReferenceError, NumericsError, ShapeError


def _layer(fam, ms, rm, ranks, seed=0):
    L = O.synthetic_layer(fam, ms, rm, ranks, seed=seed)
    return CompressedLayer(fam, ms, rm, matrix=L.matrix, core=L.core, factors=L.factors, cores=L.cores), L


def _all_tree_costs(net):
    """Brute force: minimal cost over every sequence of pairwise contractions."""
    best = [math.inf]

    def rec(alive, cost):
        if cost >= best[0]:
            return
        if len(alive) == 1:
            best[0] = cost
            return
        keys = sorted(alive)
        for a, b in itertools.combinations(keys, 2):
            ma, mb = alive[a], alive[b]
            others = set(net.out)
            for k, m in alive.items():
                if k not in (a, b):
                    others |= set(m)
            res = tuple(l for l in dict.fromkeys(ma + mb) if l in others)
            nxt = dict(alive)
            del nxt[a], nxt[b]
            nxt[max(alive) + 1] = res
            rec(nxt, cost + C._step_cost(net.sizes, ma, mb))

    rec({i: m for i, m in enumerate(net.operands)}, 0)
    return best[0]


def test_dense_single_step():
    lay, _ = _layer("dense", (6, 10), 1, ())
    p = C.plan_contraction(lay, 7)
    assert len(p.steps) == 1 and p.predicted_flops == 2 * 6 * 10 * 7


@pytest.mark.parametrize("fam,ms,rm,ranks", [
    ("tt", (8, 8, 8, 8), 2, (4, 4, 4)),
    ("tr", (8, 8, 8, 8), 2, (2, 3, 2, 3)),
    ("tucker", (8, 8, 8, 8), 2, (4, 3, 4, 3)),
    ("tt", (4, 6, 5), 1, (3, 2)),
])
def test_optimal_and_never_worse_than_left_to_right(fam, ms, rm, ranks):
    lay, _ = _layer(fam, ms, rm, ranks)
    for batch in (1, 16):
        p = C.plan_contraction(lay, batch)
        assert p.predicted_flops <= C.left_to_right_plan(lay, batch).predicted_flops
        assert p.predicted_flops == _all_tree_costs(p.network)


@pytest.mark.parametrize("fam,ms,rm,ranks", [
    ("dense", (12, 20), 1, ()),
    ("tt", (8, 8, 8, 8), 2, (4, 4, 4)),
    ("tr", (6, 10, 4), 1, (2, 3, 2)),
    ("tr", (8, 8, 8, 8), 2, (2, 3, 2, 3)),
    ("tucker", (8, 8, 8, 8), 2, (4, 3, 4, 3)),
    ("tucker", (24, 20), 1, (5, 6)),
])
def test_execute_plan_matches_reference_and_counts(fam, ms, rm, ranks):
    lay, Lo = _layer(fam, ms, rm, ranks, seed=3)
    rows, cols = lay.matrix_shape
    x = O.synthetic_x(5, cols, seed=4).T  # reference orientation (cols, M)
    ref = O.apply_reference(Lo, x)
    for plan in (C.plan_contraction(lay, 5), C.left_to_right_plan(lay, 5)):
        y, inst = PE.execute_plan(plan, lay, x)
        assert C.relative_error(ref, y) <= 1e-10
        assert inst["flops"] == plan.predicted_flops  # SPEC.md:511 instrumentation invariant
        assert inst["largest_intermediate"] == plan.largest_intermediate
    if fam != "dense":  # low ranks: the optimal plan never materialises anything W-sized
        assert C.plan_contraction(lay, 5).largest_intermediate < rows * cols


def test_flop_report():
    a, _ = _layer("dense", (16, 16), 1, ())
    assert C.flop_report([a], 4).speedup_ratio == 1.0
    t, _ = _layer("tt", (64, 64, 64, 64), 2, (32, 32, 32))  # cfg1
    r = C.flop_report({"cfg1": t}, 16)
    assert r.dense_flops == 2 * 4096 * 4096 * 16 and r.structured_flops < r.dense_flops
    # the device chain order is never better than the optimum
    assert r.structured_flops <= t.chain_flops_per_token() * 16


def test_relative_error_and_reshape_contracts():
    a = np.arange(1.0, 7.0).reshape(2, 3)
    assert C.relative_error(a, a) == 0.0
    with pytest.raises(ShapeError):
        C.relative_error(a, a.T)
    with pytest.raises(DegenerateReferenceError):
        C.relative_error(np.zeros(3), np.ones(3))
    with pytest.raises(NumericsError):
        C.relative_error(np.array([np.nan, 1.0]), np.ones(2))
    v = C.reshape_to_modes(np.zeros((12, 10)), (3, 4, 2, 5))
    assert v.shape == (3, 4, 2, 5)
    with pytest.raises(ShapeError):
        C.reshape_to_modes(np.zeros((12, 10)), (3, 4, 2, 6))
    with pytest.raises(ShapeError):
        C.reshape_to_modes(np.zeros((12, 10)), (120,))
    with pytest.raises(ShapeError):
        C.reshape_to_modes(np.zeros((2, 3, 4)), (6, 4))


def test_micro_benchmark_rejects_few_reps():
    lay, _ = _layer("dense", (4, 4), 1, ())
    with pytest.raises(ValueError):
        C.micro_benchmark(lay, None, reps=5)


@pytest.mark.gpu
def test_micro_benchmark_gpu():
    import torch

    lay, _ = _layer("tucker", (1024, 1024), 1, (64, 64))
    x = torch.randn(64, 1024, device="cuda").to(torch.bfloat16)
    r = C.micro_benchmark(lay, x, reps=10, warmup=2)
    assert r["median_ms"] > 0 and r["iqr_ms"] >= 0
