"""Pin the CPU oracle against the reference's own outputs (CPU-only).

The fixtures in tests/golden were produced by running the unmodified reference
(tests/golden/make_golden.py). These tests prove the oracle restates the
reference before any GPU result is compared against it.
"""

import math

import numpy as np
import pytest

from oracle import tn_oracle as O
from tnl_testutil import golden_layer_kwargs


def oracle_layer(rec, arrays):
    return O.OracleLayer(**golden_layer_kwargs(rec, arrays))


def test_forward_cases_match_reference(golden):
    index, arrays = golden
    assert len(index["forward"]) >= 27
    for rec in index["forward"]:
        L = oracle_layer(rec, arrays)
        x, y = arrays[rec["x"]], arrays[rec["y"]]
        # literal reference path and the chain restatement, both vs the reference's output
        assert O.relative_error(y, O.apply_reference(L, x)) <= 1e-13, rec["id"]
        assert O.relative_error(y, O.apply_chain(L, x)) <= 1e-12, rec["id"]
        if "w" in rec:
            assert O.relative_error(arrays[rec["w"]], O.reconstruct(L)) <= 1e-13
        assert O.param_count(L) == rec["param_count"] == rec["param_count_formula"]


def test_decomposition_cases_and_param_goldens(golden):
    index, arrays = golden
    seen = {}
    for rec in index["decomp"]:
        L = oracle_layer(rec, arrays)
        assert O.relative_error(arrays[rec["w"]], O.reconstruct(L)) <= 1e-13
        x, y = arrays[rec["x"]], arrays[rec["y"]]
        assert O.relative_error(y, O.apply_chain(L, x)) <= 1e-12
        assert O.param_count(L) == rec["param_count"]
        if rec["golden_param_count"] is not None:
            seen[rec["name"]] = O.param_count(L)
            assert O.param_count(L) == rec["golden_param_count"]
    # pkg/tests/test_tn_decompositions.py:159-180
    assert seen == {"tucker": 384, "tt": 320, "tr": 288}
    assert O.param_count_formula("tucker", (8, 8, 8, 8), (4, 4, 4, 4)) == 384
    assert O.param_count_formula("tt", (8, 8, 8, 8), (4, 4, 4)) == 320
    assert O.param_count_formula("tr", (8, 8, 8, 8), (3, 3, 3, 3)) == 288


def test_mode_shapes(golden):
    index, _ = golden
    for rec in index["mode_shapes"]:
        ms, rm = O.default_mode_shape(rec["rows"], rec["cols"])
        assert list(ms) == rec["mode_shape"] and rm == rec["row_mode_count"]
    # pkg/tests/test_tn_decompositions.py:38-49
    assert O.balanced_split(64) == (8, 8)
    assert O.balanced_split(128) == (8, 16)
    assert O.balanced_split(7) == (7,)
    assert O.default_mode_shape(5120, 5120) == ((64, 80, 64, 80), 2)
    assert O.default_mode_shape(25600, 5120) == ((160, 160, 64, 80), 2)


def test_cut_panels_reassociate_reconstruct(golden):
    index, arrays = golden
    for rec in index["forward"]:
        if rec["family"] == "dense":
            continue
        L = oracle_layer(rec, arrays)
        a, b = O.cut_panels(L)
        assert a.shape[1] == b.shape[0] == O.cut_rank(L)
        x, y = arrays[rec["x"]], arrays[rec["y"]]
        assert O.relative_error(y, a @ (b @ x)) <= 1e-12


def test_flop_formulas_match_survey():
    # chain flops per token at the BASELINE configs
    L = O.synthetic_layer("tt", (64, 64, 64, 64), 2, (32, 32, 32), seed=1)
    assert O.chain_flops_per_token(L) == 786_432
    for R, f in ((64, 1_318_912), (128, 2_654_208), (256, 5_373_952)):
        L = O.synthetic_layer("tucker", (5120, 5120), 1, (R, R), seed=2)
        assert O.chain_flops_per_token(L) == f
    for r, f in ((8, 1_458_176), (16, 6_422_528)):
        L = O.synthetic_layer("tr", (64, 80, 64, 80), 2, (r, r, r, r), seed=3)
        assert O.chain_flops_per_token(L) == f
    for r, f in ((32, 2_424_832), (64, 5_767_168)):
        L = O.synthetic_layer("tt", (160, 160, 64, 80), 2, (r, r, r), seed=4)
        assert O.chain_flops_per_token(L) == f


def test_tr_trace_restatement_large_closure(rng):
    # the alpha-by-alpha trace equals the reference's full-chain np.trace
    cores = [rng.standard_normal((3, 4, 2)), rng.standard_normal((2, 5, 4)), rng.standard_normal((4, 3, 3))]
    L = O.OracleLayer("tr", (4, 5, 3), 1, cores=cores)
    chain = cores[0]
    for c in cores[1:]:
        chain = np.tensordot(chain, c, axes=(chain.ndim - 1, 0))
    ref = np.trace(chain, axis1=0, axis2=chain.ndim - 1)
    assert O.relative_error(ref, O.reconstruct(L)) <= 1e-14


def test_synthetic_layers_preserve_variance():
    # SURVEY §8(d) init keeps Var(y) ~ Var(x) (avoids bf16 underflow)
    for fam, ms, rm, ranks in (
        ("tt", (64, 64, 64, 64), 2, (32, 32, 32)),
        ("tucker", (512, 512), 1, (64, 64)),
        ("tr", (16, 20, 16, 20), 2, (4, 4, 4, 4)),
    ):
        L = O.synthetic_layer(fam, ms, rm, ranks, seed=7)
        rows, cols = L.matrix_shape
        x = O.synthetic_x(32, cols, seed=8)
        y = O.forward_torch_orient(L, x)
        assert 0.3 < float(np.std(y)) < 3.0, (fam, float(np.std(y)))


def test_round_bf16_is_rne():
    v = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 0.0])
    r = O.round_bf16(v)
    assert r[0] == 1.0 and r[1] == 1.0  # tie -> even
    assert r[2] == 1.0078125
    assert abs(r[3] - (-3.140625)) < 1e-12
