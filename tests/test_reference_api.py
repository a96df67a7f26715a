"""The layer API against the UNMODIFIED reference package (CPU; skipped when it is not installed).

The reference (`minima`, /root/reference/pkg/src, installed into baseline/_ref) is imported as is:
its rank planner and its own decompositions produce the layers; this package must agree on every
bookkeeping answer (RankSpec, ranks, matrix shapes, parameter counts) and accept its layers through
``from_compressed_layer`` with the same validation.
"""

import itertools

import numpy as np
import pytest

import paper_2602_01613_b200 as tnl
from oracle import tn_oracle as O
from paper_2602_01613_b200 import modes

SHAPES = [(8, 8, 8, 8), (4, 4, 4), (6, 8, 5, 8), (2, 3, 4), (16, 16), (6, 6, 6), (1, 8, 8), (5, 7)]


def _ref_spec(minima, shape, family, target):
    T = minima.tn_decompositions
    try:
        s = T.select_ranks(shape, family, target)
        return ("ok", s.family, s.ranks, s.rel_error)
    except Exception as e:  # noqa: BLE001 — compare exception class names too
        return ("err", type(e).__name__)


def _our_spec(shape, family, target):
    try:
        s = modes.select_ranks(shape, family, target)
        return ("ok", s.family, s.ranks, s.rel_error)
    except Exception as e:  # noqa: BLE001
        return ("err", type(e).__name__)


def test_select_ranks_matches_reference_everywhere(minima):
    """tn_decompositions.py:445-510 — same RankSpec (or the same exception) for every family x
    shape x target in a grid of FixedRank / ParamBudget / RelativeError targets."""
    TC = minima.tensor_core
    n = 0
    for shape, family in itertools.product(SHAPES, ("tucker", "tt", "tr", "dense")):
        dense = int(np.prod(shape))
        budgets = sorted({1, 2, 10, 64, 100, 320, 383, 600, dense - 1, dense, dense + 5} - {0})
        targets = [(TC.ParamBudget(b), modes.ParamBudget(b)) for b in budgets if b >= 1]
        targets += [(TC.FixedRank(r), modes.FixedRank(r)) for r in (1, 2, 3, 4, 7, 16)]
        targets += [(TC.RelativeError(e), modes.RelativeError(e)) for e in (0.05, 0.5, 1.0)]
        for ref_t, our_t in targets:
            assert _our_spec(shape, family, our_t) == _ref_spec(minima, shape, family, ref_t), (shape, family, ref_t)
            n += 1
    assert n > 500


def _reference_layers(minima):
    """Layers made by the reference's own decompositions (not by this repo's generator)."""
    T = minima.tn_decompositions
    TC = minima.tensor_core
    rng = np.random.default_rng(20240811)
    t8 = rng.standard_normal((8, 8, 8, 8))
    out = [
        T.tucker_decompose(t8, (4, 3, 4, 2)),
        T.tt_decompose(t8, [TC.FixedRank(4)] * 3),
        T.tr_decompose(t8, (2, 3, 4, 2)),
        T.compress_matrix(rng.standard_normal((12, 10)), "tt", TC.ParamBudget(10**9)),
        T.compress_matrix(rng.standard_normal((64, 48)), "tucker", TC.FixedRank(5)),
        T.compress_matrix(rng.standard_normal((16, 20)), "tr", TC.ParamBudget(300)),
    ]
    for L in out[:3]:
        L.row_mode_count = 2  # decompose() sets it after construction as well (:549)
    return out


def test_from_real_compressed_layer_bookkeeping(minima):
    T = minima.tn_decompositions
    for ref in _reference_layers(minima):
        ours = tnl.from_compressed_layer(ref)
        assert ours.family == ref.family
        assert ours.mode_shape == tuple(ref.mode_shape)
        assert ours.matrix_shape == tuple(ref.matrix_shape)
        assert (ours.ranks is None and ref.ranks is None) or tuple(ours.ranks) == tuple(ref.ranks)
        assert tnl.param_count(ours) == T.param_count(ref)
        assert tnl.compression_ratio(ours) == pytest.approx(T.compression_ratio(ref))
        # arrays are taken by reference, as the reference stores them (:66-80)
        arrs = [ref.core] + list(ref.factors) if ref.family == "tucker" else list(ref.cores)
        mine = [ours.core] + list(ours.factors) if ours.family == "tucker" else list(ours.cores)
        assert all(a is b for a, b in zip(arrs, mine))
        # the oracle restatement reproduces the reference's dense matrix (parity anchor of the GPU tests)
        kw = dict(family=ref.family, mode_shape=tuple(ref.mode_shape), row_mode_count=ref.row_mode_count,
                  core=getattr(ref, "core", None), factors=list(ref.factors or []), cores=list(ref.cores or []))
        np.testing.assert_allclose(O.layer_to_matrix(O.OracleLayer(**kw)), T.layer_to_matrix(ref), rtol=0, atol=1e-12)


def test_validation_agrees_with_reference(minima):
    """Invalid layers: both constructors raise the same exception class with the same message."""
    T = minima.tn_decompositions
    rng = np.random.default_rng(5)
    cases = [
        dict(family="tt", mode_shape=(4, 4), row_mode_count=2, cores=[rng.standard_normal((1, 4, 2)), rng.standard_normal((2, 4, 1))]),
        dict(family="tt", mode_shape=(4, 4), row_mode_count=1, cores=[rng.standard_normal((2, 4, 2)), rng.standard_normal((2, 4, 1))]),
        dict(family="tr", mode_shape=(4, 4), row_mode_count=1, cores=[rng.standard_normal((2, 4, 3)), rng.standard_normal((3, 4, 1))]),
        dict(family="tucker", mode_shape=(4, 4), row_mode_count=1, core=np.ones((2, 2)), factors=[np.ones((4, 2)), np.ones((4, 3))]),
        dict(family="tt", mode_shape=(4, 4, 4), row_mode_count=1,
             cores=[rng.standard_normal((1, 4, 2)), rng.standard_normal((3, 4, 2)), rng.standard_normal((2, 4, 1))]),
        dict(family="dense", mode_shape=(4, 4), row_mode_count=1, matrix=np.ones((3, 4))),
    ]
    for kw in cases:
        with pytest.raises(Exception) as ref_exc:
            T.CompressedLayer(**kw)
        with pytest.raises(Exception) as our_exc:
            tnl.CompressedLayer(**kw)
        assert type(our_exc.value).__name__ == type(ref_exc.value).__name__
        assert str(our_exc.value) == str(ref_exc.value)


def test_size_one_modes_bookkeeping(minima):
    """default_mode_shape(1, 64) == ((1, 8, 8), 1) in both (tn_decompositions.py:45-63)."""
    T = minima.tn_decompositions
    for rows, cols in ((1, 64), (64, 1), (1, 1), (7, 64), (13, 1024), (2, 3)):
        assert modes.default_mode_shape(rows, cols) == T.default_mode_shape(rows, cols)
    assert modes.default_mode_shape(1, 64) == ((1, 8, 8), 1)


def test_plan_identity_tracks_core_replacement_and_writes():
    """The plan cache key follows the payload: replacing a core or the factor list changes the
    identity; an in-place numpy write changes the content digest (tn_decompositions.py:346-361
    re-reads the arrays on every call)."""
    L = O.synthetic_layer("tt", (4, 4, 4, 4), 2, (2, 2, 2), seed=1)
    layer = tnl.CompressedLayer("tt", L.mode_shape, 2, cores=list(L.cores))
    a = layer._identity()
    assert layer._identity() == a
    layer.cores[1] = layer.cores[1].copy()
    assert layer._identity() != a
    b = layer._identity()
    layer.row_mode_count = 1
    assert layer._identity() != b
    layer.row_mode_count = 2
    d0 = tuple(tnl.layer._array_digest(x) for x in layer._payload())
    layer.cores[2][0, 0, 0] += 1.0
    assert tuple(tnl.layer._array_digest(x) for x in layer._payload()) != d0
    torch = pytest.importorskip("torch")
    t = torch.ones(3, 4)
    k0 = tnl.layer._array_token(t)
    t.mul_(2.0)  # in-place write bumps the tensor's version counter
    assert tnl.layer._array_token(t) != k0
