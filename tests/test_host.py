"""Host-side logic on CPU: layer API validation, mode/rank arithmetic, no CPU fallback."""

import numpy as np
import pytest
import torch

import paper_2602_01613_b200 as tnl
from oracle import tn_oracle as O
from paper_2602_01613_b200 import modes
from tnl_testutil import golden_layer_kwargs


def test_layer_api_mirrors_reference_fields(golden):
    index, arrays = golden
    for rec in index["forward"] + index["decomp"]:
        kw = golden_layer_kwargs(rec, arrays)
        layer = tnl.CompressedLayer(**kw)
        assert layer.matrix_shape == O.OracleLayer(**kw).matrix_shape
        if rec["ranks"] is not None:
            assert list(layer.ranks) == rec["ranks"]
        assert tnl.param_count(layer) == rec["param_count"]
        assert tnl.compression_ratio(layer) == pytest.approx(rec["param_count"] / np.prod(rec["mode_shape"]))


def test_validation_messages_match_reference(rng):
    # tn_decompositions.py:97-126 — same exception type and wording
    with pytest.raises(tnl.ShapeError, match="row_mode_count 2 invalid for 2 modes"):
        tnl.CompressedLayer("tt", (4, 4), 2, cores=[rng.standard_normal((1, 4, 2)), rng.standard_normal((2, 4, 1))])
    with pytest.raises(tnl.ShapeError, match="tt boundary ranks must be 1"):
        tnl.CompressedLayer("tt", (4, 4), 1, cores=[rng.standard_normal((2, 4, 2)), rng.standard_normal((2, 4, 1))])
    with pytest.raises(tnl.ShapeError, match="tr closing bond mismatch"):
        tnl.CompressedLayer("tr", (4, 4), 1, cores=[rng.standard_normal((2, 4, 3)), rng.standard_normal((3, 4, 1))])
    with pytest.raises(tnl.ShapeError, match="chain bond mismatch"):
        tnl.CompressedLayer("tt", (4, 4, 4), 1, cores=[rng.standard_normal((1, 4, 2)), rng.standard_normal((3, 4, 2)),
                                                      rng.standard_normal((2, 4, 1))])
    with pytest.raises(tnl.ShapeError, match="tucker factor 1 has shape"):
        tnl.CompressedLayer("tucker", (4, 4), 1, core=np.ones((2, 2)), factors=[np.ones((4, 2)), np.ones((4, 3))])
    with pytest.raises(tnl.ShapeError, match="unknown family"):
        tnl.CompressedLayer("mpo", (4, 4), 1)
    with pytest.raises(tnl.ShapeError, match="dense layer must hold"):
        tnl.CompressedLayer("dense", (4, 4), 1, matrix=np.ones((3, 4)))


def test_no_cpu_fallback():
    L = O.synthetic_layer("tt", (4, 4, 4, 4), 2, (2, 2, 2), seed=1)
    layer = tnl.CompressedLayer("tt", L.mode_shape, 2, cores=L.cores)
    with pytest.raises(tnl.DeviceError):
        layer.forward(torch.randn(3, 16))
    if not torch.cuda.is_available():
        with pytest.raises(tnl.DeviceError):
            layer.plan(torch.bfloat16)


def test_modes_match_reference_goldens(golden):
    index, _ = golden
    for rec in index["mode_shapes"]:
        assert modes.default_mode_shape(rec["rows"], rec["cols"]) == (tuple(rec["mode_shape"]), rec["row_mode_count"])
    assert modes.param_count_formula("tucker", (8, 8, 8, 8), (4, 4, 4, 4)) == 384
    assert modes.param_count_formula("tt", (8, 8, 8, 8), (4, 4, 4)) == 320
    assert modes.param_count_formula("tr", (8, 8, 8, 8), (3, 3, 3, 3)) == 288
    for fam in ("tucker", "tt", "tr"):
        for shape in ((4, 4, 4), (2, 3, 4), (8, 8, 8, 8)):
            assert modes.maximal_ranks(fam, shape) == O.maximal_ranks(fam, shape)


def test_select_ranks_reference_cases():
    # pkg/tests/test_tn_decompositions.py:209-212, 223-238
    spec = modes.select_ranks((8, 8, 8, 8), "tt", modes.ParamBudget(320))
    assert isinstance(spec, modes.RankSpec) and spec.family == "tt" and spec.ranks == (4, 4, 4)
    r = modes.select_ranks((8, 8, 8, 8), "tucker", modes.ParamBudget(383)).ranks
    assert modes.param_count_formula("tucker", (8, 8, 8, 8), r) <= 383
    for i in range(4):
        t = list(r)
        t[i] += 1
        assert modes.param_count_formula("tucker", (8, 8, 8, 8), tuple(t)) > 383
    with pytest.raises(tnl.InfeasibleBudgetError):
        modes.select_ranks((8, 8, 8, 8), "tt", modes.ParamBudget(10))
    for fam in ("tucker", "tt", "tr"):
        assert modes.select_ranks((4, 4, 4), fam, modes.ParamBudget(64)).ranks == modes.maximal_ranks(fam, (4, 4, 4))
    # TR closure capped at 1 (tn_decompositions.py:416-417)
    assert modes.select_ranks((6, 8, 5, 8), "tr", modes.ParamBudget(600)).ranks[0] == 1
    assert modes.select_ranks((4, 4, 4), "tt", modes.FixedRank(16)).ranks == (4, 4)
    # RelativeError defers to the decomposition (tn_decompositions.py:462-463); dense has no ranks
    spec = modes.select_ranks((8, 8, 8, 8), "tr", modes.RelativeError(0.1))
    assert spec == modes.RankSpec(family="tr", ranks=None, rel_error=0.1)
    assert modes.select_ranks((4, 4), "dense", modes.FixedRank(2)) == modes.RankSpec("dense")
    with pytest.raises(tnl.RankError, match="unknown family"):
        modes.RankSpec("mpo")
    with pytest.raises(tnl.RankError, match="ranks must be >= 1"):
        modes.RankSpec("tt", ranks=(0, 2))


def test_flop_accounting_matches_oracle():
    for fam, ms, rm, ranks in (("tt", (64, 64, 64, 64), 2, (32, 32, 32)), ("tucker", (5120, 5120), 1, (256, 256)),
                               ("tr", (64, 80, 64, 80), 2, (16, 16, 16, 16)), ("tt", (160, 160, 64, 80), 2, (64, 64, 64))):
        L = O.synthetic_layer(fam, ms, rm, ranks, seed=3)
        layer = tnl.CompressedLayer(fam, ms, rm, core=L.core, factors=L.factors, cores=L.cores)
        assert layer.chain_flops_per_token() == O.chain_flops_per_token(L)
        assert layer.cut_rank == O.cut_rank(L)


def test_from_compressed_layer_adapter(golden):
    """a reference-shaped layer object (same fields as
    minima.tn_decompositions.CompressedLayer, tn_decompositions.py:66-80) converts 1:1."""
    from dataclasses import dataclass, field

    @dataclass
    class RefLayer:  # the reference dataclass's field set
        family: str
        mode_shape: tuple
        row_mode_count: int
        matrix: object = None
        core: object = None
        factors: list = field(default_factory=list)
        cores: list = field(default_factory=list)

    index, arrays = golden
    for rec in index["forward"]:
        kw = golden_layer_kwargs(rec, arrays)
        ref = RefLayer(**kw)
        layer = tnl.from_compressed_layer(ref)
        assert (layer.family, layer.mode_shape, layer.row_mode_count) == (ref.family, tuple(ref.mode_shape),
                                                                          ref.row_mode_count)
        assert layer.ranks == tnl.CompressedLayer(**kw).ranks
        assert tnl.param_count(layer) == O.param_count(O.OracleLayer(**kw))
    with pytest.raises(tnl.ShapeError):
        tnl.from_compressed_layer(RefLayer("tt", (4, 4), 1, cores=[np.zeros((1, 4, 2)), np.zeros((3, 4, 1))]))
