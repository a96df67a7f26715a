"""TNL_PLAN_CHAIN in bf16: the core-by-core chain on the tensor cores for every layer shape
(B200 only), against the float64 oracle on the same bf16-rounded cores and activations.

The chain contracts the input one core at a time, as the reference's reconstruct does
(tn_decompositions.py:351-361): TT/TR cores in order with the ring closure index carried,
Tucker factors one mode at a time around the core. Shapes with a fused chain kernel use it
(Tucker-2: tucker2_chain_kernel; a two-mode TT/TR input side: chain_in2_kernel); every other
step is a tcgen05 strided contraction step (tc_generic.cu). Intermediates are bf16, so the
tolerance allows one bf16 rounding per step on top of BF16_TOL.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2602_01613_b200 as tnl
from oracle import tn_oracle as O
from paper_2602_01613_b200 import qwen_stack as Q
from paper_2602_01613_b200 import synthetic as S

pytestmark = pytest.mark.gpu

BF16_TOL = 2e-2
CHAIN_TOL = 3e-2
DEV = "cuda"


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(a))


def oracle_of(layer):
    f = O.round_bf16
    kw = dict(family=layer.family, mode_shape=layer.mode_shape, row_mode_count=layer.row_mode_count)
    if layer.family == "tucker":
        kw.update(core=f(layer.core), factors=[f(u) for u in layer.factors])
    else:
        kw.update(cores=[f(c) for c in layer.cores])
    return O.OracleLayer(**kw)


def chain_check(layer, ms, seed, tol=CHAIN_TOL):
    p = layer.plan(torch.bfloat16, flags=tnl.PLAN_CHAIN)
    assert p.info["plan_large_name"] == "chain", p.info
    Lr = oracle_of(layer)
    rows, cols = Lr.matrix_shape
    errs = []
    for m in ms:
        x = O.round_bf16(O.synthetic_x(m, cols, seed + m))
        y = p.forward(torch.tensor(x, dtype=torch.bfloat16, device=DEV))
        torch.cuda.synchronize()
        e = rel(O.forward_torch_orient(Lr, x), y.double().cpu().numpy())
        assert e <= tol, (layer.family, layer.mode_shape, layer.row_mode_count, m, e)
        errs.append(e)
    return errs


def _layer(fam, ms, rm, ranks, seed):
    L = O.synthetic_layer(fam, ms, rm, ranks, seed=seed)
    kw = dict(family=L.family, mode_shape=L.mode_shape, row_mode_count=L.row_mode_count)
    if L.family == "tucker":
        kw.update(core=O.round_bf16(L.core), factors=[O.round_bf16(u) for u in L.factors])
    else:
        kw.update(cores=[O.round_bf16(c) for c in L.cores])
    return tnl.CompressedLayer(**kw)


@pytest.mark.parametrize("v", range(len(S.CFG2_VARIANTS)), ids=[v[0] for v in S.CFG2_VARIANTS])
def test_chain_cfg2_variants(v):
    _, fam, ms, rm, ranks = S.CFG2_VARIANTS[v]
    chain_check(_layer(fam, ms, rm, ranks, seed=70_000 + v), (1, 64, 300), seed=70_100)


@pytest.mark.parametrize("spec", [S.CFG3_GATE, S.CFG3_DOWN], ids=["gate", "down"])
def test_chain_cfg3_tt(spec):
    fam, ms, rm, ranks = spec
    chain_check(_layer(fam, ms, rm, ranks, seed=70_200), (1, 64, 300), seed=70_300)


CFG4 = [(f"{p} {k}", k, r, c) for k in ("tucker2-128", "tt64", "tr4", "tucker4")
        for p, r, c in (("gate/up", Q.FFN, Q.HIDDEN), ("down", Q.HIDDEN, Q.FFN))]


@pytest.mark.parametrize("variant", CFG4, ids=[v[0] for v in CFG4])
def test_chain_cfg4_variants(variant):
    name, kind, rows, cols = variant
    if kind == "tucker2-128":
        rows, cols = Q.KVDIM, Q.HIDDEN
    chain_check(Q._tn(kind, rows, cols, seed=70_400 + rows + cols), (1, 64, 300), seed=70_500)


# small shapes: every family, rm, ring/open, odd sizes and ranks, d = 2..5
SMALL = [  # cols % 8 == 0 (tensor-core plans)
    ("tt", (4, 6, 8), 1, (3, 4)), ("tt", (4, 6, 8), 2, (3, 4)), ("tr", (4, 6, 8), 1, (2, 3, 4)),
    ("tr", (4, 6, 8), 2, (2, 3, 4)), ("tt", (8, 8, 8, 8), 2, (5, 7, 6)), ("tr", (8, 8, 8, 8), 2, (3, 5, 2, 4)),
    ("tr", (8, 8, 8, 8), 1, (3, 5, 2, 4)), ("tr", (8, 8, 8, 8), 3, (3, 5, 2, 4)), ("tt", (4, 4, 4, 4, 4), 2, (3, 5, 4, 2)),
    ("tr", (4, 4, 4, 4, 4), 3, (2, 3, 4, 2, 3)), ("tucker", (6, 7, 8), 1, (3, 4, 2)), ("tucker", (6, 7, 8), 2, (3, 4, 2)),
    ("tucker", (8, 8, 8, 8), 2, (4, 3, 5, 2)), ("tucker", (4, 5, 6, 4, 8), 3, (2, 3, 4, 2, 3)),
    ("tt", (1, 8, 8), 1, (1, 4)), ("tr", (16, 32, 16, 32), 2, (4, 4, 4, 4)),
]


@pytest.mark.parametrize("spec", SMALL, ids=[f"{s[0]}-{s[1]}-rm{s[2]}" for s in SMALL])
def test_chain_small_shapes(spec):
    fam, ms, rm, ranks = spec
    chain_check(_layer(fam, ms, rm, ranks, seed=70_600 + sum(ms)), (1, 5, 37, 130), seed=70_700)


def test_chain_and_cut_agree_repeatedly():
    """The chain plan and the default cut plan agree on the same layer, call after call."""
    layer = _layer("tr", (64, 80, 64, 80), 2, (16, 16, 16, 16), seed=70_800)
    pc = layer.plan(torch.bfloat16, flags=tnl.PLAN_CHAIN)
    pa = layer.plan(torch.bfloat16)
    x = torch.randn(257, 5120, device=DEV).to(torch.bfloat16)
    ya = pa.forward(x).float()
    for _ in range(3):
        yc = pc.forward(x).float()
        torch.cuda.synchronize()
        assert float((yc - ya).norm() / ya.norm()) < CHAIN_TOL
