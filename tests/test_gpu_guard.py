"""Out-of-bounds store guard (B200 only; compute-sanitizer is unavailable on the pool): every plan
writes y into a strided view of a larger sentinel-filled buffer (row pitch padded past `rows`, plus a
tail after the last row); the padding must still hold the sentinel and the view must match the
oracle. Ragged row counts (not multiples of 8 / 64 / 128) exercise the tile tails."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2602_01613_b200 as tnl
from oracle import tn_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"
SENT = 12288.0  # 1.5 * 2^13: exactly representable in bf16 and fp32

CASES = [  # (family, mode_shape, rm, ranks): rows ragged vs the 64/128-row tiles
    ("tt", (10, 13, 8, 8), 2, (6, 5, 4)),          # rows 130
    ("tr", (7, 9, 8, 16), 2, (3, 4, 2, 3)),         # rows 63
    ("tucker", (6, 11, 8, 8), 2, (4, 5, 3, 6)),     # rows 66
    ("tucker", (200, 64), 1, (16, 16)),             # rows 200
    ("tt", (1, 8, 8), 1, (1, 4)),                   # rows 1
]


def _layer(spec, dtype):
    fam, ms, rm, ranks = spec
    L = O.synthetic_layer(fam, ms, rm, ranks, seed=94_000 + sum(ms))
    f = O.round_bf16 if dtype == torch.bfloat16 else (lambda a: np.asarray(a, np.float32).astype(np.float64))
    kw = dict(family=L.family, mode_shape=L.mode_shape, row_mode_count=L.row_mode_count)
    if fam == "tucker":
        kw.update(core=f(L.core), factors=[f(u) for u in L.factors])
    else:
        kw.update(cores=[f(c) for c in L.cores])
    return tnl.CompressedLayer(**kw), O.OracleLayer(**kw)


@pytest.mark.parametrize("spec", CASES, ids=[f"{c[0]}-{'x'.join(map(str, c[1]))}" for c in CASES])
@pytest.mark.parametrize("dtype,flags", [(torch.bfloat16, tnl.PLAN_AUTO), (torch.bfloat16, tnl.PLAN_CHAIN),
                                         (torch.bfloat16, tnl.PLAN_NO_DECODE), (torch.float32, tnl.PLAN_AUTO),
                                         (torch.float32, tnl.PLAN_GENERIC)],
                         ids=["bf16-auto", "bf16-chain", "bf16-nodecode", "fp32-auto", "fp32-generic"])
def test_no_store_outside_y(spec, dtype, flags):
    layer, ref = _layer(spec, dtype)
    rows, cols = ref.matrix_shape
    p = layer.plan(dtype, flags=flags)
    pad = 24
    for m in (1, 7, 64, 130):
        x = O.synthetic_x(m, cols, seed=94_500 + m)
        x = O.round_bf16(x) if dtype == torch.bfloat16 else x.astype(np.float32).astype(np.float64)
        big = torch.full((m + 2, rows + pad), SENT, dtype=dtype, device=DEV)
        out = big[:m, :rows]
        y = p.forward(torch.tensor(x, dtype=dtype, device=DEV), out=out)
        torch.cuda.synchronize()
        assert y.data_ptr() == out.data_ptr()
        b = big.float().cpu().numpy()
        assert np.all(b[:m, rows:] == SENT), (spec, flags, m, "row padding written")
        assert np.all(b[m:, :] == SENT), (spec, flags, m, "rows after the last token written")
        tol = 3e-2 if dtype == torch.bfloat16 else 1e-5
        e = float(np.linalg.norm(O.forward_torch_orient(ref, x) - b[:m, :rows]) /
                  np.linalg.norm(O.forward_torch_orient(ref, x)))
        assert e <= tol, (spec, flags, m, e)


def _stores_only_inside(run, m, rows, dtype=torch.bfloat16, pad=24):
    big = torch.full((m + 2, rows + pad), SENT, dtype=dtype, device=DEV)
    out = big[:m, :rows]
    run(out)
    torch.cuda.synchronize()
    b = big.float().cpu().numpy()
    assert np.all(b[:m, rows:] == SENT) and np.all(b[m:, :] == SENT)
    return b[:m, :rows]


@pytest.mark.parametrize("m", [1, 37, 64, 300])
def test_stack_and_mlp_store_only_inside(m):
    """The decode stack (fused boundary kernels) and the fused MLP block write only their y view."""
    from paper_2602_01613_b200.mlp import TNMLP
    from paper_2602_01613_b200.stack import TNStack

    specs = [("tucker", (1024, 1024), 1, (64, 64)), ("tr", (32, 32, 32, 32), 2, (4, 4, 4, 4)),
             ("tt", (32, 32, 32, 32), 2, (16, 16, 16))]
    layers = [_layer(s, torch.bfloat16)[0] for s in specs]
    st = TNStack(layers, torch.bfloat16)
    x = torch.randn(m, 1024, device=DEV).to(torch.bfloat16)
    ref = st.forward(x).float().cpu().numpy()
    got = _stores_only_inside(lambda out: st.forward(x, out=out), m, 1024)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-2
    g = O.synthetic_layer("tt", (32, 64, 32, 32), 2, (16, 16, 16), seed=94_900)
    u = O.synthetic_layer("tt", (32, 64, 32, 32), 2, (16, 16, 16), seed=94_901)
    d = O.synthetic_layer("tt", (32, 32, 32, 64), 2, (16, 16, 16), seed=94_902)
    mk = lambda L: tnl.CompressedLayer(L.family, L.mode_shape, L.row_mode_count, cores=[O.round_bf16(c) for c in L.cores])  # noqa: E731
    mlp = TNMLP(mk(g), mk(u), mk(d))
    ref = mlp(x).float().cpu().numpy()
    got = _stores_only_inside(lambda out: mlp.forward(x, out=out), m, 1024)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-2
