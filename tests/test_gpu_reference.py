"""GPU parity for the configurations and reference paths round 1 left untested (B200 only).

* layers made by the UNMODIFIED reference (`minima`, installed in baseline/_ref) through
  ``from_compressed_layer`` -> forward, against the reference's own ``layer_to_matrix(L) @ x``
  (tn_decompositions.py:364-365, sensitivity.py:154-160), and the INTEGRATION.md §2 binding run
  verbatim;
* size-1 modes (tn_decompositions.py:45-48: ``default_mode_shape(1, 64) == ((1, 8, 8), 1)``);
* core mutation / replacement (the reference re-reads its arrays on every call, :346-361);
* caller-supplied ``out`` validation;
* ragged output widths (N % 256 in {64, 128, 192}) on the CTA-pair and persistent GEMMs;
* cfg2 fp32 at M = 16 for all seven variants ("+fp32 parity at M=16");
* every cfg4 projection variant at its real Qwen3-32B shape, M in {1, 64, 300};
* a short QwenTNStack (every MLP family) against a float64 restatement of the decoder step.

Tolerances (BASELINE north_star): fp32 rel-err <= 1e-5 vs float64; bf16 rel-err <= 2e-2 vs the
float64 oracle on the same bf16-rounded cores and activations.
"""

import os
import re
import sys
import types

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2602_01613_b200 as tnl
from oracle import tn_oracle as O
from paper_2602_01613_b200 import qwen_stack as Q

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 2e-2
DEV = "cuda"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(a))


def oracle_of(layer: tnl.CompressedLayer, bf16: bool) -> O.OracleLayer:
    f = O.round_bf16 if bf16 else (lambda a: np.asarray(a, dtype=np.float64))
    kw = dict(family=layer.family, mode_shape=layer.mode_shape, row_mode_count=layer.row_mode_count)
    if layer.family == "tucker":
        kw.update(core=f(layer.core), factors=[f(u) for u in layer.factors])
    elif layer.family in ("tt", "tr"):
        kw.update(cores=[f(c) for c in layer.cores])
    else:
        kw.update(matrix=f(layer.matrix))
    return O.OracleLayer(**kw)


def fwd(layer, x64, dtype, flags=tnl.PLAN_AUTO):
    y = layer.plan(dtype, flags=flags).forward(torch.tensor(x64, dtype=dtype, device=DEV))
    torch.cuda.synchronize()
    return y.double().cpu().numpy()


# --- the unmodified reference -------------------------------------------------------------


def _ref_layers(minima):
    T, TC = minima.tn_decompositions, minima.tensor_core
    rng = np.random.default_rng(20240811)
    t8 = rng.standard_normal((8, 8, 8, 8))
    out = [T.tucker_decompose(t8, (4, 3, 4, 2)), T.tt_decompose(t8, [TC.FixedRank(4)] * 3),
           T.tr_decompose(t8, (2, 3, 4, 2)), T.tt_decompose(rng.standard_normal((16, 16, 16, 16)), [TC.FixedRank(8)] * 3)]
    for L in out:
        L.row_mode_count = 2
    out += [T.compress_matrix(rng.standard_normal((64, 48)), "tucker", TC.FixedRank(5)),
            T.compress_matrix(rng.standard_normal((16, 20)), "tr", TC.ParamBudget(300)),
            T.compress_matrix(rng.standard_normal((256, 128)), "tt", TC.ParamBudget(4000))]
    return out


def test_real_reference_layers_forward(minima):
    """from_compressed_layer(real minima layer) -> forward == minima.layer_to_matrix(L) @ x."""
    T = minima.tn_decompositions
    for i, ref in enumerate(_ref_layers(minima)):
        layer = tnl.from_compressed_layer(ref)
        rows, cols = ref.matrix_shape
        for m in (1, 16, 130):
            x = np.random.default_rng(100 + i).standard_normal((cols, m))  # reference orientation
            y_ref = T.layer_to_matrix(ref) @ x  # the reference's own forward (sensitivity.py:156)
            x32 = x.astype(np.float32).astype(np.float64)
            y_ref32 = T.layer_to_matrix(ref) @ x32
            got = tnl.apply_compressed(layer, torch.tensor(x32, dtype=torch.float32, device=DEV))
            assert rel(y_ref32, got.double().cpu().numpy()) <= FP32_TOL, (ref.family, m)
            xb = O.round_bf16(x.T)
            yb = fwd(layer, xb, torch.bfloat16)
            ref_b = O.forward_torch_orient(oracle_of(layer, bf16=True), xb)
            assert rel(ref_b, yb) <= BF16_TOL, (ref.family, m)
            assert rel(y_ref.T, yb) <= 5e-2  # bf16 cores + activations vs the exact float64 result
        w = tnl.layer_to_matrix(layer).double().cpu().numpy()
        assert rel(T.layer_to_matrix(ref), w) <= 1e-6


def _load_integration_stub():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 2."):text.index("## 3.")]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    mod = types.ModuleType("minima_structured_inference")
    os.environ["TNL_LIBRARY"] = tnl._native.lib_path()
    exec(compile(code, "INTEGRATION.md#2", "exec"), mod.__dict__)
    return mod


def test_integration_stub_runs(minima):
    """The reference-side ctypes binding of INTEGRATION.md §2, executed verbatim."""
    T = minima.tn_decompositions
    stub = _load_integration_stub()
    for i, ref in enumerate(_ref_layers(minima)):
        rows, cols = ref.matrix_shape
        x = np.random.default_rng(200 + i).standard_normal((cols, 9))
        y = stub.apply_compressed(ref, x)
        x32 = x.astype(np.float32).astype(np.float64)
        assert y.shape == (rows, 9)
        assert rel(T.layer_to_matrix(ref) @ x32, y) <= FP32_TOL
    # the stub re-plans when the reference layer's arrays change in place
    ref = _ref_layers(minima)[1]
    x = np.random.default_rng(7).standard_normal((ref.matrix_shape[1], 3))
    stub.apply_compressed(ref, x)
    ref.cores[1] *= 2.0
    assert rel(T.layer_to_matrix(ref) @ x, stub.apply_compressed(ref, x)) <= FP32_TOL
    with pytest.raises(minima.errors.ShapeError):
        stub.apply_compressed(ref, np.ones((ref.matrix_shape[1] + 1, 2)))


# --- size-1 modes -----------------------------------------------------------------------


@pytest.mark.parametrize("spec", [
    ("tt", (1, 8, 8), 1, (1, 4)), ("tucker", (1, 8, 8), 1, (1, 4, 4)), ("tr", (1, 8, 8), 1, (2, 2, 2)),
    ("tt", (4, 1, 4, 16), 2, (4, 4, 4)), ("tr", (8, 1, 1, 64), 2, (2, 2, 2, 2)), ("tucker", (16, 1, 1, 32), 2, (4, 1, 1, 8)),
    ("tt", (64, 1), 1, (1,)), ("tr", (32, 1), 1, (3, 3)),
])
def test_size_one_modes(spec):
    fam, ms, rm, ranks = spec
    L = O.synthetic_layer(fam, ms, rm, ranks, seed=61_000)
    kw = dict(family=fam, mode_shape=ms, row_mode_count=rm, core=L.core, factors=L.factors, cores=L.cores)
    layer = tnl.CompressedLayer(**kw)
    rows, cols = layer.matrix_shape
    for m in (1, 5, 200):
        x = O.synthetic_x(m, cols, seed=61_001).astype(np.float32).astype(np.float64)
        ref = O.forward_torch_orient(O.OracleLayer(**kw), x)
        assert rel(ref, fwd(layer, x, torch.float32)) <= FP32_TOL, (spec, m)
        xb = O.round_bf16(x)
        assert rel(O.forward_torch_orient(oracle_of(layer, True), xb), fwd(layer, xb, torch.bfloat16)) <= BF16_TOL
    w = tnl.reconstruct(layer).double().cpu().numpy()
    assert w.shape == ms and rel(O.reconstruct(O.OracleLayer(**kw)), w) <= 1e-6


# --- mutation / replacement of the payload -------------------------------------------------


def test_core_mutation_is_seen_by_reconstruct_and_forward():
    L = O.synthetic_layer("tr", (8, 16, 8, 16), 2, (4, 4, 4, 4), seed=62_000)
    cores = [c.copy() for c in L.cores]
    layer = tnl.CompressedLayer("tr", L.mode_shape, 2, cores=cores)
    x = O.synthetic_x(16, 128, seed=62_001).astype(np.float32).astype(np.float64)
    xt = torch.tensor(x, dtype=torch.float32, device=DEV)
    w0 = tnl.layer_to_matrix(layer).double().cpu().numpy()
    layer.forward(xt)
    # in-place numpy write: the reference-API functions re-read (crc32), forward(check_cores=True) too
    cores[2] *= -3.0
    ref = O.OracleLayer("tr", L.mode_shape, 2, cores=cores)
    w1 = tnl.layer_to_matrix(layer).double().cpu().numpy()
    assert rel(O.layer_to_matrix(ref), w1) <= 1e-6 and rel(w0, w1) > 0.5
    y = layer.forward(xt, check_cores=True).double().cpu().numpy()
    assert rel(O.forward_torch_orient(ref, x), y) <= FP32_TOL
    # replacing a core re-plans with no explicit invalidate()
    layer.cores[0] = cores[0] * 0.5
    ref = O.OracleLayer("tr", L.mode_shape, 2, cores=list(layer.cores))
    y = layer.forward(xt).double().cpu().numpy()
    assert rel(O.forward_torch_orient(ref, x), y) <= FP32_TOL
    # torch cores written in place (version counter)
    tl = tnl.CompressedLayer("tr", L.mode_shape, 2, cores=[torch.tensor(c, dtype=torch.float32) for c in L.cores])
    tl.forward(xt)
    tl.cores[1].mul_(2.0)
    ref = O.OracleLayer("tr", L.mode_shape, 2, cores=[c.double().numpy() for c in tl.cores])
    assert rel(O.forward_torch_orient(ref, x), tl.forward(xt).double().cpu().numpy()) <= FP32_TOL
    # apply_compressed (reference orientation) re-reads as well
    cores[3][:] = 0.25 * cores[3]
    ref = O.OracleLayer("tr", L.mode_shape, 2, cores=list(layer.cores))
    got = tnl.apply_compressed(layer, xt.t().contiguous()).double().cpu().numpy()
    assert rel(O.apply_reference(ref, x.T), got) <= FP32_TOL


def test_out_validation():
    L = O.synthetic_layer("tucker", (256, 512), 1, (32, 32), seed=63_000)
    layer = tnl.CompressedLayer("tucker", (256, 512), 1, core=L.core, factors=L.factors)
    p = layer.plan(torch.bfloat16)
    x = torch.randn(8, 512, device=DEV, dtype=torch.bfloat16)
    for bad in (torch.empty(8, 255, device=DEV, dtype=torch.bfloat16),       # too narrow
                torch.empty(8, 256, device=DEV, dtype=torch.float32),        # wrong dtype
                torch.empty(256, 8, device=DEV, dtype=torch.bfloat16).t(),   # transposed view
                torch.empty(8, 256, dtype=torch.bfloat16)):                  # host tensor
        with pytest.raises(tnl.ShapeError):
            p.forward(x, out=bad)
    ok = torch.empty(8, 320, device=DEV, dtype=torch.bfloat16)[:, :256]  # padded row pitch is fine
    p.forward(x, out=ok)
    torch.cuda.synchronize()
    assert torch.equal(ok, p.forward(x))


# --- ragged output widths (ADVICE: staging-ring reuse on dead chunks) --------------------------


@pytest.mark.parametrize("rows", [4160, 4224, 4288, 3200])
@pytest.mark.parametrize("m", [200, 300, 4096])
def test_ragged_output_width(rows, m):
    """N % 256 in {64, 128, 192}: the last 256-wide output tile has dead 64-column chunks. M = 200
    runs the persistent GEMM, M >= 256 the CTA-pair GEMM; M = 4096 keeps many stores in flight."""
    L = O.synthetic_layer("tucker", (rows, 1024), 1, (64, 64), seed=64_000 + rows)
    layer = tnl.CompressedLayer("tucker", (rows, 1024), 1, core=L.core, factors=L.factors)
    x = O.round_bf16(O.synthetic_x(m, 1024, seed=64_001))
    y = fwd(layer, x, torch.bfloat16)
    assert rel(O.forward_torch_orient(oracle_of(layer, True), x), y) <= BF16_TOL
    # the same width as an output-mode shard of the 25600-row gate layer (8-way: 3200 rows)
    if rows == 3200:
        G = Q._tn("tt64", 25600, 5120, seed=64_100)
        xs = O.round_bf16(O.synthetic_x(m, 5120, seed=64_101))
        p = G.plan(torch.bfloat16, row_range=(3200, 6400))
        ys = p.forward(torch.tensor(xs, dtype=torch.bfloat16, device=DEV)).double().cpu().numpy()
        full = O.forward_torch_orient(oracle_of(G, True), xs)
        assert rel(full[:, 3200:6400], ys) <= BF16_TOL


# --- cfg2 fp32 at M = 16 (all seven variants) ------------------------------------------------


@pytest.mark.parametrize("variant", range(7))
def test_cfg2_fp32_m16(variant):
    from paper_2602_01613_b200 import synthetic as S

    name, fam, ms, rm, ranks = S.CFG2_VARIANTS[variant]
    layer = S.make_layer(fam, ms, rm, ranks, seed=20_000 + 100 * variant)
    x = S.make_x(16, 5120, seed=20_000 + 9_999).astype(np.float64)
    ref = O.forward_torch_orient(oracle_of(layer, bf16=False), x)
    for flags in (tnl.PLAN_AUTO, tnl.PLAN_GENERIC):
        assert rel(ref, fwd(layer, x, torch.float32, flags)) <= FP32_TOL, (name, flags)


# --- cfg4: every projection variant at its real shape -------------------------------------------

CFG4_VARIANTS = [
    ("q tucker2-256", "tucker2-256", Q.QDIM, Q.HIDDEN), ("k/v tucker2-128", "tucker2-128", Q.KVDIM, Q.HIDDEN),
    ("o tucker2-256", "tucker2-256", Q.HIDDEN, Q.QDIM),
] + [(f"{p} {k}", k, r, c) for k in ("tucker2-256", "tt64", "tr4", "tucker4")
     for p, r, c in (("gate/up", Q.FFN, Q.HIDDEN), ("down", Q.HIDDEN, Q.FFN))]


@pytest.mark.parametrize("variant", CFG4_VARIANTS, ids=[v[0] for v in CFG4_VARIANTS])
def test_cfg4_projection_variants(variant):
    name, kind, rows, cols = variant
    layer = Q._tn(kind, rows, cols, seed=65_000 + rows + cols)
    Lr = oracle_of(layer, bf16=True)
    for m in (1, 64, 300):
        x = O.round_bf16(O.synthetic_x(m, cols, seed=65_100 + m))
        y = fwd(layer, x, torch.bfloat16)
        assert rel(O.forward_torch_orient(Lr, x), y) <= BF16_TOL, (name, m)


# --- a short Qwen3 stack against a float64 restatement ---------------------------------------


def _rms(x, eps=1e-6):
    return x / np.sqrt(np.mean(x * x, axis=1, keepdims=True) + eps)


def _silu(g):
    return g / (1.0 + np.exp(-g))


def _stack_oracle(st, x):
    """Qwen3 pre-norm decoder step, attention core a pass-through (qwen_stack.py docstring):
    h = rms(x); x += Lo(Lq(h)); h = rms(x); x += Ld(silu(Lg(h)) * Lu(h)). float64 arithmetic on
    the bf16-rounded cores; activations re-rounded to bf16 where the device stores them."""
    R = O.round_bf16
    for blk in st.layers:
        lay = {n: oracle_of(blk[n][1], bf16=True) for n in ("q", "o", "gate", "up", "down")}
        h = R(_rms(x))
        q = R(O.forward_torch_orient(lay["q"], h))
        x = R(x + R(O.forward_torch_orient(lay["o"], q)))
        h = R(_rms(x))
        hh = R(_silu(O.forward_torch_orient(lay["gate"], h)) * O.forward_torch_orient(lay["up"], h))
        x = R(x + R(O.forward_torch_orient(lay["down"], hh)))
    return x


@pytest.mark.parametrize("m", [1, 64, 300])
def test_qwen_stack_matches_oracle(m):
    st = Q.QwenTNStack(n_layers=4, seed=66_000, mlp_kinds=["tt64", "tr4", "tucker4", "tucker2-256"])
    x0 = O.round_bf16(O.synthetic_x(m, Q.HIDDEN, seed=66_100))
    xt = torch.tensor(x0, dtype=torch.bfloat16, device=DEV)
    st.forward(xt)
    torch.cuda.synchronize()
    got = xt.double().cpu().numpy()
    ref = _stack_oracle(st, x0)
    assert np.isfinite(got).all()
    assert rel(ref, got) <= BF16_TOL
    assert rel(ref - x0, got - x0) <= 2 * BF16_TOL  # the four layers' contribution itself


# --- the fused Tucker-2 chain (N2: U1 -> G -> U0 in one kernel, T1/T2 on chip) ------------------


@pytest.mark.parametrize("shape", [(5120, 5120, 64), (5120, 5120, 128), (5120, 5120, 256), (8192, 5120, 256),
                                   (1024, 5120, 128), (25600, 5120, 256), (5120, 25600, 256), (4160, 1024, 128),
                                   (5120, 8192, 192)])
@pytest.mark.parametrize("m", [65, 300, 4096])
def test_tucker2_fused_chain(shape, m):
    """TNL_PLAN_CHAIN on Tucker-2 at prefill sizes runs tucker2_chain_kernel (one launch): against
    the oracle on the same bf16 values, and against the merged-cut plan."""
    rows, cols, R = shape
    L = O.synthetic_layer("tucker", (rows, cols), 1, (R, R), seed=67_000 + rows + R)
    layer, Lr = tnl.CompressedLayer("tucker", (rows, cols), 1, core=O.round_bf16(L.core),
                                    factors=[O.round_bf16(u) for u in L.factors]), None
    x = O.round_bf16(O.synthetic_x(m, cols, seed=67_100 + m))
    p = layer.plan(torch.bfloat16, flags=tnl.PLAN_CHAIN)
    assert p.info["plan_large_name"] == "chain"
    tnl.launch_count(reset=True)
    y = p.forward(torch.tensor(x, dtype=torch.bfloat16, device=DEV))
    torch.cuda.synchronize()
    n_launch = tnl.launch_count(reset=True)
    if R in (64, 128, 256):
        assert n_launch == 1  # the whole chain is one kernel
    else:  # R = 192: outside the fused kernel's shapes -> the three-launch chain
        assert n_launch >= 3
    ref = O.forward_torch_orient(oracle_of(layer, bf16=True), x)
    got = y.double().cpu().numpy()
    assert rel(ref, got) <= BF16_TOL
    cut = fwd(layer, x, torch.bfloat16, tnl.PLAN_CUT)
    assert rel(cut, got) <= BF16_TOL


# --- shared-input group (tnl_group_*: k, v, q of one hidden state) ------------------------------


@pytest.mark.parametrize("m", [16, 300, 8192])
def test_group_matches_separate_forwards(m):
    """One stacked first step over x for k, v, q (prefill) == each layer's own forward, with and
    without the folded RMSNorm row scale; decode-sized M runs the layers one by one."""
    import ctypes

    from paper_2602_01613_b200 import _native as N
    from paper_2602_01613_b200.stack import TNGroup

    lays = [Q._tn("tucker2-128", Q.KVDIM, Q.HIDDEN, seed=68_001), Q._tn("tucker2-128", Q.KVDIM, Q.HIDDEN, seed=68_002),
            Q._tn("tucker2-256", Q.QDIM, Q.HIDDEN, seed=68_003)]
    g = TNGroup(lays)
    x = torch.randn(m, Q.HIDDEN, device=DEV).to(torch.bfloat16)
    ys = g.forward(x)
    for lay, y in zip(lays, ys):
        ref = lay.plan(torch.bfloat16).forward(x)
        torch.cuda.synchronize()
        assert rel(ref.double().cpu().numpy(), y.double().cpu().numpy()) <= 1e-2
        assert rel(O.forward_torch_orient(oracle_of(lay, True), x.double().cpu().numpy()),
                   y.double().cpu().numpy()) <= BF16_TOL
    if m > 64:  # folded RMSNorm: y_i = layer_i(x / rms(x))
        lib = N.load()
        ss = torch.zeros(m, dtype=torch.float32, device=DEV)
        st = torch.cuda.current_stream().cuda_stream
        N.check(lib.tnl_rms_stats(ctypes.c_void_p(x.data_ptr()), Q.HIDDEN, m, Q.HIDDEN, ctypes.c_void_p(ss.data_ptr()),
                                  ctypes.c_void_p(st)))
        opts = N.FwdOpts(0, ss.data_ptr(), Q.HIDDEN, 1e-6)
        ys = g.forward(x, opts=opts)
        xn = (x.float() * torch.rsqrt(x.float().pow(2).mean(-1, keepdim=True) + 1e-6)).double().cpu().numpy()
        torch.cuda.synchronize()
        for lay, y in zip(lays, ys):
            assert rel(O.forward_torch_orient(oracle_of(lay, True), xn), y.double().cpu().numpy()) <= BF16_TOL


@pytest.mark.parametrize("m,n", [(1, 8), (7, 5120), (8192, 5120), (300, 25600), (13, 1032)])
def test_rms_stats(m, n):
    """tnl_rms_stats (warp per row) against float64 sums of squares of the same bf16 values."""
    import ctypes

    from paper_2602_01613_b200 import _native as N

    x = torch.randn(m, n + 8, device=DEV).to(torch.bfloat16)[:, :n]  # padded row pitch
    ss = torch.full((m,), -1.0, dtype=torch.float32, device=DEV)
    N.check(N.load().tnl_rms_stats(ctypes.c_void_p(x.data_ptr()), n + 8, m, n, ctypes.c_void_p(ss.data_ptr()),
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    torch.cuda.synchronize()
    ref = (x.double() ** 2).sum(-1).cpu().numpy()
    assert np.max(np.abs(ss.double().cpu().numpy() - ref) / ref) <= 1e-5


@pytest.mark.parametrize("kind", ["tt64", "tr4", "tucker4", "tucker2-256"])
def test_rms_fused_matches_stats_pass(kind):
    """rms_fused (the stacked input steps sum the squares of x while streaming it) == the separate
    statistics pass + ss_in, for the k/v/q group and every cfg4 MLP kind, at M = 8192."""
    import ctypes

    from paper_2602_01613_b200 import _native as N
    from paper_2602_01613_b200.mlp import TNMLP
    from paper_2602_01613_b200.stack import TNGroup

    lib = N.load()
    m = 8192
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    x = torch.randn(m, Q.HIDDEN, device=DEV).to(torch.bfloat16)
    ss = torch.zeros(m, dtype=torch.float32, device=DEV)
    N.check(lib.tnl_rms_stats(ctypes.c_void_p(x.data_ptr()), Q.HIDDEN, m, Q.HIDDEN, ctypes.c_void_p(ss.data_ptr()), st))
    o_stats, o_fused = N.FwdOpts(0, ss.data_ptr(), Q.HIDDEN, 1e-6), N.FwdOpts(0, None, Q.HIDDEN, 1e-6, 1)
    if kind == "tt64":  # the group once is enough
        g = TNGroup([Q._tn("tucker2-128", Q.KVDIM, Q.HIDDEN, seed=69_001), Q._tn("tucker2-256", Q.QDIM, Q.HIDDEN, seed=69_002)])
        a = g.forward(x, opts=o_stats)
        b = g.forward(x, opts=o_fused)
        torch.cuda.synchronize()
        for ya, yb in zip(a, b):
            assert rel(ya.double().cpu().numpy(), yb.double().cpu().numpy()) <= 5e-3
    lays = [Q._tn(kind, r, c, seed=69_100 + i) for i, (r, c) in enumerate(((Q.FFN, Q.HIDDEN), (Q.FFN, Q.HIDDEN),
                                                                             (Q.HIDDEN, Q.FFN)))]
    blk = TNMLP(*lays)
    ws = blk.workspace(m)
    ya = torch.zeros(m, Q.HIDDEN, device=DEV, dtype=torch.bfloat16)
    yb = torch.zeros(m, Q.HIDDEN, device=DEV, dtype=torch.bfloat16)
    for y, o in ((ya, o_stats), (yb, o_fused)):
        N.check(lib.tnl_mlp_forward_ex(blk.handle, ctypes.c_void_p(x.data_ptr()), m, Q.HIDDEN, ctypes.c_void_p(y.data_ptr()),
                                       Q.HIDDEN, ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.byref(o), st))
    torch.cuda.synchronize()
    assert torch.isfinite(yb.float()).all()
    assert rel(ya.double().cpu().numpy(), yb.double().cpu().numpy()) <= 5e-3
