"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle (B200 only).

Tolerances (BASELINE north_star): fp32 path rel-err <= 1e-5 against the
float64 oracle; bf16 path rel-err <= 2e-2 against the float64 oracle evaluated
on the same bf16-rounded cores and activations.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2602_01613_b200 as tnl
from oracle import tn_oracle as O
from tnl_testutil import golden_layer_kwargs

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 2e-2
DEV = "cuda"


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(a))


def to_layer(L: O.OracleLayer, round_bf16=False):
    f = O.round_bf16 if round_bf16 else (lambda a: a)
    kw = dict(family=L.family, mode_shape=L.mode_shape, row_mode_count=L.row_mode_count)
    if L.family == "tucker":
        kw["core"] = f(L.core)
        kw["factors"] = [f(u) for u in L.factors]
    elif L.family in ("tt", "tr"):
        kw["cores"] = [f(c) for c in L.cores]
    else:
        kw["matrix"] = f(L.matrix)
    return tnl.CompressedLayer(**kw), O.OracleLayer(**kw)


def run(layer, x64, dtype, flags=tnl.PLAN_AUTO):
    x = torch.tensor(x64, dtype=dtype, device=DEV)
    y = layer.plan(dtype, flags=flags).forward(x)
    torch.cuda.synchronize()
    return y.float().cpu().numpy()


def check_bf16(L64: O.OracleLayer, m: int, seed: int, flags=tnl.PLAN_AUTO, tol=BF16_TOL):
    layer, Lr = to_layer(L64, round_bf16=True)
    rows, cols = Lr.matrix_shape
    x = O.round_bf16(O.synthetic_x(m, cols, seed))
    y = run(layer, x, torch.bfloat16, flags)
    ref = O.forward_torch_orient(Lr, x)
    e = rel(ref, y)
    assert e <= tol, (L64.family, L64.mode_shape, m, flags, e)
    return e


# --- golden fixtures (reference outputs) ------------------------------------


def test_golden_fp32_generic(golden):
    index, arrays = golden
    for rec in index["forward"] + index["decomp"]:
        layer = tnl.CompressedLayer(**golden_layer_kwargs(rec, arrays))
        x, y = arrays[rec["x"]], arrays[rec["y"]]
        out = run(layer, x.T, torch.float32, tnl.PLAN_GENERIC)
        assert rel(y.T, out) <= FP32_TOL, (rec["family"], rec["mode_shape"], rel(y.T, out))


def test_golden_fp32_auto(golden):
    """fp32 AUTO plans (the FFMA merged cut where it needs fewer flops than the chain) against the
    reference outputs, same 1e-5 bar as the chain."""
    index, arrays = golden
    names = set()
    for rec in index["forward"] + index["decomp"]:
        layer = tnl.CompressedLayer(**golden_layer_kwargs(rec, arrays))
        x, y = arrays[rec["x"]], arrays[rec["y"]]
        out = run(layer, x.T, torch.float32, tnl.PLAN_AUTO)
        names.add(layer.plan(torch.float32).info["plan_large_name"])
        assert rel(y.T, out) <= FP32_TOL, (rec["family"], rec["mode_shape"], rel(y.T, out))
    assert "cut" in names


@pytest.mark.parametrize("flags", [tnl.PLAN_AUTO, tnl.PLAN_CUT, tnl.PLAN_CHAIN, tnl.PLAN_GENERIC])
def test_golden_bf16_plans(golden, flags):
    index, arrays = golden
    for rec in index["forward"] + index["decomp"]:
        kw = golden_layer_kwargs(rec, arrays)
        L = O.OracleLayer(**kw)
        layer, Lr = to_layer(L, round_bf16=True)
        x = O.round_bf16(arrays[rec["x"]].T)
        out = run(layer, x, torch.bfloat16, flags)
        ref = O.forward_torch_orient(Lr, x)
        assert rel(ref, out) <= BF16_TOL, (rec["family"], rec["mode_shape"], flags, rel(ref, out))


def test_golden_reconstruct(golden):
    index, arrays = golden
    for rec in index["forward"] + index["decomp"]:
        if "w" not in rec:
            continue
        layer = tnl.CompressedLayer(**golden_layer_kwargs(rec, arrays))
        w = tnl.reconstruct(layer).cpu().numpy()
        assert w.shape == tuple(rec["mode_shape"])
        assert rel(arrays[rec["w"]], w) <= 1e-6
        m = tnl.layer_to_matrix(layer).cpu().numpy()
        assert m.shape == tuple(layer.matrix_shape)
        assert tnl.param_count(layer) == rec["param_count"]


# --- BASELINE config shapes -------------------------------------------------------


def test_cfg1_tt_fp32():
    """cfg1: TT 4096->4096, (64,64|64,64) r32, M=16, fp32 (<= 1e-5)."""
    L = O.synthetic_layer("tt", (64, 64, 64, 64), 2, (32, 32, 32), seed=10_000 + 100)
    L32 = O.OracleLayer("tt", L.mode_shape, 2, cores=[c.astype(np.float32).astype(np.float64) for c in L.cores])
    layer = tnl.CompressedLayer("tt", L.mode_shape, 2, cores=[c.astype(np.float32) for c in L.cores])
    x = O.synthetic_x(16, 4096, seed=10_000 + 9_999).astype(np.float32).astype(np.float64)
    ref = O.forward_torch_orient(L32, x)
    for flags in (tnl.PLAN_AUTO, tnl.PLAN_GENERIC):
        y = run(layer, x, torch.float32, flags)
        assert rel(ref, y) <= FP32_TOL
    assert layer.plan(torch.float32).info["plan_large_name"] == "cut"  # FFMA merged cut (fewer flops)
    # bf16 variant of cfg1 (merged cut and the tcgen05 core-by-core chain)
    check_bf16(L, 16, seed=11)
    check_bf16(L, 16, seed=11, flags=tnl.PLAN_CHAIN)
    check_bf16(L, 300, seed=12, flags=tnl.PLAN_CHAIN)


@pytest.mark.parametrize("spec", [("tt", (64, 64, 64, 64), 2, (32, 32, 32)), ("tr", (5120, 5120), 1, (16, 16)),
                                  ("tucker", (40, 24, 16), 1, (5, 4, 6)), ("tr", (6, 10, 8, 4), 2, (3, 2, 4, 2))])
def test_fp32_small_m_cut_repeated(spec):
    """fp32 merged cut at M <= 32 (dec32.cu: split-K phase A into the zero-at-rest accumulator,
    phase B with the last-CTA re-zero) against the float64 oracle, call after call, M straddling
    the 32-token limit (M = 33 takes the generic FFMA steps)."""
    fam, ms, rm, ranks = spec
    L = O.synthetic_layer(fam, ms, rm, ranks, seed=50_500)
    kw = dict(family=L.family, mode_shape=L.mode_shape, row_mode_count=L.row_mode_count)
    if fam == "tucker":
        kw.update(core=L.core.astype(np.float32), factors=[u.astype(np.float32) for u in L.factors])
        L32 = O.OracleLayer(core=L.core.astype(np.float32).astype(np.float64),
                            factors=[u.astype(np.float32).astype(np.float64) for u in L.factors], **{k: kw[k] for k in ("family", "mode_shape", "row_mode_count")})
    else:
        kw.update(cores=[c.astype(np.float32) for c in L.cores])
        L32 = O.OracleLayer(cores=[c.astype(np.float32).astype(np.float64) for c in L.cores],
                            **{k: kw[k] for k in ("family", "mode_shape", "row_mode_count")})
    layer = tnl.CompressedLayer(**kw)
    p = layer.plan(torch.float32)
    rows, cols = layer.matrix_shape
    for m in (1, 5, 16, 32, 33, 1):
        x = O.synthetic_x(m, cols, seed=50_600 + m).astype(np.float32).astype(np.float64)
        for _ in range(2):
            y = p.forward(torch.tensor(x, dtype=torch.float32, device=DEV))
            torch.cuda.synchronize()
            assert rel(O.forward_torch_orient(L32, x), y.double().cpu().numpy()) <= FP32_TOL, (spec, m)


@pytest.mark.parametrize("R", [64, 128, 256])
@pytest.mark.parametrize("m", [1, 7, 16, 64, 200])
def test_cfg2_tucker2(R, m):
    L = O.synthetic_layer("tucker", (5120, 5120), 1, (R, R), seed=20_000 + R)
    for flags in (tnl.PLAN_AUTO, tnl.PLAN_CHAIN):
        check_bf16(L, m, seed=20_000 + 9_999 + m, flags=flags)


@pytest.mark.parametrize("ab", [(8, 8), (16, 16)])
@pytest.mark.parametrize("m", [1, 16, 64])
def test_cfg2_tr2(ab, m):
    L = O.synthetic_layer("tr", (5120, 5120), 1, ab, seed=21_000 + ab[0])
    check_bf16(L, m, seed=21_999 + m)


@pytest.mark.parametrize("r", [8, 16])
@pytest.mark.parametrize("m", [1, 16, 64, 129])
def test_cfg2_tr4(r, m):
    L = O.synthetic_layer("tr", (64, 80, 64, 80), 2, (r, r, r, r), seed=22_000 + r)
    for flags in (tnl.PLAN_AUTO, tnl.PLAN_CHAIN):
        check_bf16(L, m, seed=22_999 + m, flags=flags)


@pytest.mark.parametrize("which", ["gate", "down"])
def test_cfg3_mlp_tt(which):
    ms = (160, 160, 64, 80) if which == "gate" else (64, 80, 160, 160)
    L = O.synthetic_layer("tt", ms, 2, (64, 64, 64), seed=30_000 + len(which))
    for flags in (tnl.PLAN_AUTO, tnl.PLAN_CHAIN):
        for m in (256, 40):
            check_bf16(L, m, seed=30_999 + m, flags=flags)


@pytest.mark.parametrize("r", [32, 128])
def test_cfg3_ranks_projections_and_block(r):
    """cfg3 at the other SURVEY ranks (r in {32, 64, 128}): gate/down projections (cut and chain
    plans) and the MLP block (fused when the kernels take the ranks, else unfused) vs the oracle."""
    from paper_2602_01613_b200.mlp import TNMLP

    specs = [(160, 160, 64, 80), (160, 160, 64, 80), (64, 80, 160, 160)]
    Ls = [O.synthetic_layer("tt", ms, 2, (r, r, r), seed=52_000 + 10 * r + i) for i, ms in enumerate(specs)]
    for L in (Ls[0], Ls[2]):
        for flags in (tnl.PLAN_AUTO, tnl.PLAN_CHAIN):
            for m in (1, 64, 256):
                check_bf16(L, m, seed=52_999 + m, flags=flags)
    pairs = [to_layer(L, round_bf16=True) for L in Ls]
    mlp = TNMLP(*[p[0] for p in pairs])
    for m in (1, 64, 256):
        x = O.round_bf16(O.synthetic_x(m, 5120, seed=53_000 + m))
        y = mlp(torch.tensor(x, dtype=torch.bfloat16, device=DEV))
        torch.cuda.synchronize()
        assert rel(_mlp_ref(*[p[1] for p in pairs], x), y.float().cpu().numpy()) <= 2 * BF16_TOL, (r, m, mlp.fused)


def test_cfg3_full_size_properties():
    """M=8192 prefill: token independence and linearity (up to the fp32 summation order of the
    split-K first step); sampled rows match the oracle."""
    L = O.synthetic_layer("tt", (160, 160, 64, 80), 2, (64, 64, 64), seed=31_000)
    layer, Lr = to_layer(L, round_bf16=True)
    x = torch.randn(8192, 5120, device=DEV).to(torch.bfloat16)
    p = layer.plan(torch.bfloat16)
    y = p.forward(x)
    idx = torch.tensor([0, 1, 127, 128, 4095, 8191], device=DEV)
    y_sub = p.forward(x[idx[:3]].contiguous().repeat(40, 1))[:3]  # M=120 keeps the large-M orientation
    d = (y[idx[:3]].float() - y_sub.float()).norm() / y_sub.float().norm()
    assert float(d) < 1e-2
    xs = x[idx].float().cpu().numpy().astype(np.float64)
    ref = O.forward_torch_orient(Lr, xs)
    assert rel(ref, y[idx].float().cpu().numpy()) <= BF16_TOL
    # 1024 rows against the oracle: every token tile (64) and tile position contributes
    g = torch.Generator().manual_seed(31_001)
    rows = torch.cat([torch.arange(0, 8192, 128), torch.randperm(8192, generator=g)[:960]]).to(DEV)
    ref_r = O.forward_torch_orient(Lr, x[rows].float().cpu().numpy().astype(np.float64))
    got_r = y[rows].float().cpu().numpy()
    assert rel(ref_r, got_r) <= BF16_TOL
    per_row = np.linalg.norm(ref_r - got_r, axis=1) / np.linalg.norm(ref_r, axis=1)
    assert float(per_row.max()) <= 2 * BF16_TOL  # no bad tile hides behind the aggregate
    # linearity: f(2x) == 2 f(x) (power-of-two scaling is exact; only summation order varies)
    y2 = p.forward((2 * x.float()).to(torch.bfloat16))
    d2 = (y2.float() - 2 * y.float()).norm() / (2 * y.float()).norm()
    assert float(d2) < 1e-2


# --- sharding, host path, edge cases -----------------------------------------------


@pytest.mark.parametrize("G", [2, 4])
def test_row_sharded_plans_concat_to_full(G):
    L = O.synthetic_layer("tucker", (1024, 512), 1, (64, 64), seed=40_000)
    layer, _ = to_layer(L, round_bf16=True)
    x = torch.randn(300, 512, device=DEV).to(torch.bfloat16)
    full = layer.plan(torch.bfloat16).forward(x)
    rows = 1024
    parts = [layer.plan(torch.bfloat16, row_range=(g * rows // G, (g + 1) * rows // G)).forward(x) for g in range(G)]
    assert torch.equal(torch.cat(parts, dim=1), full)


def test_forward_host_matches_device():
    L = O.synthetic_layer("tr", (64, 80, 64, 80), 2, (8, 8, 8, 8), seed=41_000)
    layer, _ = to_layer(L, round_bf16=True)
    p = layer.plan(torch.bfloat16, max_m=64)
    x = torch.randn(64, 5120).to(torch.bfloat16).pin_memory()
    yh = torch.empty(64, 5120, dtype=torch.bfloat16).pin_memory()
    p.forward_host(x, yh)
    torch.cuda.synchronize()
    yd = p.forward(x.to(DEV))
    # decode split-K reductions are fp32 atomics: equal up to summation order
    d = (yh.float() - yd.cpu().float()).norm() / yd.cpu().float().norm()
    assert float(d) < 5e-3


def test_edge_cases():
    L = O.synthetic_layer("tt", (16, 16, 16, 16), 2, (8, 8, 8), seed=42_000)
    layer, Lr = to_layer(L, round_bf16=True)
    p = layer.plan(torch.bfloat16)
    # M = 0
    y = p.forward(torch.empty(0, 256, dtype=torch.bfloat16, device=DEV))
    assert y.shape == (0, 256)
    # strided x (ldx > cols)
    big = torch.randn(33, 512, device=DEV).to(torch.bfloat16)
    xs = big[:, :256]
    y1 = p.forward(xs)
    y2 = p.forward(xs.contiguous())
    assert torch.equal(y1, y2)
    # shape / device errors mirror the reference exception types
    with pytest.raises(tnl.ShapeError):
        p.forward(torch.randn(4, 255, device=DEV).to(torch.bfloat16))
    with pytest.raises(tnl.DeviceError):
        layer.forward(torch.randn(4, 256).to(torch.bfloat16))
    # reference orientation
    xr = torch.randn(256, 5, device=DEV).to(torch.bfloat16)
    yr = tnl.apply_compressed(layer, xr)
    ref = O.apply_chain(Lr, xr.float().cpu().numpy().astype(np.float64))
    assert rel(ref, yr.float().cpu().numpy()) <= BF16_TOL


def test_dense_family():
    L = O.synthetic_layer("dense", (16, 32, 8, 16), 2, (), seed=43_000)
    for m in (3, 100):
        check_bf16(L, m, seed=43_001 + m)


def test_launch_counter_counts_kernels():
    L = O.synthetic_layer("tucker", (512, 512), 1, (64, 64), seed=44_000)
    layer, _ = to_layer(L, round_bf16=True)
    p = layer.plan(torch.bfloat16)
    x = torch.randn(256, 512, device=DEV).to(torch.bfloat16)
    p.forward(x)
    tnl.launch_count(reset=True)
    p.forward(x)
    assert tnl.launch_count() >= 2


@pytest.mark.parametrize("m", [1, 5, 8, 9, 33, 64])
def test_decode_repeat_zero_at_rest(m):
    """The decode accumulator is re-zeroed by the last CTA: repeated calls agree with the oracle."""
    L = O.synthetic_layer("tucker", (5120, 5120), 1, (128, 128), seed=45_000)
    layer, Lr = to_layer(L, round_bf16=True)
    p = layer.plan(torch.bfloat16)
    assert p.info["decode_max_m"] == 64
    x = O.round_bf16(O.synthetic_x(m, 5120, seed=45_001))
    xt = torch.tensor(x, dtype=torch.bfloat16, device=DEV)
    ref = O.forward_torch_orient(Lr, x)
    for _ in range(3):
        y = p.forward(xt)
        torch.cuda.synchronize()
        assert rel(ref, y.float().cpu().numpy()) <= BF16_TOL


def test_stack_graph_replay_matches_eager():
    from paper_2602_01613_b200.stack import TNStack

    Ls = [O.synthetic_layer(f, ms, rm, rk, seed=46_000 + i) for i, (f, ms, rm, rk) in enumerate(
        [("tucker", (1024, 1024), 1, (64, 64)), ("tr", (32, 32, 32, 32), 2, (4, 4, 4, 4)),
         ("tt", (32, 32, 32, 32), 2, (16, 16, 16))])]
    layers = [to_layer(L, round_bf16=True)[0] for L in Ls]
    st = TNStack(layers, torch.bfloat16)
    x = torch.randn(16, 1024, device=DEV).to(torch.bfloat16)
    ye = st.forward(x).clone()
    st.capture(16, host_io=True)
    st.x_host.copy_(x.cpu())
    for _ in range(3):
        st.replay()
    torch.cuda.synchronize()
    d = (st.y_host.float() - ye.cpu().float()).norm() / ye.cpu().float().norm()
    assert float(d) < 1e-2


@pytest.mark.parametrize("zero_copy", [False, True])
@pytest.mark.parametrize("mb", [1, 2, 3])
def test_stack_graph_host_io_microbatches(mb, zero_copy):
    """Host I/O per token group (graph) == the eager device pass: through tnl_copy_async, or zero-copy
    (tnl_stack_forward_host: the first kernel reads pinned x, the last writes pinned y)."""
    from paper_2602_01613_b200.stack import TNStack

    Ls = [O.synthetic_layer("tucker", (1024, 1024), 1, (64, 64), seed=46_100 + i) for i in range(3)]
    st = TNStack([to_layer(L, round_bf16=True)[0] for L in Ls], torch.bfloat16)
    x = torch.randn(37, 1024, device=DEV).to(torch.bfloat16)
    ye = st.forward(x).clone()
    st.capture(37, host_io=True, microbatches=mb, zero_copy=zero_copy)
    st.x_host.copy_(x.cpu())
    st.y_host.zero_()
    st.replay()
    torch.cuda.synchronize()
    d = (st.y_host.float() - ye.cpu().float()).norm() / ye.cpu().float().norm()
    assert float(d) < 1e-2
    x2 = torch.randn(37, 1024, device=DEV).to(torch.bfloat16)  # new host input, same graph
    st.x_host.copy_(x2.cpu())
    st.replay()
    torch.cuda.synchronize()
    y2 = st.forward(x2)
    d = (st.y_host.float() - y2.cpu().float()).norm() / y2.cpu().float().norm()
    assert float(d) < 1e-2


@pytest.mark.parametrize("nbytes", [16, 4096 + 7, 655360, 3 * 2**20 + 5])
def test_copy_async_roundtrip(nbytes):
    import ctypes

    from paper_2602_01613_b200 import _native as N

    lib = N.load()
    src = torch.randint(0, 255, (nbytes,), dtype=torch.uint8).pin_memory()
    dev = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    back = torch.zeros(nbytes, dtype=torch.uint8).pin_memory()
    s = torch.cuda.current_stream().cuda_stream
    N.check(lib.tnl_copy_async(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(src.data_ptr()), nbytes, ctypes.c_void_p(s)))
    N.check(lib.tnl_copy_async(ctypes.c_void_p(back.data_ptr()), ctypes.c_void_p(dev.data_ptr()), nbytes, ctypes.c_void_p(s)))
    torch.cuda.synchronize()
    assert torch.equal(dev.cpu(), src) and torch.equal(back, src)
    pageable = torch.zeros(64, dtype=torch.uint8)
    with pytest.raises(Exception):
        N.check(lib.tnl_copy_async(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(pageable.data_ptr()), 64,
                                   ctypes.c_void_p(s)))


def test_chain_plan_selected_for_two_mode_inputs():
    L = O.synthetic_layer("tr", (64, 80, 64, 80), 2, (16, 16, 16, 16), seed=47_000)
    layer, _ = to_layer(L, round_bf16=True)
    assert layer.plan(torch.bfloat16, flags=tnl.PLAN_CHAIN).info["plan_large_name"] == "chain"
    assert layer.plan(torch.bfloat16).info["plan_large_name"] == "cut"


@pytest.mark.parametrize("m", [64, 37, 16, 5])
def test_stack_fused_matches_oracle_chain(m):
    """tnl_stack_forward (one fused kernel per layer boundary) vs the oracle applied layer by layer
    on the same bf16 values (the oracle re-rounds each intermediate to bf16, as the GPU does)."""
    from paper_2602_01613_b200.stack import TNStack

    specs = [("tucker", (5120, 5120), 1, (256, 256)), ("tr", (64, 80, 64, 80), 2, (8, 8, 8, 8)),
             ("tr", (5120, 5120), 1, (16, 16)), ("tucker", (5120, 5120), 1, (64, 64)),
             ("tr", (64, 80, 64, 80), 2, (16, 16, 16, 16))]
    Ls = [O.synthetic_layer(f, ms, rm, rk, seed=48_000 + i) for i, (f, ms, rm, rk) in enumerate(specs)]
    pairs = [to_layer(L, round_bf16=True) for L in Ls]
    st = TNStack([p[0] for p in pairs], torch.bfloat16)
    x = O.round_bf16(O.synthetic_x(m, 5120, seed=48_999))
    y = st.forward(torch.tensor(x, dtype=torch.bfloat16, device=DEV))
    y2 = st.forward(torch.tensor(x, dtype=torch.bfloat16, device=DEV))  # accumulators re-zeroed
    torch.cuda.synchronize()
    ref = x
    for _, Lr in pairs:
        ref = O.round_bf16(O.forward_torch_orient(Lr, ref))
    assert rel(ref, y.float().cpu().numpy()) <= 3 * BF16_TOL
    assert rel(ref, y2.float().cpu().numpy()) <= 3 * BF16_TOL
    # and against the per-layer C-ABI path
    cur = torch.tensor(x, dtype=torch.bfloat16, device=DEV)
    for layer, _ in pairs:
        cur = layer.plan(torch.bfloat16).forward(cur)
    d = (cur.float() - y.float()).norm() / cur.float().norm()
    assert float(d) < 2e-2


@pytest.mark.parametrize("mb", [1, 2])
def test_stack_flag_handoff_replays(mb):
    """21 boundaries of the cfg2 variants in one CUDA graph (flag handoff between the boundary
    kernels, zero-at-rest accumulators and flags): 30 replays with a fresh input each, every one
    against the per-layer C-ABI path. A premature read, a missed zeroing or a stale flag shows up
    as a wrong replay."""
    from paper_2602_01613_b200 import synthetic as S
    from paper_2602_01613_b200.stack import TNStack

    layers = []
    for c in range(3):
        for v, (_, fam, ms, rm, ranks) in enumerate(S.CFG2_VARIANTS):
            L = O.synthetic_layer(fam, ms, rm, ranks, seed=49_000 + 10 * c + v)
            layers.append(to_layer(L, round_bf16=True)[0])
    st = TNStack(layers, torch.bfloat16)
    st.capture(64, host_io=False, microbatches=mb)
    plans = [l.plan(torch.bfloat16) for l in layers]
    g = torch.Generator(device="cpu").manual_seed(49_999)
    for it in range(30):
        x = torch.randn(64, 5120, generator=g).to(torch.bfloat16).to(DEV)
        st.x_dev.copy_(x)
        st.replay()
        torch.cuda.synchronize()
        cur = x
        for p in plans:
            cur = p.forward(cur)
        d = (cur.float() - st.y_dev.float()).norm() / cur.float().norm()
        assert float(d) < 2e-2, (it, float(d))


@pytest.mark.parametrize("spec", [("tucker", (5120, 5120), 1, (128, 128)), ("tr", (64, 80, 64, 80), 2, (16, 16, 16, 16)),
                                  ("tr", (5120, 5120), 1, (8, 8)), ("tt", (16, 16, 16, 16), 2, (8, 8, 8))])
@pytest.mark.parametrize("m", [1, 5, 8])
def test_decode_gemv_variant(spec, m):
    """CUDA-core GEMV decode variant (warp per weight row, no atomics) for M <= 8."""
    fam, ms, rm, rk = spec
    L = O.synthetic_layer(fam, ms, rm, rk, seed=49_000 + m)
    check_bf16(L, m, seed=49_500 + m, flags=tnl.PLAN_GEMV)


def _mlp_ref(Lg, Lu, Ld, x):
    g = O.forward_torch_orient(Lg, x)
    u = O.forward_torch_orient(Lu, x)
    h = O.round_bf16(g / (1.0 + np.exp(-g)) * u)
    return O.forward_torch_orient(Ld, h)


@pytest.mark.parametrize("m", [300, 5, 2048])
@pytest.mark.parametrize("fused", [True, False])
def test_mlp_block(m, fused):
    """y = down(silu(gate(x)) * up(x)): fused (h on chip) and unfused vs the oracle."""
    from paper_2602_01613_b200.mlp import TNMLP

    Lg = O.synthetic_layer("tt", (32, 32, 16, 32), 2, (16, 16, 16), seed=50_001)
    Lu = O.synthetic_layer("tr", (32, 32, 16, 32), 2, (2, 8, 8, 8), seed=50_002)
    Ld = O.synthetic_layer("tucker", (512, 1024), 1, (32, 32), seed=50_003)
    (g, Lgr), (u, Lur), (d, Ldr) = (to_layer(L, round_bf16=True) for L in (Lg, Lu, Ld))
    mlp = TNMLP(g, u, d, fused=fused)
    assert mlp.fused == fused
    x = O.round_bf16(O.synthetic_x(m, 512, seed=50_004))
    y = mlp(torch.tensor(x, dtype=torch.bfloat16, device=DEV))
    torch.cuda.synchronize()
    ref = _mlp_ref(Lgr, Lur, Ldr, x)
    assert rel(ref, y.float().cpu().numpy()) <= 2 * BF16_TOL


def test_mlp_block_cfg3():
    """cfg3: Qwen3-32B MLP (5120 -> 25600 -> 5120), TT r64 gate/up/down, fused."""
    from paper_2602_01613_b200.mlp import TNMLP

    Ls = [O.synthetic_layer("tt", ms, 2, (64, 64, 64), seed=51_000 + i) for i, ms in
          enumerate([(160, 160, 64, 80), (160, 160, 64, 80), (64, 80, 160, 160)])]
    pairs = [to_layer(L, round_bf16=True) for L in Ls]
    mlp = TNMLP(*[p[0] for p in pairs])
    assert mlp.fused
    x = O.round_bf16(O.synthetic_x(256, 5120, seed=51_009))
    y = mlp(torch.tensor(x, dtype=torch.bfloat16, device=DEV))
    ref = _mlp_ref(*[p[1] for p in pairs], x)
    assert rel(ref, y.float().cpu().numpy()) <= 2 * BF16_TOL


@pytest.mark.parametrize("m", [1, 37, 64])
def test_mlp_decode_gated_cfg3(m):
    """Decode MLP (M <= 64) at the cfg3 shape through the gated boundary kernel (gate/up phase B,
    SiLU*mul and down's phase A in one launch) vs the oracle; repeated calls (zero-at-rest slots)."""
    from paper_2602_01613_b200.mlp import TNMLP

    Ls = [O.synthetic_layer("tt", ms, 2, (64, 64, 64), seed=51_100 + i) for i, ms in
          enumerate([(160, 160, 64, 80), (160, 160, 64, 80), (64, 80, 160, 160)])]
    pairs = [to_layer(L, round_bf16=True) for L in Ls]
    mlp = TNMLP(*[p[0] for p in pairs])
    x = O.round_bf16(O.synthetic_x(m, 5120, seed=51_109))
    xt = torch.tensor(x, dtype=torch.bfloat16, device=DEV)
    ys = [mlp(xt).float().cpu().numpy() for _ in range(3)]
    ref = _mlp_ref(*[p[1] for p in pairs], x)
    for y in ys:
        assert rel(ref, y) <= 2 * BF16_TOL


@pytest.mark.parametrize("m", [1, 37, 64])
def test_mlp_decode_gated_large_rank(m):
    """Decode MLP with gate + up cut 512 (Tucker-2 R256, the cfg4 edge layers): the large gated
    boundary (down's B_in loaded into the gate's A blocks once the gate MMAs completed) vs the oracle."""
    from paper_2602_01613_b200.mlp import TNMLP

    Ls = [O.synthetic_layer("tucker", sh, 1, (256, 256), seed=51_200 + i) for i, sh in
          enumerate([(25600, 5120), (25600, 5120), (5120, 25600)])]
    pairs = [to_layer(L, round_bf16=True) for L in Ls]
    mlp = TNMLP(*[p[0] for p in pairs])
    x = O.round_bf16(O.synthetic_x(m, 5120, seed=51_209))
    xt = torch.tensor(x, dtype=torch.bfloat16, device=DEV)
    ys = [mlp(xt).float().cpu().numpy() for _ in range(3)]
    ref = _mlp_ref(*[p[1] for p in pairs], x)
    for y in ys:
        assert rel(ref, y) <= 2 * BF16_TOL


def test_qwen_stack_fused_mlp_matches_unfused():
    """cfg4 driver: the stack with fused TNMLP blocks (TT r64 / TR4 layers) equals the unfused stack."""
    from paper_2602_01613_b200.qwen_stack import QwenTNStack

    st_f = QwenTNStack(8, fused_mlp=True)
    st_u = QwenTNStack(8, fused_mlp=False)
    assert st_f.fused_mlp_count() == 2 and st_u.fused_mlp_count() == 0  # layers 3 (TT r64), 4 (TR4)
    torch.manual_seed(0)
    x0 = (0.5 * torch.randn(256, 5120, device=DEV)).to(torch.bfloat16)
    xf, xu = x0.clone(), x0.clone()
    st_f.forward(xf)
    st_u.forward(xu)
    torch.cuda.synchronize()
    assert torch.isfinite(xf.float()).all()
    assert rel(xu.float().cpu().numpy(), xf.float().cpu().numpy()) <= 2 * BF16_TOL


@pytest.mark.parametrize("rg,rd,variant", [(64, 64, "pair"), (128, 64, "ts"), (64, 256, "ss"), (128, 256, "ss")])
def test_mlp_kernel_variants(rg, rd, variant):
    """Each middle-kernel variant (csrc/mlp.cu) against the oracle, selected by the rank layout:
    pair (cut ranks <= 64 and r_d = 64: three TMEM G/U pairs), TS (T needs 128 TMEM columns:
    two pairs), SS (r_d = 256 leaves no room for T in TMEM). M = 300: a ragged last tile and an
    odd tile count (the pair grid pads to an even count)."""
    from paper_2602_01613_b200.mlp import TNMLP

    hid, inter = 512, 1024
    Lg = O.synthetic_layer("tucker", (inter, hid), 1, (rg, rg), seed=52_001)
    Lu = O.synthetic_layer("tucker", (inter, hid), 1, (rg, rg), seed=52_002)
    Ld = O.synthetic_layer("tucker", (hid, inter), 1, (rd, rd), seed=52_003)
    (g, Lgr), (u, Lur), (d, Ldr) = (to_layer(L, round_bf16=True) for L in (Lg, Lu, Ld))
    mlp = TNMLP(g, u, d)
    assert mlp.fused, variant
    x = O.round_bf16(O.synthetic_x(300, hid, seed=52_004))
    y = mlp(torch.tensor(x, dtype=torch.bfloat16, device=DEV))
    torch.cuda.synchronize()
    assert rel(_mlp_ref(Lgr, Lur, Ldr, x), y.float().cpu().numpy()) <= 2 * BF16_TOL


@pytest.mark.parametrize("rg,rd,m", [(256, 256, 300), (256, 64, 129), (192, 128, 300), (256, 256, 5)])
def test_mlp_dual_path(rg, rd, m):
    """Ranks the on-chip middle kernel cannot hold: gate/up output GEMMs + SiLU*mul in one kernel
    (csrc/dual_gemm.cu), then the down layer; M = 5 takes the decode path (three layers)."""
    from paper_2602_01613_b200.mlp import TNMLP

    hid, inter = 512, 1024 + 64  # intermediate not a multiple of the 128-wide tile
    Lg = O.synthetic_layer("tucker", (inter, hid), 1, (rg, rg), seed=53_001)
    Lu = O.synthetic_layer("tucker", (inter, hid), 1, (rg, rg), seed=53_002)
    Ld = O.synthetic_layer("tucker", (hid, inter), 1, (rd, rd), seed=53_003)
    (g, Lgr), (u, Lur), (d, Ldr) = (to_layer(L, round_bf16=True) for L in (Lg, Lu, Ld))
    mlp = TNMLP(g, u, d)
    assert not mlp.fused
    x = O.round_bf16(O.synthetic_x(m, hid, seed=53_004))
    y = mlp(torch.tensor(x, dtype=torch.bfloat16, device=DEV))
    torch.cuda.synchronize()
    assert rel(_mlp_ref(Lgr, Lur, Ldr, x), y.float().cpu().numpy()) <= 2 * BF16_TOL


@pytest.mark.parametrize("fused", [True, False])
def test_mlp_decode_fork_shared_workspace(fused):
    """Decode MLP (M <= 64): up runs on a forked stream with workspace slot 1 while gate uses
    slot 0. Prefill and decode calls alternate on ONE workspace (prefill scratch must never land in
    either slot's zero-at-rest accumulator), and the decode call also runs as a CUDA graph."""
    from paper_2602_01613_b200.mlp import TNMLP

    Lg = O.synthetic_layer("tucker", (1024, 512), 1, (64, 64), seed=54_001)
    Lu = O.synthetic_layer("tt", (32, 32, 16, 32), 2, (16, 32, 16), seed=54_002)
    Ld = O.synthetic_layer("tucker", (512, 1024), 1, (128, 128), seed=54_003)
    (g, Lgr), (u, Lur), (d, Ldr) = (to_layer(L, round_bf16=True) for L in (Lg, Lu, Ld))
    mlp = TNMLP(g, u, d, fused=fused)
    ws = torch.zeros(max(mlp.workspace_bytes(m) for m in (300, 64, 16, 1)), dtype=torch.uint8, device=DEV)
    for i, m in enumerate((16, 300, 1, 64, 300, 16, 16)):
        x = O.round_bf16(O.synthetic_x(m, 512, seed=54_010 + i))
        y = mlp.forward(torch.tensor(x, dtype=torch.bfloat16, device=DEV), ws=ws)
        torch.cuda.synchronize()
        assert rel(_mlp_ref(Lgr, Lur, Ldr, x), y.float().cpu().numpy()) <= 2 * BF16_TOL, (i, m)
    # graph capture of the forked decode call, replayed twice on new inputs
    x = O.round_bf16(O.synthetic_x(16, 512, seed=54_100))
    xd = torch.tensor(x, dtype=torch.bfloat16, device=DEV)
    yd = torch.empty(16, 512, dtype=torch.bfloat16, device=DEV)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        mlp.forward(xd, out=yd, ws=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        mlp.forward(xd, out=yd, ws=ws)
    for k in range(2):
        x = O.round_bf16(O.synthetic_x(16, 512, seed=54_200 + k))
        xd.copy_(torch.tensor(x, dtype=torch.bfloat16))
        gr.replay()
        torch.cuda.synchronize()
        assert rel(_mlp_ref(Lgr, Lur, Ldr, x), yd.float().cpu().numpy()) <= 2 * BF16_TOL, k


@pytest.mark.parametrize("m,n,with_o", [(1, 5120, True), (300, 5120, True), (17, 1024, False), (64, 8192, True)])
def test_add_rmsnorm(m, n, with_o):
    """Stack plumbing: x += o; h = x / rms(x) (one pass) vs torch (fp32 reference on the bf16 sum)."""
    from paper_2602_01613_b200.qwen_stack import QwenTNStack

    torch.manual_seed(m + n)
    x = torch.randn(m, n, device=DEV).to(torch.bfloat16)
    o = torch.randn(m, n, device=DEV).to(torch.bfloat16) if with_o else None
    ref_x = (x.float() + o.float()).to(torch.bfloat16) if with_o else x.clone()
    ref_h = torch.nn.functional.rms_norm(ref_x.float(), (n,), eps=1e-6)
    h = torch.empty_like(x)
    QwenTNStack.add_rmsnorm(x, o, h)
    torch.cuda.synchronize()
    assert torch.equal(x, ref_x)
    assert rel(ref_h.cpu().numpy(), h.float().cpu().numpy()) <= 1e-2


@pytest.mark.parametrize("spec", [("tucker", (5120, 5120), 1, (256, 256)), ("tt", (160, 160, 64, 80), 2, (64, 64, 64))])
def test_forward_ex_folded_norm_accumulate(spec):
    """tnl_forward_ex (prefill): y += f(x / rms(x)) with the statistics from tnl_rms_stats, vs the
    unfolded path (normalised input through tnl_forward, then a torch add)."""
    import ctypes

    from paper_2602_01613_b200 import _native as N

    f, ms, rm, rk = spec
    L = O.synthetic_layer(f, ms, rm, rk, seed=52_000)
    layer, _ = to_layer(L, round_bf16=True)
    rows, cols = layer.matrix_shape
    m = 300
    torch.manual_seed(2)
    x = (3 * torch.randn(m, cols, device=DEV)).to(torch.bfloat16)
    r = torch.randn(m, rows, device=DEV).to(torch.bfloat16)
    lib = N.load()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ss = torch.empty(m, device=DEV)
    N.check(lib.tnl_rms_stats(ctypes.c_void_p(x.data_ptr()), cols, m, cols, ctypes.c_void_p(ss.data_ptr()), s))
    torch.cuda.synchronize()
    want = (x.float() ** 2).sum(1)
    assert rel(want.cpu().numpy(), ss.cpu().numpy()) <= 1e-5
    h = (x.float() * torch.rsqrt(want[:, None] / cols + 1e-6)).to(torch.bfloat16)
    pl = layer.plan(torch.bfloat16)
    ref = pl.forward(h).float() + r.float()
    y = r.clone()
    ws = pl.workspace(m)
    o = N.FwdOpts(1, ss.data_ptr(), cols, 1e-6)
    N.check(lib.tnl_forward_ex(pl.handle, ctypes.c_void_p(x.data_ptr()), m, cols, ctypes.c_void_p(y.data_ptr()), rows,
                               ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.byref(o), s))
    torch.cuda.synchronize()
    # y is accumulated in bf16 (TMA reduce-add): one extra bf16 rounding of the sum vs the fp32 ref
    assert rel(ref.cpu().numpy(), y.float().cpu().numpy()) <= BF16_TOL


@pytest.mark.parametrize("m", [300, 1024])
def test_qwen_stack_folded_prefill(m):
    """cfg4 prefill with the residual adds and RMSNorms folded into the projections' epilogues
    equals the pass with separate add+norm kernels (bf16 pipelines; rounding differs)."""
    from paper_2602_01613_b200.qwen_stack import QwenTNStack

    st = QwenTNStack(6)  # Tucker-2 R256 MLP (dual path) on layers 0-1 / 4-5, TT r64 / TR4 fused on 2 / 3
    torch.manual_seed(3)
    x0 = torch.randn(m, 5120, device=DEV).to(torch.bfloat16)
    outs = {}
    for fold in (True, False):
        st.fold_prefill = fold
        x = x0.clone()
        st.forward(x)
        torch.cuda.synchronize()
        assert torch.isfinite(x.float()).all()
        outs[fold] = x.float().cpu().numpy()
    assert rel(outs[False], outs[True]) <= BF16_TOL


def test_qwen_stack_decode_matches_prefill():
    """Regression: every plan and MLP block of a stack share one workspace; decode (M <= 64) must
    give the same tokens as the prefill path (per-token independence), which failed when an MLP's
    scratch overlapped a wider plan's zero-at-rest decode accumulator."""
    from paper_2602_01613_b200.qwen_stack import QwenTNStack

    st = QwenTNStack(8)
    torch.manual_seed(3)
    x = (0.5 * torch.randn(300, 5120, device=DEV)).to(torch.bfloat16)
    xp, xd = x.clone(), x[:64].clone()
    st.forward(xp)
    st.forward(xd)
    torch.cuda.synchronize()
    assert torch.isfinite(xd.float()).all()
    assert rel(xp[:64].float().cpu().numpy(), xd.float().cpu().numpy()) <= 2 * BF16_TOL


@pytest.mark.parametrize("spec", [("tucker", (5120, 5120), 1, (256, 256)), ("tr", (5120, 5120), 1, (16, 16)),
                                  ("tucker", (8192, 5120), 1, (256, 256))])
@pytest.mark.parametrize("m", [256, 300, 600])
def test_prefill_pair_gemm(spec, m):
    """Rank-256 prefill steps take the CTA-pair GEMM (csrc/tc_gemm_pair.cu): 256-row tiles, an odd
    token-tile count (300: the pair's second tile is past M) and split-K (600: step 1 reduces in
    fp32 over K-splits), vs the oracle; plus the chain plan (three Tucker-2 steps)."""
    fam, ms, rm, ranks = spec
    L = O.synthetic_layer(fam, ms, rm, ranks, seed=54_000 + m)
    check_bf16(L, m, seed=54_100 + m)
    if fam == "tucker":
        check_bf16(L, m, seed=54_200 + m, flags=tnl.PLAN_CHAIN)


def test_output_sharded_layer_single_rank_nccl():
    """OutputShardedLayer through a real NCCL group (world 1 on this box): the rank's rows are computed
    into its slot of the gather buffer and gathered in place; equals the plain forward."""
    import socket

    import torch.distributed as dist

    from paper_2602_01613_b200.sharded import OutputShardedLayer

    L = O.synthetic_layer("tt", (160, 160, 64, 80), 2, (64, 64, 64), seed=53_000)
    layer, _ = to_layer(L, round_bf16=True)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        # M = 8192: every prefill step is deterministic (split-K over CTA pairs through DSMEM, no
        # fp32 atomics), so the comparison is bitwise
        x = torch.randn(8192, 5120, device=DEV).to(torch.bfloat16)
        ref = layer.plan(torch.bfloat16).forward(x)
        for exchange in ("p2p", "allgather"):  # symmetric-memory in-place exchange / NCCL all-gather
            osl = OutputShardedLayer(layer, dtype=torch.bfloat16, device=torch.device(DEV, 0), exchange=exchange)
            y = osl(x)
            y2 = osl(x)  # the symmetric buffer is reused across calls
            torch.cuda.synchronize()
            assert torch.equal(ref, y) and torch.equal(ref, y2), exchange
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_output_shards_store_in_place_bitwise(G):
    """What G ranks of the P2P exchange assemble, emulated on one GPU: every rank's row-restricted
    plan stores its slice straight into its columns of ONE token-major y (strided TMA store, no
    gather buffer, no permute); the result equals the single-GPU forward bit for bit."""
    from paper_2602_01613_b200.sharded import output_shard_ranges

    for spec, seed in ((("tt", (160, 160, 64, 80), 2, (64, 64, 64)), 55_000),
                       (("tucker", (5120, 5120), 1, (128, 128)), 55_100), (("tr", (64, 80, 64, 80), 2, (8, 8, 8, 8)), 55_200)):
        L = O.synthetic_layer(*spec, seed=seed)
        layer, _ = to_layer(L, round_bf16=True)
        rows, cols = layer.matrix_shape
        x = torch.randn(8192, cols, device=DEV).to(torch.bfloat16)  # deterministic prefill steps (no atomics)
        ref = layer.plan(torch.bfloat16).forward(x)
        y = torch.full((8192, rows), float("nan"), device=DEV, dtype=torch.bfloat16)
        for lo, hi in output_shard_ranges(layer.mode_shape, layer.row_mode_count, G):
            layer.plan(torch.bfloat16, row_range=(lo, hi)).forward(x, out=y[:, lo:hi])
        torch.cuda.synchronize()
        assert torch.equal(ref, y), (spec, G)


def test_prefill_splitk2_pair_deterministic():
    """Narrow first step (cut <= 64) with >= 50 token tiles: split-K over a CTA pair, the partial
    exchanged through DSMEM (no fp32 buffer / atomics) — oracle parity and bitwise repeatability."""
    L = O.synthetic_layer("tt", (32, 32, 64, 80), 2, (64, 64, 64), seed=54_000)
    layer, Lr = to_layer(L, round_bf16=True)
    m = 50 * 128 + 37  # 51 token tiles (ragged last tile) -> split-K 2
    x = O.round_bf16(O.synthetic_x(m, 5120, seed=54_009))
    xt = torch.tensor(x, dtype=torch.bfloat16, device=DEV)
    y1 = layer.forward(xt)
    y2 = layer.forward(xt)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    ref = O.forward_torch_orient(Lr, x[:512])
    assert rel(ref, y1[:512].float().cpu().numpy()) <= BF16_TOL
    tail = O.forward_torch_orient(Lr, x[-200:])  # rows of the ragged last tile
    assert rel(tail, y1[-200:].float().cpu().numpy()) <= BF16_TOL


def test_qwen_stack_decode_microbatches():
    """cfg4 decode graph with two concurrent token groups (own workspaces / side streams) equals
    the single-group graph."""
    from paper_2602_01613_b200.qwen_stack import QwenTNStack

    st = QwenTNStack(6)
    torch.manual_seed(4)
    x0 = torch.randn(64, 5120, device=DEV).to(torch.bfloat16)
    outs = []
    for mb in (1, 2):
        g = st.capture(64, microbatches=mb)
        st.x.copy_(x0)
        g.replay()
        torch.cuda.synchronize()
        outs.append(st.x.float().cpu().numpy())
    assert np.isfinite(outs[1]).all()
    assert rel(outs[0], outs[1]) <= 1e-2


def test_stack_forward_host_rejects_pageable_and_prefill():
    """tnl_stack_forward_host: pageable host buffers and prefill-sized M are refused (no fallback)."""
    from paper_2602_01613_b200.stack import TNStack

    L = O.synthetic_layer("tucker", (1024, 1024), 1, (64, 64), seed=55_000)
    st = TNStack([to_layer(L, round_bf16=True)[0]] * 2, torch.bfloat16)
    xp = torch.zeros(8, 1024, dtype=torch.bfloat16)  # pageable
    yp = torch.zeros(8, 1024, dtype=torch.bfloat16)
    with pytest.raises(Exception):
        st.forward_host(xp, yp)
    xh = torch.zeros(100, 1024, dtype=torch.bfloat16).pin_memory()
    yh = torch.zeros(100, 1024, dtype=torch.bfloat16).pin_memory()
    with pytest.raises(Exception):
        st.forward_host(xh, yh)  # M = 100 > 64: not a fused decode stack
    xs, ys = xh[:8], yh[:8]
    xs.copy_(torch.randn(8, 1024).to(torch.bfloat16))
    st.forward_host(xs, ys)
    torch.cuda.synchronize()
    ref = st.forward(xs.cuda()).cpu()
    assert rel(ref.float().numpy(), ys.float().numpy()) <= 1e-2
