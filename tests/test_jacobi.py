"""One-sided Jacobi sweeps + deterministic SVD.

CPU: the oracle restatement of `_jacobi_cy.pyx:11-53` is pinned bit-for-bit against the
reference's own compiled kernel (`oracle/_ref`, built from the reference's C by
`oracle/build_ref.py`) and against golden fixtures produced by running the reference
(`tests/golden/make_golden_jacobi.py`: `_jacobi_py.jacobi_sweeps`, `tensor_core.full_svd`).
GPU: `tnl_jacobi_sweeps` (csrc/jacobi.cu) against the oracle — equal up to the summation order
of the dot products, the latitude the reference grants its own numpy twin
(`_jacobi_py.py:7-8`) — and the reference's TestTruncatedSvd suite
(`pkg/tests/test_tensor_core.py:148-235`) re-run on the GPU-backed SVD.
"""

import os

import numpy as np
import pytest

from oracle import build_ref
from oracle import tn_oracle as O

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "jacobi.npz"))
NAMES = [str(n) for n in GOLD["names"]]
TOL_SUM = 1e-11  # summation-order latitude (relative to the row norms)


def _setup(a):
    m, n = a.shape
    aa = a.T if m < n else a
    return aa.T.copy(), np.eye(aa.shape[1])


def _close(ref, got, scale):
    return float(np.max(np.abs(ref - got))) <= TOL_SUM * max(1.0, scale)


def _numerical_rank(name):
    v = GOLD[f"{name}.values"]
    return int(np.count_nonzero(v > 1e-10 * max(float(v[0]), 1e-300))) if v.size else 0


def _degenerate(name):
    """Rank-deficient but not exactly-zero columns: rotations inside the numerical null space
    depend on rounding, so the sweep count, work/rot and the null-space singular vectors are
    order-sensitive; only the spectrum and the range singular vectors are compared."""
    v = GOLD[f"{name}.values"]
    return 0 < _numerical_rank(name) < v.size and not np.any(v == 0.0)


def _check_svd(name, left, values, right):
    a = GOLD[f"{name}.a"]
    scale = max(1.0, float(np.linalg.norm(a)))
    assert np.max(np.abs(values - GOLD[f"{name}.values"])) <= 1e-10 * scale
    r = _numerical_rank(name) if _degenerate(name) else values.size
    assert np.max(np.abs(left[:, :r] - GOLD[f"{name}.left"][:, :r]), initial=0.0) <= 1e-9
    assert np.max(np.abs(right[:, :r] - GOLD[f"{name}.right"][:, :r]), initial=0.0) <= 1e-9
    assert np.max(np.abs((left * values) @ right.T - a)) <= 1e-10 * scale


# ---------------------------------------------------------------- CPU: oracle pinning


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_golden(name):
    a = GOLD[f"{name}.a"]
    work, rot = _setup(a)
    sweeps = O.jacobi_sweeps(work, rot, O.JACOBI_TOL, O.JACOBI_MAX_SWEEPS)
    if not _degenerate(name):
        assert sweeps == int(GOLD[f"{name}.sweeps"])
        scale = float(np.linalg.norm(a))
        assert _close(GOLD[f"{name}.work"], work, scale)
        assert _close(GOLD[f"{name}.rot"], rot, 1.0)
    _check_svd(name, *O.jacobi_svd(a))


def test_oracle_one_sweep_exit():
    a = GOLD["one_sweep.a"]
    work, rot = a.T.copy(), np.eye(a.shape[1])
    assert O.jacobi_sweeps(work, rot, 1e-12, 1) == int(GOLD["one_sweep.sweeps"]) == 1
    assert _close(GOLD["one_sweep.work"], work, float(np.linalg.norm(a)))


def test_oracle_bitexact_vs_compiled_reference():
    """The restatement equals the reference's compiled `_jacobi_cy` bit for bit."""
    ref = build_ref.load()
    if ref is None:
        pytest.skip("oracle/_ref not built (python oracle/build_ref.py)")
    rng = np.random.default_rng(5)
    for n, m in [(2, 3), (5, 7), (8, 8), (6, 13), (12, 12)]:
        a = rng.standard_normal((n, m))
        w1, r1 = a.copy(), np.eye(n)
        w2, r2 = a.copy(), np.eye(n)
        s1 = ref.jacobi_sweeps(w1, r1, 1e-12, 60)
        s2 = O.jacobi_sweeps(w2, r2, 1e-12, 60)
        assert s1 == s2
        assert w1.tobytes() == w2.tobytes() and r1.tobytes() == r2.tobytes()


def test_api_shape_errors_before_device():
    from paper_2602_01613_b200 import jacobi as J
    from paper_2602_01613_b200.errors import RankError, ShapeError

    with pytest.raises(ShapeError):
        J.jacobi_sweeps(np.zeros((3, 4), np.float32), np.eye(3), 1e-12, 5)
    with pytest.raises(ShapeError):
        J.jacobi_sweeps(np.zeros((3, 4)), np.eye(4), 1e-12, 5)
    with pytest.raises(ShapeError):
        J.full_svd(np.zeros((2, 2, 2)))
    with pytest.raises(RankError):
        J.FixedRank(0)
    with pytest.raises(RankError):
        J.RelativeError(1.5)
    with pytest.raises(RankError):
        J.ParamBudget(0)


# ---------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_sweeps_match_reference(name):
    from paper_2602_01613_b200 import jacobi as J

    a = GOLD[f"{name}.a"]
    work, rot = _setup(a)
    w0, r0 = work.copy(), rot.copy()
    sweeps = J.jacobi_sweeps(work, rot, J.JACOBI_TOL, J.JACOBI_MAX_SWEEPS)
    so = O.jacobi_sweeps(w0, r0, O.JACOBI_TOL, O.JACOBI_MAX_SWEEPS)
    if not _degenerate(name):
        assert sweeps == so == int(GOLD[f"{name}.sweeps"])
        scale = float(np.linalg.norm(a))
        assert _close(w0, work, scale) and _close(r0, rot, 1.0)
        assert _close(GOLD[f"{name}.work"], work, scale)


@pytest.mark.gpu
def test_gpu_batched_matches_oracle():
    import torch

    from paper_2602_01613_b200 import jacobi as J

    rng = np.random.default_rng(11)
    b, n, m, nv = 37, 12, 40, 12
    work = rng.standard_normal((b, n, m))
    work[3] = 0.0  # all rows zero: every pair skipped, one sweep
    work[5, 2] = 0.0  # one zero row
    rot = np.broadcast_to(np.eye(n), (b, n, nv)).copy()
    wt = torch.tensor(work, device="cuda")
    rt = torch.tensor(rot, device="cuda")
    sweeps = J.jacobi_sweeps_batched(wt, rt).cpu().numpy()
    wg, rg = wt.cpu().numpy(), rt.cpu().numpy()
    for i in range(b):
        w0, r0 = work[i].copy(), rot[i].copy()
        s0 = O.jacobi_sweeps(w0, r0, O.JACOBI_TOL, O.JACOBI_MAX_SWEEPS)
        assert int(sweeps[i]) == s0, i
        assert _close(w0, wg[i], float(np.linalg.norm(work[i]))) and _close(r0, rg[i], 1.0), i
    assert int(sweeps[3]) == 1 and np.array_equal(wg[3], work[3])


@pytest.mark.gpu
def test_gpu_max_sweeps_and_tol():
    from paper_2602_01613_b200 import jacobi as J

    a = GOLD["one_sweep.a"]
    work, rot = a.T.copy(), np.eye(a.shape[1])
    assert J.jacobi_sweeps(work, rot, 1e-12, 1) == 1
    assert _close(GOLD["one_sweep.work"], work, float(np.linalg.norm(a)))
    work, rot = a.T.copy(), np.eye(a.shape[1])
    assert J.jacobi_sweeps(work, rot, 1e-12, 0) == 0 and np.array_equal(work, a.T)
    with pytest.raises(ValueError):
        J.jacobi_sweeps(work, rot, 1e-12, -1)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_full_svd_matches_reference(name):
    from paper_2602_01613_b200 import jacobi as J

    res = J.full_svd(GOLD[f"{name}.a"])
    _check_svd(name, res.left, res.values, res.right)


# the reference's TestTruncatedSvd (pkg/tests/test_tensor_core.py:148-235), GPU-backed


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)  # pkg/tests/conftest.py:5-7


@pytest.mark.gpu
class TestTruncatedSvdGPU:
    def test_rank_one_matrix(self):
        from paper_2602_01613_b200.jacobi import FixedRank, truncated_svd

        m = np.array([[1.0, 2.0], [2.0, 4.0]])
        res = truncated_svd(m, FixedRank(1))
        assert res.values == pytest.approx([5.0])
        assert np.allclose(res.reconstruct(), m, atol=1e-12)

    def test_relative_error_identity_needs_full_rank(self):
        from paper_2602_01613_b200.jacobi import RelativeError, truncated_svd

        assert truncated_svd(np.eye(3), RelativeError(0.5)).rank == 3

    def test_full_rank_reconstruction(self, rng):
        from paper_2602_01613_b200.jacobi import FixedRank, truncated_svd

        m = rng.standard_normal((8, 5))
        res = truncated_svd(m, FixedRank(5))
        assert O.relative_error(m, res.reconstruct()) <= 1e-10

    def test_orthonormal_blocks(self, rng):
        from paper_2602_01613_b200.jacobi import full_svd

        for shape in [(6, 6), (8, 3), (3, 8)]:
            res = full_svd(rng.standard_normal(shape))
            r = res.rank
            assert np.max(np.abs(res.left.T @ res.left - np.eye(r))) <= 1e-10
            assert np.max(np.abs(res.right.T @ res.right - np.eye(r))) <= 1e-10

    def test_values_sorted_nonnegative(self, rng):
        from paper_2602_01613_b200.jacobi import full_svd

        res = full_svd(rng.standard_normal((7, 4)))
        assert np.all(res.values >= 0) and np.all(np.diff(res.values) <= 0)

    def test_eckart_young_against_eigh_oracle(self, rng):
        from paper_2602_01613_b200.jacobi import FixedRank, truncated_svd

        for _ in range(10):
            m = rng.standard_normal((6, 6))
            sigma = np.sqrt(np.clip(np.sort(np.linalg.eigvalsh(m.T @ m))[::-1], 0, None))
            for r in (1, 3, 5):
                res = truncated_svd(m, FixedRank(r))
                err = float(np.linalg.norm(m - res.reconstruct()))
                assert err == pytest.approx(np.sqrt(np.sum(sigma[r:] ** 2)), abs=1e-9)

    def test_fixed_rank_pads_with_zeros(self):
        from paper_2602_01613_b200.jacobi import FixedRank, truncated_svd

        res = truncated_svd(np.array([[1.0, 2.0], [2.0, 4.0]]), FixedRank(2))
        assert res.values[0] == pytest.approx(5.0) and res.values[1] <= 1e-12
        assert np.max(np.abs(res.left.T @ res.left - np.eye(2))) <= 1e-10

    def test_zero_matrix(self):
        from paper_2602_01613_b200.jacobi import full_svd

        res = full_svd(np.zeros((4, 3)))
        assert np.all(res.values == 0)
        assert np.max(np.abs(res.left.T @ res.left - np.eye(3))) <= 1e-10
        assert np.max(np.abs(res.right.T @ res.right - np.eye(3))) <= 1e-10

    def test_sign_convention(self, rng):
        from paper_2602_01613_b200.jacobi import full_svd

        res = full_svd(rng.standard_normal((6, 4)))
        for j in range(res.rank):
            col = res.left[:, j]
            assert col[int(np.argmax(np.abs(col)))] > 0

    def test_param_budget_rank(self, rng):
        from paper_2602_01613_b200.errors import InfeasibleBudgetError
        from paper_2602_01613_b200.jacobi import ParamBudget, truncated_svd

        m = rng.standard_normal((8, 5))
        assert truncated_svd(m, ParamBudget(14)).rank == 1
        assert truncated_svd(m, ParamBudget(41)).rank == 2
        assert truncated_svd(m, ParamBudget(10**6)).rank == 5
        with pytest.raises(InfeasibleBudgetError):
            truncated_svd(m, ParamBudget(13))

    def test_fixed_rank_exceeds_min_dim(self):
        from paper_2602_01613_b200.errors import RankError
        from paper_2602_01613_b200.jacobi import FixedRank, truncated_svd

        with pytest.raises(RankError):
            truncated_svd(np.ones((3, 5)), FixedRank(4))

    def test_determinism_bitwise(self, rng):
        from paper_2602_01613_b200.jacobi import FixedRank, truncated_svd

        m = rng.standard_normal((9, 6))
        a = truncated_svd(m.copy(), FixedRank(4))
        b = truncated_svd(m.copy(), FixedRank(4))
        assert a.left.tobytes() == b.left.tobytes()
        assert a.values.tobytes() == b.values.tobytes()
        assert a.right.tobytes() == b.right.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,nv", [(6, 300, 6), (5, 40, 290), (33, 33, 33), (1, 8, 1)])
def test_gpu_sweeps_generic_and_edge_shapes(n, m, nv):
    """Rows longer than the register-resident variant (m or nv > 256 -> generic kernel), odd
    sizes, and the single-row problem (no pair: one sweep, nothing rotated)."""
    import torch

    from paper_2602_01613_b200 import jacobi as J

    rng = np.random.default_rng(n * 1000 + m + nv)
    work = rng.standard_normal((2, n, m))
    rot = rng.standard_normal((2, n, nv))
    wt, rt = torch.tensor(work, device="cuda"), torch.tensor(rot, device="cuda")
    sweeps = J.jacobi_sweeps_batched(wt, rt).cpu().numpy()
    for i in range(2):
        w0, r0 = work[i].copy(), rot[i].copy()
        s0 = O.jacobi_sweeps(w0, r0, O.JACOBI_TOL, O.JACOBI_MAX_SWEEPS)
        assert int(sweeps[i]) == s0
        assert _close(w0, wt[i].cpu().numpy(), float(np.linalg.norm(work[i])))
        assert _close(r0, rt[i].cpu().numpy(), float(np.linalg.norm(rot[i])))


# ---------------------------------------------------------------- GPU: parallel order, device finish


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_parallel_order_svd_matches_reference(name):
    """Round-robin sweeps (tnl_jacobi_sweeps_parallel) + device post-processing against the
    reference's full_svd: same spectrum (<= 1e-10 relative), same singular vectors where they are
    determined (distinct values; the sign convention fixes the sign)."""
    from paper_2602_01613_b200 import jacobi as J

    a = GOLD[f"{name}.a"]
    res = J.full_svd(a, parallel=True)
    scale = max(1.0, float(np.linalg.norm(a)))
    v_ref = GOLD[f"{name}.values"]
    assert np.max(np.abs(res.values - v_ref), initial=0.0) <= 1e-10 * scale
    assert np.max(np.abs((res.left * res.values) @ res.right.T - a), initial=0.0) <= 1e-10 * scale
    if v_ref.size:
        gaps = np.abs(np.diff(v_ref))
        distinct = np.ones(v_ref.size, bool)
        distinct[:-1] &= gaps > 1e-6 * scale
        distinct[1:] &= gaps > 1e-6 * scale
        distinct &= v_ref > 1e-8 * scale
        assert np.max(np.abs(res.left[:, distinct] - GOLD[f"{name}.left"][:, distinct]), initial=0.0) <= 1e-8
        assert np.max(np.abs(res.right[:, distinct] - GOLD[f"{name}.right"][:, distinct]), initial=0.0) <= 1e-8
    k = min(a.shape)
    for u in (res.left, res.right):
        assert np.max(np.abs(u.T @ u - np.eye(k)), initial=0.0) <= 1e-10


@pytest.mark.gpu
def test_gpu_parallel_order_large_unfolding():
    """A Qwen-shaped unfolding (5120 x 640): spectrum vs LAPACK (float64) <= 1e-10 relative,
    orthonormal factors, exact reconstruction."""
    from paper_2602_01613_b200 import jacobi as J

    rng = np.random.default_rng(77)
    a = rng.standard_normal((5120, 640)) @ np.diag(np.linspace(1.0, 1e-3, 640)) @ np.linalg.qr(
        rng.standard_normal((640, 640)))[0]
    res = J.full_svd(a, parallel=True)
    s = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(res.values - s)) <= 1e-10 * s[0]
    assert np.all(np.diff(res.values) <= 0)
    assert np.max(np.abs(res.left.T @ res.left - np.eye(640))) <= 1e-10
    assert np.max(np.abs(res.right.T @ res.right - np.eye(640))) <= 1e-10
    assert np.max(np.abs((res.left * res.values) @ res.right.T - a)) <= 1e-10 * s[0]


@pytest.mark.gpu
def test_gpu_svd_finish_completes_zero_columns():
    """Exactly-zero columns: the device completion reproduces the reference's greedy canonical
    pick (tensor_core.py:185-200) — the reference's own _complete_basis on the same range vectors."""
    from paper_2602_01613_b200 import jacobi as J

    a = np.zeros((7, 4))
    a[2, 0] = 3.0
    a[:, 2] = np.arange(7.0)
    res = J.full_svd(a)
    # oracle: the reference's post-processing restated in numpy (oracle/tn_oracle.jacobi_svd)
    left, values, right = O.jacobi_svd(a)
    assert np.max(np.abs(res.values - values)) <= 1e-12 * 10
    assert np.max(np.abs(res.left - left)) <= 1e-10
    assert np.max(np.abs(res.right - right)) <= 1e-10
