"""Algebraic properties of the public drop-in API on the B200 build, the ones
the reference's unit tests pin for the hot path's building blocks:

  Nystrom factor           tests/test_randnla.py:22-99 of the reference
  Woodbury applies         tests/test_randnla.py:102-150
  power-iteration stepsize tests/test_randnla.py:153-175
  kernel values / blocks   tests/test_kernels.py:21-141
  exact SAP step           tests/test_solvers.py:104-143

The problems, seeds and sizes here are our own. Bars are the reference's for
fp64 work (factor, applies, the fp64 tile); block products through the
tensor-core kernel are fp32-accurate, so their bars are stated relative to the
product's scale (1e-5).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sap = pytest.importorskip("paper_2505_13723_b200")


def _psd(rng, dim):
    A = rng.standard_normal((dim, dim + 3))
    return A @ A.T / (dim + 3)


def _factor(rng, M, rank):
    om = rng.standard_normal((M.shape[0], rank))
    return sap.rand_nystrom(M @ om, om, rank)


def _lowrank(f):
    return (f.U * f.S) @ f.U.T


# ---------------------------------------------------------------------------
# Nystrom factor


def test_nystrom_of_identity_is_a_projector_with_unit_spectrum():
    rng = np.random.default_rng(101)
    om = rng.standard_normal((30, 7))
    f = sap.rand_nystrom(om.copy(), om, 7)
    np.testing.assert_allclose(f.S, 1.0, atol=1e-8)
    P = f.U @ f.U.T
    assert np.abs(P @ P - P).max() < 1e-10
    # the range of the projector is the sketch's range
    assert np.abs(P @ om - om).max() < 1e-10


@pytest.mark.parametrize("dim", [1, 9, 25])
def test_full_rank_nystrom_reconstructs(dim):
    rng = np.random.default_rng(102 + dim)
    M = _psd(rng, dim)
    f = _factor(rng, M, dim)
    assert np.linalg.norm(_lowrank(f) - M) <= 1e-8 * np.linalg.norm(M)


def test_zero_sketch_gives_zero_spectrum_and_plain_scaling():
    rng = np.random.default_rng(103)
    f = sap.rand_nystrom(np.zeros((12, 4)), rng.standard_normal((12, 4)), 4)
    assert np.all(f.S == 0.0)
    g = rng.standard_normal(12)
    np.testing.assert_allclose(sap.apply_inv(f, 0.25, g), g / 0.25, rtol=1e-14)


def test_factor_columns_orthonormal_and_spectrum_sorted():
    rng = np.random.default_rng(104)
    f = _factor(rng, _psd(rng, 35), 12)
    assert np.linalg.norm(f.U.T @ f.U - np.eye(12)) <= 1e-8
    assert np.all(np.diff(f.S) <= 0.0) and np.all(f.S >= 0.0)


def test_spectrum_interlaces_the_true_eigenvalues():
    rng = np.random.default_rng(105)
    M = _psd(rng, 44)
    top = np.linalg.eigvalsh(M)[::-1]
    slack = 44 * np.finfo(np.float64).eps * np.trace(M)
    for rank in (3, 17, 44):
        f = _factor(rng, M, rank)
        assert np.all(f.S <= top[:rank] + slack + 1e-12)


def test_error_shrinks_with_rank_on_nested_sketches():
    rng = np.random.default_rng(106)
    M = _psd(rng, 28)
    om = rng.standard_normal((28, 28))
    Y = M @ om
    errs = [np.linalg.norm(_lowrank(sap.rand_nystrom(Y, om, r)) - M) for r in (2, 6, 14, 28)]
    assert all(a >= b - 1e-12 for a, b in zip(errs, errs[1:]))


def test_retry_recovers_a_numerically_singular_block():
    t = np.linspace(0.0, 10.0, 50)[:, None]
    M = np.exp(-0.5 * (t - t.T) ** 2 / 0.6)
    om = np.random.default_rng(107).standard_normal((50, 50))
    f = sap.rand_nystrom_retry(M @ om, om, 50)
    assert np.linalg.norm(_lowrank(f) - M) <= 1e-6 * np.linalg.norm(M)


def test_rank_deficient_test_matrix_is_a_contract_error():
    rng = np.random.default_rng(108)
    M = _psd(rng, 10)
    om = rng.standard_normal((10, 5))
    om[:, 4] = 2.0 * om[:, 1]
    with pytest.raises(sap.ContractError):
        sap.rand_nystrom(M @ om, om, 5)


def test_nystrom_shape_and_rank_contracts():
    om = np.ones((6, 3))
    with pytest.raises(sap.ContractError):
        sap.rand_nystrom(np.ones((6, 2)), om, 2)
    with pytest.raises(sap.ContractError):
        sap.rand_nystrom(om, om, 4)
    with pytest.raises(sap.ContractError):
        sap.rand_nystrom(om, om, 0)


# ---------------------------------------------------------------------------
# Woodbury applies


@pytest.mark.parametrize("dim,rank,rho", [(5, 2, 1e-3), (40, 13, 0.4), (70, 30, 3.0)])
def test_apply_inv_solves_the_regularised_system(dim, rank, rho):
    rng = np.random.default_rng(200 + dim)
    f = _factor(rng, _psd(rng, dim), rank)
    P = _lowrank(f) + rho * np.eye(dim)
    G = rng.standard_normal((dim, 3))
    for g in (G[:, 0], G):
        want = np.linalg.solve(P, g)
        for fn in (sap.apply_inv, sap.apply_inv_plain):
            got = fn(f, rho, g)
            assert got.shape == g.shape
            assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)


def test_apply_inv_of_empty_factor_and_zero_vector():
    f = sap.NystromFactor.empty(7)
    g = np.linspace(-1.0, 1.0, 7)
    np.testing.assert_allclose(sap.apply_inv(f, 4.0, g), g / 4.0, rtol=1e-15)
    np.testing.assert_allclose(sap.apply_inv_sqrt(f, 4.0, g), g / 2.0, rtol=1e-15)
    rng = np.random.default_rng(201)
    f2 = _factor(rng, _psd(rng, 7), 3)
    assert np.all(sap.apply_inv(f2, 0.5, np.zeros(7)) == 0.0)


def test_apply_inv_with_zero_modes_in_the_spectrum():
    rng = np.random.default_rng(202)
    U, _ = np.linalg.qr(rng.standard_normal((14, 4)))
    f = sap.NystromFactor(U, np.array([3.0, 0.5, 0.0, 0.0]))
    rho = 0.2
    g = rng.standard_normal(14)
    want = np.linalg.solve(_lowrank(f) + rho * np.eye(14), g)
    assert np.linalg.norm(sap.apply_inv(f, rho, g) - want) < 1e-10


def test_apply_inv_sqrt_scales_range_and_complement():
    rng = np.random.default_rng(203)
    U, _ = np.linalg.qr(rng.standard_normal((16, 5)))
    s, rho = 2.5, 0.1
    f = sap.NystromFactor(U, np.full(5, s))
    inside = U @ rng.standard_normal(5)
    np.testing.assert_allclose(sap.apply_inv_sqrt(f, rho, inside), inside / np.sqrt(s + rho),
                               atol=1e-13)
    v = rng.standard_normal(16)
    outside = v - U @ (U.T @ v)
    np.testing.assert_allclose(sap.apply_inv_sqrt(f, rho, outside), outside / np.sqrt(rho),
                               atol=1e-13)


def test_apply_inv_sqrt_twice_is_the_inverse():
    rng = np.random.default_rng(204)
    f = _factor(rng, _psd(rng, 20), 9)
    rho = 0.35
    V = rng.standard_normal((20, 2))
    twice = sap.apply_inv_sqrt(f, rho, sap.apply_inv_sqrt(f, rho, V))
    assert np.linalg.norm(twice - sap.apply_inv_plain(f, rho, V)) <= 1e-10 * np.linalg.norm(V)


def test_applies_reject_nonpositive_rho():
    f = sap.NystromFactor.empty(3)
    for fn in (sap.apply_inv, sap.apply_inv_plain, sap.apply_inv_sqrt):
        with pytest.raises(sap.ContractError):
            fn(f, 0.0, np.ones(3))


# ---------------------------------------------------------------------------
# power-iteration stepsize


def test_stepsize_of_a_scaled_identity():
    eta = sap.rand_power_stepsize(lambda v: 4.0 * v, sap.NystromFactor.empty(9), 2.0, seed=3)
    assert eta == pytest.approx(0.5, rel=1e-12)


def test_stepsize_with_an_exact_preconditioner_is_one():
    rng = np.random.default_rng(301)
    f = _factor(rng, _psd(rng, 18), 6)
    rho = 0.15
    P = _lowrank(f) + rho * np.eye(18)
    assert abs(sap.rand_power_stepsize(lambda v: P @ v, f, rho, seed=2) - 1.0) <= 1e-6


def test_stepsize_errors():
    f = sap.NystromFactor.empty(4)
    with pytest.raises(sap.ContractError):
        sap.rand_power_stepsize(lambda v: v, f, 1.0, iters=0)
    with pytest.raises(sap.NumericalError):
        sap.rand_power_stepsize(lambda v: -v, f, 1.0)


# ---------------------------------------------------------------------------
# kernel values and blocks


FAMILIES = ("rbf", "matern32", "matern52")


def test_kernel_value_at_zero_distance_is_the_variance():
    x = np.array([1.1, -0.4, 0.25])
    for fam in FAMILIES:
        spec = sap.KernelSpec(fam, np.array([0.3, 1.0, 2.2]), 0.8)
        assert sap.kernel_eval(spec, x, x) == pytest.approx(0.8, rel=1e-6)


def test_kernel_values_against_closed_forms():
    forms = {
        "rbf": lambda r: np.exp(-0.5 * r * r),
        "matern32": lambda r: (1 + np.sqrt(3) * r) * np.exp(-np.sqrt(3) * r),
        "matern52": lambda r: (1 + np.sqrt(5) * r + 5 * r * r / 3) * np.exp(-np.sqrt(5) * r),
    }
    ls, var = 1.7, 0.6
    pts = np.array([[0.0], [0.4], [1.3], [2.9], [5.0]])
    for fam, form in forms.items():
        spec = sap.KernelSpec(fam, np.array([ls]), var)
        o = sap.KernelOracle(spec, pts, 0.1)
        K = o.dense()
        want = var * form(np.abs(pts - pts.T) / ls)
        np.testing.assert_allclose(K, want, rtol=1e-12, atol=1e-15)
        for j in range(1, 5):
            assert sap.kernel_eval(spec, pts[0], pts[j]) == pytest.approx(want[0, j], rel=1e-6)


def test_kernels_decay_monotonically_and_are_symmetric():
    rng = np.random.default_rng(401)
    for fam in FAMILIES:
        spec = sap.KernelSpec(fam, np.array([0.9, 1.4]), 1.0)
        vals = [sap.kernel_eval(spec, np.zeros(2), np.array([r, 0.0])) for r in (0.5, 1, 2, 4)]
        assert all(a > b > 0.0 for a, b in zip(vals, vals[1:]))
        for _ in range(5):
            x, y = rng.standard_normal(2), rng.standard_normal(2)
            assert sap.kernel_eval(spec, x, y) == sap.kernel_eval(spec, y, x)


def test_kernel_dimension_mismatch_is_a_contract_error():
    spec = sap.KernelSpec("rbf", np.ones(2), 1.0)
    with pytest.raises(sap.ContractError):
        sap.kernel_eval(spec, np.zeros(2), np.zeros(3))


@pytest.mark.parametrize("fam", FAMILIES)
def test_block_rows_and_block_match_the_dense_matrix(fam):
    rng = np.random.default_rng(402)
    X = rng.standard_normal((90, 4))
    o = sap.KernelOracle(sap.KernelSpec(fam, np.array([0.7, 1.2, 0.9, 2.0]), 1.4), X, 0.1)
    K = o.dense()
    B = np.sort(rng.choice(90, 23, replace=False))
    M = rng.standard_normal((90, 5))
    got = sap.block_rows_times(o, B, M)
    assert np.abs(got - K[B] @ M).max() <= 1e-5 * np.abs(K[B] @ M).max()
    assert np.abs(sap.block_block(o, B) - K[np.ix_(B, B)]).max() <= 1e-12


def test_block_rows_of_zero_and_of_a_basis_vector():
    rng = np.random.default_rng(403)
    o = sap.KernelOracle(sap.KernelSpec("matern32", np.ones(3), 2.3),
                         rng.standard_normal((25, 3)), 0.5)
    assert np.all(sap.block_rows_times(o, np.array([2, 9, 11]), np.zeros((25, 3))) == 0.0)
    e = np.zeros(25)
    e[9] = 1.0
    out = sap.block_rows_times(o, np.array([9]), e)
    assert out.reshape(-1)[0] == pytest.approx(2.3, rel=1e-6)


def test_dense_matrix_is_symmetric_psd_with_variance_diagonal():
    rng = np.random.default_rng(404)
    for fam in FAMILIES:
        o = sap.KernelOracle(sap.KernelSpec(fam, np.array([0.6, 0.6]), 1.9),
                             rng.standard_normal((40, 2)), 1e-3)
        K = o.dense()
        assert np.abs(K - K.T).max() == 0.0
        assert np.all(np.diag(K) == 1.9)
        assert np.linalg.eigvalsh(K).min() >= -1e-10


def test_duplicate_block_indices_are_rejected():
    rng = np.random.default_rng(405)
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.ones(2), 1.0), rng.standard_normal((8, 2)), 0.5)
    with pytest.raises(sap.ContractError):
        sap.block_block(o, np.array([0, 3, 3]))


def test_full_matmul_and_cross_matmul_match_dense():
    rng = np.random.default_rng(406)
    X = rng.standard_normal((600, 3))
    spec = sap.KernelSpec("matern52", np.array([0.8, 1.0, 1.3]), 1.0)
    o = sap.KernelOracle(spec, X, 0.5)
    K = o.dense()
    M = rng.standard_normal((600, 4))
    assert np.abs(o.matmul(M) - K @ M).max() <= 1e-5 * np.abs(K @ M).max()
    Xs = rng.standard_normal((11, 3))
    w = rng.standard_normal(600)
    want = sap.cross_kernel(spec, Xs, X) @ w
    assert np.abs(o.cross_matmul(Xs, w) - want).max() <= 1e-5 * np.abs(want).max()


# ---------------------------------------------------------------------------
# exact sketch-and-project


def test_sap_one_full_block_step_is_the_direct_solve():
    rng = np.random.default_rng(501)
    X = rng.uniform(-1, 1, size=(40, 2))
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.array([0.5, 0.5]), 1.0), X, 0.3)
    Y = rng.standard_normal((40, 2))
    want = np.linalg.solve(o.dense() + 0.3 * np.eye(40), Y)
    res = sap.solve(o, Y, sap.RunConfig(lam=0.3, solver_id="sap", blocksize=40, max_iters=1,
                                        residual_every=0))
    assert np.linalg.norm(res.W - want) <= 1e-8 * np.linalg.norm(want)


def test_sap_single_point_system():
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.ones(1), 1.0), np.zeros((1, 1)), 0.25)
    res = sap.solve(o, np.array([3.0]), sap.RunConfig(lam=0.25, solver_id="sap", blocksize=1,
                                                      max_iters=1, residual_every=0))
    assert float(np.ravel(res.W)[0]) == pytest.approx(3.0 / 1.25, rel=1e-12)


def test_sap_zero_rhs_stays_zero():
    rng = np.random.default_rng(502)
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.ones(2), 1.0), rng.standard_normal((24, 2)), 0.5)
    cfg = sap.RunConfig(lam=0.5, solver_id="sap", blocksize=6, max_iters=20, residual_every=5)
    res = sap.solve(o, np.zeros(24), cfg)
    assert np.all(res.W == 0.0)
    assert res.trace.final_residual() == 0.0
