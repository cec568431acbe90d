"""The reference's acceptance criteria for the hot path, run on the B200
implementation (tests/test_acceptance.py of the reference, same problems,
seeds and bars unless noted):

  #4 solver/oracle equivalence  test_acceptance.py:107-157
  #5 Nystrom and Woodbury        test_acceptance.py:160-193
  #6 randomized powering         test_acceptance.py:196-219
  #7 pathwise conditioning       test_acceptance.py:222-254

Deviation: block products are fp32-accurate (the reference is fp64), so #4's
PCG-versus-dense bar is 1e-5 instead of 1e-6.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sap = pytest.importorskip("paper_2505_13723_b200")


def _dense_solve(o, lam, y):
    return np.linalg.solve(o.dense() + lam * np.eye(o.n), y)


def test_criterion_04_solvers_reach_tolerance():
    rng = np.random.default_rng(6)
    # full-block exact step equals the direct solve
    Xs = rng.uniform(-1, 1, size=(200, 2))
    os_ = sap.KernelOracle(sap.KernelSpec("rbf", np.array([0.5, 0.5]), 1.0), Xs, 0.3)
    ys = rng.standard_normal(200)
    direct = _dense_solve(os_, 0.3, ys)
    full = sap.solve(os_, ys, sap.RunConfig(lam=0.3, solver_id="sap", blocksize=200, max_iters=1))
    assert np.linalg.norm(full.W - direct) / np.linalg.norm(direct) <= 1e-8
    n, lam = 500, 8.0
    X = rng.uniform(-1, 1, size=(n, 2))
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.array([0.15, 0.15]), 1.0), X, lam)
    y = rng.standard_normal(n)
    dense = _dense_solve(o, lam, y)
    ada = sap.solve(o, y, sap.RunConfig(lam=lam, solver_id="adasap", max_passes=50,
                                        residual_every=100, seed=7))
    sdd = sap.solve(o, y, sap.RunConfig(lam=lam, solver_id="sdd", stepsize_scale=1.0,
                                        max_passes=80, residual_every=100, seed=8))
    pcg = sap.solve(o, y, sap.RunConfig(lam=lam, solver_id="pcg", nystrom_rank=100, tol=1e-8,
                                        max_iters=n, seed=9))
    assert ada.trace.final_residual() <= 1e-4
    assert sdd.trace.final_residual() <= 1e-4
    assert pcg.trace.final_residual() <= 1e-4
    assert np.linalg.norm(pcg.W - dense) / np.linalg.norm(dense) <= 1e-5


def test_criterion_05_nystrom_and_woodbury():
    rng = np.random.default_rng(10)
    X = rng.uniform(-1, 1, size=(100, 2))
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.array([0.6, 0.6]), 1.0), X, 1e-3)
    block = np.sort(rng.choice(100, 48, replace=False))
    Kbb = o.block(block)
    omega = rng.standard_normal((48, 48))
    factor = sap.rand_nystrom(Kbb @ omega, omega, 48)
    recon = (factor.U * factor.S) @ factor.U.T
    assert np.linalg.norm(recon - Kbb) / np.linalg.norm(Kbb) <= 1e-8
    inv_err = sqrt_err = 0.0
    for dim, rank in ((16, 8), (48, 20), (64, 32)):
        G = rng.standard_normal((dim, dim))
        M = G @ G.T / dim
        om = rng.standard_normal((dim, rank))
        fac = sap.rand_nystrom(M @ om, om, rank)
        rho = float(fac.S[-1]) + 0.05
        g = rng.standard_normal(dim)
        dense = np.linalg.solve((fac.U * fac.S) @ fac.U.T + rho * np.eye(dim), g)
        got = sap.apply_inv(fac, rho, g)
        inv_err = max(inv_err, np.linalg.norm(got - dense) / np.linalg.norm(dense))
        twice = sap.apply_inv_sqrt(fac, rho, sap.apply_inv_sqrt(fac, rho, g))
        sqrt_err = max(sqrt_err, np.linalg.norm(twice - got) / np.linalg.norm(dense))
    assert inv_err <= 1e-10 and sqrt_err <= 1e-10


def test_criterion_06_randomized_powering():
    from paper_2505_13723_b200.rng import substream
    hits, lam = 0, 1e-2
    for seed in range(100):
        rng = np.random.default_rng(seed)
        G = rng.standard_normal((16, 16))
        M = G @ G.T / 16
        omega = rng.standard_normal((16, 8))
        factor = sap.rand_nystrom(M @ omega, omega, 8)
        rho = float(factor.S[-1]) + lam
        H = M + lam * np.eye(16)
        eta = sap.rand_power_stepsize(lambda v: H @ v, factor, rho, iters=10,
                                      seed=substream(seed, "power"))
        w, V = np.linalg.eigh((factor.U * factor.S) @ factor.U.T + rho * np.eye(16))
        half = (V / np.sqrt(w)) @ V.T
        top = np.linalg.eigvalsh(half @ H @ half)[-1]
        hits += abs(eta - 1.0 / top) <= 0.1 / top
    assert hits >= 95


def test_criterion_07_pathwise_conditioning():
    rng = np.random.default_rng(11)
    n, t, s, lam = 30, 5, 2000, 0.05
    X = rng.uniform(-2, 2, size=(n, 2))
    Xstar = rng.uniform(-2, 2, size=(t, 2))
    spec = sap.KernelSpec("rbf", np.array([0.8, 0.8]), 1.0)
    o = sap.KernelOracle(spec, X, lam)
    y = rng.standard_normal(n)
    K = o.dense()
    A = K + lam * np.eye(n)
    cross = sap.cross_kernel(spec, Xstar, X)
    exact_mean = cross @ np.linalg.solve(A, y)
    exact_cov = sap.cross_kernel(spec, Xstar, Xstar) - cross @ np.linalg.solve(A, cross.T)
    cfg = sap.RunConfig(lam=lam, solver_id="sap", blocksize=n, max_iters=1, residual_every=0)

    def solve_fn(orc, rhs):
        return sap.solve(orc, rhs, cfg).W

    prior = sap.ExactPrior(spec, X, Xstar)
    out = sap.pathwise_sample(o, prior, y, s, seed=12, solve_fn=solve_fn, Xstar=Xstar)
    mean_se = np.sqrt(np.diag(exact_cov) / s)
    mean_dev = np.max(np.abs(out.sample_mean() - exact_mean) / mean_se)
    var = np.diag(exact_cov)
    cov_se = np.sqrt((np.outer(var, var) + exact_cov ** 2) / s)
    cov_dev = np.max(np.abs(out.sample_covariance() - exact_cov) / cov_se)
    assert mean_dev <= 4.0 and cov_dev <= 4.0
