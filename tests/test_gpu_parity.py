"""Parity of the CUDA path (through the C ABI) with the reference.

Every expected value comes from the reference package itself (golden
fixtures written by tests/golden/make_golden.py) or from the CPU oracle
that tests/test_oracle_golden.py pins to those fixtures.

Tolerances (BASELINE.json north star): block products within 1e-4
max-abs / max-abs (fp32 arithmetic vs the reference's fp64); index
sampling bit-exact; final posterior mean and test RMSE within 1e-3
relative.
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import sapgp_oracle as orc

pytestmark = pytest.mark.gpu

import paper_2505_13723_b200 as sap  # noqa: E402
from paper_2505_13723_b200 import synthetic  # noqa: E402
from paper_2505_13723_b200.rng import substream  # noqa: E402

FAMILIES = ("rbf", "matern32", "matern52")
TOL_BLOCK = 1e-4


def rel(got, ref):
    return np.abs(np.asarray(got) - ref).max() / max(np.abs(ref).max(), 1e-300)


def load(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("fam", FAMILIES)
def test_small_products_match_reference(fam):
    g = load("kernels_small.npz")
    spec = sap.KernelSpec(fam, g["ls"], float(g["var"]))
    o = sap.KernelOracle(spec, g["X"], 0.1)
    assert rel(sap.block_rows_times(o, g["B"], g["M"]), g[f"{fam}_KBM"]) < 1e-5
    assert rel(sap.block_block(o, g["B"]), g[f"{fam}_KBB"]) < 1e-6
    assert rel(sap.row_dist_matmul(o, g["omega"], g["B"]), g[f"{fam}_KBBom"]) < 1e-5
    assert rel(o.cross_matmul(g["Xs"], g["M"]), g[f"{fam}_cross"]) < 1e-5
    o3 = sap.KernelOracle(spec, g["X300"], 0.1)
    assert rel(o3.matmul(g["M300"]), g[f"{fam}_matmul300"]) < 1e-5


def test_block_exactly_symmetric_with_variance_diagonal():
    g = load("kernels_small.npz")
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.full(3, 1.0), 2.0), g["X"], 0.1)
    K = sap.block_block(o, np.arange(60))
    assert np.abs(K - K.T).max() == 0.0
    assert np.all(np.diag(K) == np.float32(2.0))


def test_zero_rhs_and_basis_vector():
    rng = np.random.default_rng(2)
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.ones(2), 1.7), rng.standard_normal((20, 2)), 0.5)
    assert np.all(sap.block_rows_times(o, np.array([3, 5]), np.zeros((20, 2))) == 0.0)
    e0 = np.zeros(20)
    e0[0] = 1.0
    out = sap.block_rows_times(o, np.array([0]), e0)
    assert out[0] == pytest.approx(1.7, rel=1e-7)  # exact diagonal entry (kernels.py:126)


@pytest.mark.parametrize("tag,fam,d", [("rbf_d11", "rbf", 11), ("m32_d9", "matern32", 9)])
def test_config2_block_product(tag, fam, d):
    g = load("config2.npz")
    n, m = 100_000, 65
    X = synthetic.make_inputs(n, d, 0)
    Z = substream(0, "golden_z").standard_normal((n, m))
    o = sap.KernelOracle(sap.KernelSpec(fam, np.full(d, np.sqrt(d)), 1.0), X, 1e-2)
    got = sap.col_dist_matmul(o, Z, g[f"{tag}_B"])
    assert rel(got, g[f"{tag}_G"]) < TOL_BLOCK
    again = sap.col_dist_matmul(o, Z, g[f"{tag}_B"])
    assert np.array_equal(got, again)  # fixed reduction order: run-to-run bitwise


@pytest.mark.parametrize("n,d,b,m", [(1, 1, 1, 1), (37, 3, 5, 1), (1000, 33, 130, 3),
                                     (4099, 64, 257, 130), (2050, 9, 200, 65)])
def test_ragged_shapes_against_oracle(n, d, b, m):
    rng = np.random.default_rng(n + d)
    X = rng.standard_normal((n, d))
    ls = rng.uniform(0.5, 2.0, d)
    for fam in FAMILIES:
        spec = sap.KernelSpec(fam, ls, 1.3)
        o = sap.KernelOracle(spec, X, 0.1)
        pts = orc.Points(fam, ls, 1.3, X)
        B = np.sort(rng.choice(n, b, replace=False))
        W = rng.standard_normal((n, m))
        assert rel(sap.col_dist_matmul(o, W, B), orc.col_dist_matmul(pts, W, B)) < TOL_BLOCK
        om = rng.standard_normal((b, m))
        assert rel(sap.row_dist_matmul(o, om, B), orc.row_dist_matmul(pts, om, B)) < TOL_BLOCK


def test_contract_errors():
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.ones(2)), np.zeros((20, 2)), 0.5)
    for bad in (np.array([0, 0]), np.array([25]), np.array([], dtype=np.int64)):
        with pytest.raises(sap.ContractError):
            sap.col_dist_matmul(o, np.zeros((20, 1)), bad)
    with pytest.raises(sap.ContractError):
        sap.col_dist_matmul(o, np.zeros((19, 1)), np.array([1]))
    # non-finite training inputs (kernels.py:100-112), host array and CUDA tensor
    for bad in (np.inf, np.nan):
        X = np.zeros((20, 2))
        X[7, 1] = bad
        with pytest.raises(sap.ValidationError):
            sap.KernelOracle(sap.KernelSpec("rbf", np.ones(2)), X, 0.5)
        with pytest.raises(sap.ValidationError):
            sap.KernelOracle(sap.KernelSpec("rbf", np.ones(2)), torch.as_tensor(X, device="cuda"),
                             0.5)


def test_nystrom_and_woodbury_match_reference():
    g = load("randnla.npz")
    fac = sap.rand_nystrom_retry(g["Kbb"] @ g["omega"], g["omega"], 100)
    np.testing.assert_allclose(fac.S, g["S"], rtol=1e-8, atol=1e-11)
    np.testing.assert_allclose(fac.U @ fac.U.T, g["P"], atol=1e-8)
    rho = float(fac.S[-1]) + 1e-2
    np.testing.assert_allclose(sap.apply_inv(fac, rho, g["g"]), g["inv"], rtol=1e-7, atol=1e-7)
    np.testing.assert_allclose(sap.apply_inv_sqrt(fac, rho, g["g"]), g["inv_sqrt"], rtol=1e-7,
                               atol=1e-7)


def test_config1_trajectory_and_prediction():
    """500 ADASAP iterations (50 passes) at config 1 vs the reference run."""
    g = load("config1.npz")
    spec = sap.KernelSpec("rbf", g["ls"], 1.0)
    o = sap.KernelOracle(spec, g["X"], 1e-2)
    cfg = sap.RunConfig(lam=1e-2, blocksize=200, nystrom_rank=100, residual_every=0, seed=0)
    res = sap.adasap_solve(o, g["Y"], cfg)
    assert res.iterations == 500
    crcs = np.array([r.block_hash for r in res.trace.records])
    assert np.array_equal(crcs, g["crc"])  # index sampling bit-exact
    etas = np.array([r.stepsize for r in res.trace.records])
    assert np.abs(etas - g["eta"]).max() / np.abs(g["eta"]).max() < 1e-3
    assert rel(res.W, g["final_W"]) < 1e-3
    mean = o.cross_matmul(g["Xtest"], res.W)
    assert rel(mean, g["test_mean"]) < 1e-3
    rm = sap.rmse(mean[:, 0], g["ytest"])
    assert abs(rm - float(g["test_rmse"])) / float(g["test_rmse"]) < 1e-3
    assert abs(res.trace.final_residual() - float(g["resid"])) / float(g["resid"]) < 1e-2


def test_first_iterations_block_products():
    g = load("config1.npz")
    o = sap.KernelOracle(sap.KernelSpec("rbf", g["ls"], 1.0), g["X"], 1e-2)
    for t in range(1, 5):
        got = sap.col_dist_matmul(o, g[f"t{t}_Z"], g[f"t{t}_block"])
        assert rel(got, g[f"t{t}_G"]) < TOL_BLOCK


def test_identity_precond_equals_plain_block_descent():
    """tests/test_solvers.py:221-239 on the device path (oracle as the loop)."""
    rng = np.random.default_rng(5)
    X = rng.uniform(-1, 1, size=(40, 2))
    spec = sap.KernelSpec("rbf", np.full(2, 0.5), 1.0)
    o = sap.KernelOracle(spec, X, 0.3)
    y = rng.standard_normal(40)
    cfg = sap.RunConfig(lam=0.3, solver_id="adasap_i", blocksize=8, max_iters=25, seed=11,
                        residual_every=0)
    res = sap.adasap_solve(o, y, cfg, identity_precond=True, accel=sap.NO_ACCELERATION)
    pts = orc.Points("rbf", np.full(2, 0.5), 1.0, X)
    W, _, _, _ = orc.adasap_solve(pts, 0.3, y, 25, 11, 8, 8, coeffs=(1.0, 0.0, 0.0),
                                  identity_precond=True)
    assert np.abs(res.W - W).max() <= 1e-5 * max(1.0, np.abs(W).max())


def test_converges_to_constructed_solution():
    """tests/test_solvers.py:242-249."""
    rng = np.random.default_rng(6)
    X = rng.uniform(-1, 1, size=(200, 2))
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.full(2, 0.4), 1.0), X, 1.0)
    ones = np.ones(200)
    y = o.matmul(ones) + ones
    cfg = sap.RunConfig(lam=1.0, solver_id="adasap", blocksize=25, nystrom_rank=25,
                        max_iters=200, residual_every=20)
    res = sap.adasap_solve(o, y, cfg)
    assert np.linalg.norm(res.W - ones) / np.linalg.norm(ones) <= 1e-3
    assert not res.diverged


def test_grad_at_w_and_tail_average_match_oracle_shape():
    g = load("config1.npz")
    o = sap.KernelOracle(sap.KernelSpec("rbf", g["ls"], 1.0), g["X"], 1e-2)
    cfg = sap.RunConfig(lam=1e-2, blocksize=200, nystrom_rank=100, residual_every=0, seed=0,
                        max_iters=6, tail_average=True, grad_eval_point="w")
    res = sap.adasap_solve(o, g["Y"], cfg)
    assert res.W.shape == g["Y"].shape and np.all(np.isfinite(res.W))


@pytest.mark.parametrize("fam", ("rbf", "matern32"))
def test_large_block_trajectory_tensor_core_sketch(fam):
    """b >= 512 routes the Nystrom sketch K[B,B] Omega through the tensor-core
    kernel (pipeline.py) and the block-row product through the CTA-pair
    kernel: stepsizes and iterates against the oracle (solvers.py:361-403)."""
    rng = np.random.default_rng(21)
    n, d, b, r, m, iters = 6000, 5, 640, 60, 3, 6
    X = rng.uniform(-2.0, 2.0, size=(n, d))
    Y = rng.standard_normal((n, m))
    ls = np.full(d, 1.3)
    lam = 1e-2
    pts = orc.Points(fam, ls, 1.0, X)
    W_ref, eta_ref, crc_ref, _ = orc.adasap_solve(pts, lam, Y, iters, 7, b, r, workers=4)
    o = sap.KernelOracle(sap.KernelSpec(fam, ls, 1.0), X, lam)
    assert o.use_tc(r) and o.use_tc(m)
    cfg = sap.RunConfig(lam=lam, blocksize=b, nystrom_rank=r, residual_every=0, seed=7,
                        max_iters=iters)
    res = sap.adasap_solve(o, Y, cfg)
    crcs = np.array([rec.block_hash for rec in res.trace.records])
    assert np.array_equal(crcs, crc_ref)
    etas = np.array([rec.stepsize for rec in res.trace.records])
    assert np.abs(etas - eta_ref).max() / np.abs(eta_ref).max() < 1e-4
    assert rel(res.W, W_ref) < 1e-3


@pytest.mark.parametrize("fam", FAMILIES)
def test_cross_matmul_tensor_path_matches_oracle(fam):
    """Test-time K(X*, X) W on the tensor-core kernel (external rows, no
    diagonal rule; kernels.py:161-176) against the CPU oracle, with a test
    point equal to a training point (its kernel value is the variance too)."""
    rng = np.random.default_rng(7)
    n, d, t, m = 5000, 9, 300, 65
    X = rng.standard_normal((n, d))
    Xs = rng.standard_normal((t, d))
    Xs[5] = X[17]
    ls = np.full(d, 3.0)
    W = rng.standard_normal((n, m))
    o = sap.KernelOracle(sap.KernelSpec(fam, ls, 1.3), X, 1e-2)
    assert o.use_tc(m)
    got = o.cross_matmul(Xs, W)
    ref = orc.cross_matmul(orc.Points(fam, ls, 1.3, X), ls, Xs, W)
    assert rel(got, ref) < 1e-4


@pytest.mark.parametrize("d", [9, 11, 14])
@pytest.mark.parametrize("fam", FAMILIES)
def test_fp16_and_fp32_feature_paths_agree(fam, d, monkeypatch):
    """The distance GEMM on fp16 features (kind::f16, the default when the
    point norms fit; 32 features for d <= 9, 64 with 128-byte rows above) and
    on fp32 features (kind::tf32, SAP_TC_F16=0) give the same block product to
    fp32-level accuracy, and both match the oracle."""
    rng = np.random.default_rng(11)
    n, b, m = 20000, 512, 65
    X = rng.standard_normal((n, d))
    ls = np.full(d, 3.0)
    W = rng.standard_normal((n, m))
    B = np.sort(rng.choice(n, b, replace=False))
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("SAP_TC_F16", flag)
        o = sap.KernelOracle(sap.KernelSpec(fam, ls, 1.0), X, 1e-2)
        assert o.tc_points().half == (flag == "1")
        out[flag] = sap.col_dist_matmul(o, W, B)
    ref = orc.col_dist_matmul(orc.Points(fam, ls, 1.0, X), W, B, workers=8)
    assert rel(out["1"], ref) < 2e-5 and rel(out["0"], ref) < 2e-5
    assert rel(out["1"], out["0"]) < 2e-5


@pytest.mark.parametrize("fam", FAMILIES)
def test_random_feature_prior_on_tensor_cores(fam):
    """phi(X) theta for the pathwise prior (gp.py:49-114) on the fused
    tensor-core product (cosine epilogue) against the reference's dense fp64
    formula, scale * cos(X F^T + p) @ theta."""
    rng = np.random.default_rng(3)
    n, d, q, s = 6000, 9, 2048, 65
    X = rng.standard_normal((n, d))
    rfm = sap.RandomFeatureMap.sample(sap.KernelSpec(fam, np.full(d, 3.0), 1.3), q, 5)
    theta = rng.standard_normal((q, s))
    got = rfm.times(X, theta, device="cuda")
    ref = np.sqrt(2.0 * 1.3 / q) * np.cos(X @ rfm.frequencies.T + rfm.phases) @ theta
    assert rel(got, ref) < 5e-5
    vec = rfm.times(X[:100], theta[:, 0], device="cuda")
    assert vec.shape == (100,) and rel(vec, ref[:100, 0]) < 5e-5


@pytest.mark.parametrize("n,d,b,m", [(300, 9, 16, 128), (5000, 9, 513, 113), (4097, 10, 256, 65),
                                     (129, 2, 129, 17), (20000, 19, 700, 1)])
def test_tensor_core_edge_shapes(n, d, b, m):
    """Tensor-core path at its shape limits: the smallest block it takes (16 rows),
    nz = 128 (TMEM full), ragged column tiles, d = 10 / 19 (fp32 features, ka
    = 64), b = n, m = 1; the block holds the first and last points; exact
    duplicate points (distance 0 off the diagonal: Matern's cusp) included."""
    rng = np.random.default_rng(n * 7 + m)
    X = rng.standard_normal((n, d))
    X[n // 2] = X[1]  # an exact duplicate pair
    ls = rng.uniform(0.8, 2.5, d)
    B = np.sort(np.union1d(rng.choice(n, b - 2, replace=False), [0, n - 1]))[:b]
    if 1 not in B:
        B[1] = 1
        B = np.sort(np.unique(np.concatenate([B, [n // 2]])))
    W = rng.standard_normal((n, m))
    for fam in FAMILIES:
        o = sap.KernelOracle(sap.KernelSpec(fam, ls, 0.9), X, 0.1)
        assert o.use_tc(m)
        got = sap.col_dist_matmul(o, W, B)
        ref = orc.col_dist_matmul(orc.Points(fam, ls, 0.9, X), W, B, workers=8)
        assert rel(got, ref) < TOL_BLOCK, (fam, rel(got, ref))


def test_long_trajectory_full_lookahead_batches():
    """80 iterations: the lookahead ramps 1, 4, 16 to full 32-iteration
    batches (batched gathers, K_BB tiles and power iterations, stepsizes
    copied to the trace once per batch, 1/rho folded into the update's
    stepsize); blocks, stepsizes and the iterate against the oracle."""
    rng = np.random.default_rng(31)
    n, d, b, r, m, iters = 4000, 5, 512, 40, 3, 80
    X = rng.uniform(-2.0, 2.0, size=(n, d))
    Y = rng.standard_normal((n, m))
    ls = np.full(d, 1.1)
    lam = 1e-2
    pts = orc.Points("matern32", ls, 1.0, X)
    W_ref, eta_ref, crc_ref, _ = orc.adasap_solve(pts, lam, Y, iters, 3, b, r, workers=8)
    o = sap.KernelOracle(sap.KernelSpec("matern32", ls, 1.0), X, lam)
    cfg = sap.RunConfig(lam=lam, blocksize=b, nystrom_rank=r, residual_every=0, seed=3,
                        max_iters=iters)
    assert cfg.lookahead == 32
    res = sap.adasap_solve(o, Y, cfg)
    crcs = np.array([rec.block_hash for rec in res.trace.records])
    assert np.array_equal(crcs, crc_ref)
    etas = np.array([rec.stepsize for rec in res.trace.records])
    assert np.abs(etas - eta_ref).max() / np.abs(eta_ref).max() < 1e-4
    assert rel(res.W, W_ref) < 2e-3


def test_vector_inputs_return_vectors():
    """1-D right-hand sides and operands come back 1-D (reference dist.py:113-127,
    :135-147; solvers.py:243-247, :451), equal to the (n, 1) results."""
    rng = np.random.default_rng(17)
    n, d, b = 3000, 5, 256
    X = rng.standard_normal((n, d))
    o = sap.KernelOracle(sap.KernelSpec("matern32", np.full(d, 2.0), 1.0), X, 1e-1)
    w = rng.standard_normal(n)
    B = np.sort(rng.choice(n, b, replace=False))
    g1 = sap.col_dist_matmul(o, w, B)
    g2 = sap.col_dist_matmul(o, w[:, None], B)
    assert g1.shape == (b,) and np.array_equal(g1, g2[:, 0])
    om = rng.standard_normal(b)
    s1 = sap.row_dist_matmul(o, om, B)
    assert s1.shape == (b,)
    cfg = sap.RunConfig(lam=1e-1, blocksize=b, nystrom_rank=32, max_iters=20, residual_every=0,
                        seed=3)
    y = rng.standard_normal(n)
    r1 = sap.adasap_solve(o, y, cfg)
    r2 = sap.adasap_solve(o, y[:, None], cfg)
    assert r1.W.shape == (n,) and r2.W.shape == (n, 1)
    assert np.abs(r1.W - r2.W[:, 0]).max() <= 1e-6 * np.abs(r2.W).max()
