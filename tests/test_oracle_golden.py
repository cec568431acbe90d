"""Pin the CPU oracle against fixtures produced by the real reference.

The fixtures were written by tests/golden/make_golden.py running the
unmodified reference package; every check here is oracle-vs-reference.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import sapgp_oracle as orc
from paper_2505_13723_b200 import synthetic

FAMILIES = ("rbf", "matern32", "matern52")


def load(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.mark.parametrize("fam", FAMILIES)
def test_small_block_products(fam):
    g = load("kernels_small.npz")
    pts = orc.Points(fam, g["ls"], float(g["var"]), g["X"])
    np.testing.assert_array_equal(orc.col_dist_matmul(pts, g["M"], g["B"]), g[f"{fam}_KBM"])
    np.testing.assert_array_equal(orc.block_block(pts, g["B"]), g[f"{fam}_KBB"])
    np.testing.assert_array_equal(orc.row_dist_matmul(pts, g["omega"], g["B"]), g[f"{fam}_KBBom"])
    np.testing.assert_allclose(orc.cross_matmul(pts, g["ls"], g["Xs"], g["M"]),
                               g[f"{fam}_cross"], rtol=0, atol=1e-13)
    p300 = orc.Points(fam, g["ls"], float(g["var"]), g["X300"])
    np.testing.assert_allclose(orc.full_matmul(p300, g["M300"]), g[f"{fam}_matmul300"],
                               rtol=0, atol=1e-12)


def test_worker_count_bitwise():
    g = load("kernels_small.npz")
    pts = orc.Points("matern32", g["ls"], 1.3, g["X300"])
    B = np.sort(np.random.default_rng(0).choice(300, 40, replace=False))
    ref = orc.col_dist_matmul(pts, g["M300"], B)
    for w in (2, 4):
        assert np.array_equal(orc.col_dist_matmul(pts, g["M300"], B, workers=w), ref)


def test_rng_blocks():
    g = load("rng.npz")
    for seed, n, b, t, crc, first, last in g["rows"]:
        if n > 1_000_000:
            continue  # the 1e7 draw is slow on CPU; covered by the GPU-box test
        blk = orc.uniform_block(seed, t, n, b)
        assert orc.block_crc(blk) == crc and blk[0] == first and blk[-1] == last
    np.testing.assert_array_equal(orc.substream(0, "omega", 3).standard_normal((5, 4)), g["omega"])
    np.testing.assert_array_equal(orc.substream(0, "power", 3).standard_normal(6), g["power"])


def test_randnla():
    g = load("randnla.npz")
    U, S = orc.rand_nystrom_retry(g["Kbb"] @ g["omega"], g["omega"], 100)
    np.testing.assert_allclose(S, g["S"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(U @ U.T, g["P"], atol=1e-9)
    rho = float(S[-1]) + 1e-2
    assert rho == pytest.approx(float(g["rho"]), rel=1e-9)
    np.testing.assert_allclose(orc.apply_inv(U, S, rho, g["g"]), g["inv"], rtol=1e-8, atol=1e-8)
    np.testing.assert_allclose(orc.apply_inv_sqrt(U, S, rho, g["g"]), g["inv_sqrt"],
                               rtol=1e-8, atol=1e-8)
    Kbb = g["Kbb"]
    eta = orc.rand_power_stepsize(lambda v: Kbb @ v + 1e-2 * v, U, S, rho, 10,
                                  orc.substream(0, "power", 1))
    assert eta == pytest.approx(float(g["eta"]), rel=1e-9)


def test_config1_first_iterations():
    g = load("config1.npz")
    pts = orc.Points("rbf", g["ls"], 1.0, g["X"])
    lam, b, r = 1e-2, 200, 100
    co = orc.accel_coeffs(lam, 2000, b)
    W = np.zeros_like(g["Y"])
    V, Z = W.copy(), W.copy()
    for t in range(5):
        np.testing.assert_allclose(Z, g[f"t{t}_Z"], rtol=0, atol=1e-9)
        rec = {}
        W, V, Z, eta, blk = orc.adasap_step(pts, lam, g["Y"], W, V, Z, t, 0, b, r, co,
                                            record=rec)
        np.testing.assert_array_equal(blk, g[f"t{t}_block"])
        np.testing.assert_allclose(rec["G"], g[f"t{t}_G"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(rec["S"], g[f"t{t}_S"], rtol=1e-8, atol=1e-10)
        assert eta == pytest.approx(float(g[f"t{t}_eta"]), rel=1e-8)
        np.testing.assert_allclose(W, g[f"t{t}_W"], rtol=0, atol=1e-8)


def test_synthetic_problem_matches_fixture():
    g = load("config1.npz")
    prob = synthetic.make_problem(2000, 8, "rbf", 9, seed=0, lam=1e-2)
    np.testing.assert_array_equal(prob.X, g["X"])
    np.testing.assert_allclose(prob.Y, g["Y"], rtol=0, atol=1e-12)


@pytest.mark.slow
def test_config1_full_solve():
    g = load("config1.npz")
    pts = orc.Points("rbf", g["ls"], 1.0, g["X"])
    W, etas, crcs, _ = orc.adasap_solve(pts, 1e-2, g["Y"], 500, 0, 200, 100)
    np.testing.assert_array_equal(crcs, g["crc"])
    np.testing.assert_allclose(etas, g["eta"], rtol=1e-7)
    np.testing.assert_allclose(W, g["final_W"], rtol=0, atol=1e-6 * np.abs(g["final_W"]).max())


def test_oracle_baselines_match_reference():
    """Exact SAP, SDD and (P)CG restatements against the reference's own runs
    (tests/golden/baselines.npz, solvers.py:269-584)."""
    g = np.load(os.path.join(GOLDEN, "baselines.npz"))
    c1 = np.load(os.path.join(GOLDEN, "config1.npz"))
    pts = orc.Points("rbf", c1["ls"], 1.0, c1["X"])
    est, res, crcs = orc.sdd_solve(pts, 1e-2, c1["Y"], 400, 0, 200, 10.0, residual_every=50,
                                   workers=4)
    assert np.array_equal(crcs, g["sdd_crc"])
    np.testing.assert_allclose(est, g["sdd_W"], rtol=0, atol=1e-9 * np.abs(g["sdd_W"]).max())
    np.testing.assert_allclose(res, g["sdd_res"], rtol=1e-9)
    W, res, crcs = orc.sap_solve(pts, 1e-2, c1["Y"], 60, 0, 200, residual_every=10, workers=4)
    assert np.array_equal(crcs, g["sap_crc"])
    np.testing.assert_allclose(W, g["sap_W"], rtol=0, atol=1e-9 * np.abs(g["sap_W"]).max())
    np.testing.assert_allclose(res, g["sap_res"], rtol=1e-8)
    for tag, rank in (("pcg", 100), ("cg", 0)):
        X, res, it = orc.pcg_solve(pts, 1e-2, c1["Y"], 40, 0, rank)
        assert it == int(g[f"{tag}_iters"])
        np.testing.assert_allclose(X, g[f"{tag}_W"], rtol=0,
                                   atol=1e-7 * np.abs(g[f"{tag}_W"]).max())
        np.testing.assert_allclose(res, g[f"{tag}_res"], rtol=1e-6)
