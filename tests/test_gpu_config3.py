"""Parity at the headline shapes against the live reference (fixtures written
by tests/golden/make_golden.py from /root/reference; inputs regenerated here
from the same named substreams):

* config 3 (n=1e6, d=9, b=2000, m=65): one block product K[B,:]Z per family
  (Matern-3/2, RBF) within 1e-4 (dist.py:108-127), a 5-iteration Matern-3/2
  ADASAP trajectory (block crc32s equal, stepsizes within 1e-4, sampled rows
  of W within 1e-3; solvers.py:361-456), and the hot-path fp32 K_BB tile
  (sap_ktile_f32_batch) against the oracle's block (kernels.py:129-136);
* config 2 (n=1e5, d=11, RBF, b=1000, m=65, pathwise right-hand sides) for one
  pass (100 iterations): crc32s, stepsizes, sampled rows of W, the posterior
  mean at the 1000 test points and the test RMSE within 1e-3.
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

import paper_2505_13723_b200 as sap  # noqa: E402
from paper_2505_13723_b200 import kernels as K  # noqa: E402
from paper_2505_13723_b200 import synthetic  # noqa: E402
from paper_2505_13723_b200.rng import substream  # noqa: E402

N3, D3, B3, M3 = 1_000_000, 9, 2000, 65
TOL_BLOCK = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def rel(got, ref):
    return np.abs(np.asarray(got) - ref).max() / max(np.abs(ref).max(), 1e-300)


def fixture(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    return np.load(path)


@pytest.fixture(scope="module")
def x3():
    return synthetic.make_inputs(N3, D3, 0)


def spec3(fam):
    return sap.KernelSpec(fam, np.full(D3, np.sqrt(D3)), 1.0)


@pytest.mark.parametrize("fam", ["matern32", "rbf"])
def test_config3_block_product_matches_reference(fam, x3):
    g = fixture("config3.npz")
    Z = substream(0, "golden_z3").standard_normal((N3, M3))
    o = sap.KernelOracle(spec3(fam), x3, 1e-2)
    got = sap.col_dist_matmul(o, Z, g[f"{fam}_B"])
    assert rel(got, g[f"{fam}_G"]) < TOL_BLOCK


def test_config3_trajectory_matches_reference(x3):
    g = fixture("config3.npz")
    Y = substream(0, "golden_y3").standard_normal((N3, M3))
    o = sap.KernelOracle(spec3("matern32"), x3, 1e-2)
    cfg = sap.RunConfig(lam=1e-2, blocksize=B3, nystrom_rank=100, residual_every=0, seed=0,
                        max_iters=5)
    res = sap.adasap_solve(o, Y, cfg)
    crcs = np.array([r.block_hash for r in res.trace.records])
    assert np.array_equal(crcs, g["traj_crc"])
    etas = np.array([r.stepsize for r in res.trace.records])
    assert np.abs(etas - g["traj_eta"]).max() / np.abs(g["traj_eta"]).max() < 1e-4
    assert rel(res.W[g["traj_rows"]], g["traj_W_rows"]) < 1e-3
    cn = np.linalg.norm(res.W, axis=0)
    assert np.abs(cn - g["traj_W_colnorm"]).max() / g["traj_W_colnorm"].max() < 1e-3


@pytest.mark.parametrize("fam", ["matern32", "rbf"])
def test_hot_path_kbb_tile_matches_oracle(fam, x3):
    """The lookahead's fp32 K_BB (sap_ktile_f32_batch), the power iteration's
    operand, against the oracle's block_block (fp64) at b = 2000, n = 1e6."""
    from oracle import sapgp_oracle as orc
    dev = torch.device("cuda", 0)
    o = sap.KernelOracle(spec3(fam), x3, 1e-2, device=dev)
    pts = o.points
    blocks = [orc.uniform_block(0, t, N3, B3) for t in range(2)]
    Xb = torch.empty((2, B3, pts.ldx), dtype=torch.float32, device=dev)
    rsq = torch.empty((2, B3), dtype=torch.float32, device=dev)
    for q, blk in enumerate(blocks):
        pts.gather(torch.as_tensor(blk, device=dev), out=(Xb[q], rsq[q]))
    out = torch.zeros((2, B3, B3), dtype=torch.float32, device=dev)
    K.ktile_f32_batch(o.spec, Xb, rsq, pts.d, out)
    P = orc.Points(fam, np.full(D3, np.sqrt(D3)), 1.0, x3)
    for q, blk in enumerate(blocks):
        ref = orc.block_block(P, blk)
        got = out[q].double().cpu().numpy()
        assert rel(got, ref) < 1e-5
        assert np.array_equal(np.diag(got), np.full(B3, 1.0))  # exact variance diagonal


def test_config2_one_pass_trajectory_and_prediction():
    g = fixture("config2_traj.npz")
    prob = synthetic.make_problem(100_000, 11, "rbf", 65, seed=0, lam=1e-2)  # host RHS
    # the regenerated right-hand sides are the fixture's (host fp64 arithmetic)
    assert rel(np.linalg.norm(prob.Y, axis=0), g["Y_colnorm"]) < 1e-12
    o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
    cfg = sap.RunConfig(lam=prob.lam, blocksize=1000, nystrom_rank=100, residual_every=0, seed=0,
                        max_passes=1.0)
    res = sap.adasap_solve(o, prob.Y, cfg)
    assert res.iterations == int(g["iters"]) == 100
    crcs = np.array([r.block_hash for r in res.trace.records])
    assert np.array_equal(crcs, g["crc"])
    etas = np.array([r.stepsize for r in res.trace.records])
    assert np.abs(etas - g["eta"]).max() / np.abs(g["eta"]).max() < 1e-4
    assert rel(res.W[g["rows"]], g["W_rows"]) < 1e-3
    mean = o.cross_matmul(prob.Xtest, res.W)
    assert rel(mean, g["test_mean"]) < 1e-3
    rm = sap.rmse(mean[:, 0], prob.ytest)
    assert abs(rm - float(g["test_rmse"])) / float(g["test_rmse"]) < 1e-3
