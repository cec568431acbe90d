"""Pathwise posterior sampling (gp.py:204-233) with the right-hand sides
assembled on the device (device_resident=True: fused tensor-core cosine
product for f(X), device zeta, no n x m host arrays) against the host path."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2505_13723_b200 as sap  # noqa: E402
from paper_2505_13723_b200 import gp, synthetic  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def test_device_resident_pathwise_matches_host_path():
    n, d, s = 6000, 9, 16
    prob = synthetic.make_problem(n, d, "matern32", s + 1, seed=2, lam=1e-2)
    o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
    rfm = gp.RandomFeatureMap.sample(prob.spec(), 1024, 7)
    prior = gp.RandomFeaturePrior(rfm, prob.X, prob.Xtest)
    cfg = sap.RunConfig(lam=prob.lam, blocksize=600, nystrom_rank=60, max_iters=60,
                        residual_every=0, seed=1)

    def solve_fn(oracle, Y):
        return sap.adasap_solve(oracle, Y, cfg).W

    host = gp.pathwise_sample(o, prior, prob.y, s, 11, solve_fn, Xstar=prob.Xtest)
    dev = gp.pathwise_sample(o, prior, prob.y, s, 11, solve_fn, Xstar=prob.Xtest,
                             device_resident=True)
    assert torch.is_tensor(dev.sample_weights) and dev.sample_weights.is_cuda
    ref = host.sample_values
    # fp32 cosine features on the tensor cores vs the fp64 host product: ~5e-5
    assert np.abs(dev.sample_values - ref).max() / np.abs(ref).max() < 1e-3
    assert np.abs(dev.mean_values - host.mean_values).max() / np.abs(host.mean_values).max() < 1e-4


def test_device_problem_builder_matches_host_generator():
    """synthetic.make_problem_device (the n = 1e8 path: chunked device zeta
    continuing the numpy stream, fused cosine products, column-major fp32)
    equals make_problem's host arrays up to the fp32 cosine product."""
    n, d, m = 30_000, 9, 17
    host = synthetic.make_problem(n, d, "matern32", m, seed=4, lam=1e-2)
    dev = synthetic.make_problem_device(n, d, "matern32", m, seed=4, lam=1e-2, device="cuda",
                                        chunk_rows=7_000)
    assert np.array_equal(dev.X, host.X) and np.array_equal(dev.Xtest, host.Xtest)
    np.testing.assert_allclose(dev.y, host.y, rtol=0, atol=1e-4)
    Y = dev.Ycm.T.double().cpu().numpy()
    assert np.abs(Y - host.Y).max() / np.abs(host.Y).max() < 1e-4
    assert np.abs(dev.f_test - host.f_test).max() / np.abs(host.f_test).max() < 1e-4
