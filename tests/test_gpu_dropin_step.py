"""The per-step API as a drop-in (solvers.py:189-202, :361-403): reference-style
code -- ``SolverState.zeros`` + a loop of ``adasap_step`` -- runs unchanged
against this package and follows the reference's own iterates.

Fixtures: tests/golden/config1.npz holds the reference's adasap_step iterates
(W, stepsize, block) for t = 0..4 at config 1 (n=2000, d=8, b=200, m=9, r=100).
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

import paper_2505_13723_b200 as sap  # noqa: E402
from paper_2505_13723_b200.solvers import SolverState, adasap_step  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def rel(got, ref):
    return np.abs(np.asarray(got) - ref).max() / max(np.abs(ref).max(), 1e-300)


def _config1():
    g = np.load(os.path.join(GOLDEN, "config1.npz"))
    o = sap.KernelOracle(sap.KernelSpec("rbf", g["ls"], 1.0), g["X"], 1e-2)
    cfg = sap.RunConfig(lam=1e-2, blocksize=200, nystrom_rank=100, residual_every=0, seed=0)
    return g, o, cfg


def test_reference_style_step_loop_matches_reference_iterates():
    g, o, cfg = _config1()
    n, m = g["Y"].shape
    accel = sap.resolve_accel(cfg, n, 200)
    # the reference's own pattern (tests/test_solvers.py:199-219, golden/make_golden.py)
    state = SolverState.zeros(n, m, accelerated=True)
    for t in range(5):
        assert state.iteration == t
        state, eta, block = adasap_step(o, state, g["Y"], cfg, accel)
        assert np.array_equal(block, g[f"t{t}_block"])
        assert abs(eta - float(g[f"t{t}_eta"])) <= 1e-4 * abs(float(g[f"t{t}_eta"]))
        W = state.W  # written back lazily, a fresh float64 host array
        assert isinstance(W, np.ndarray) and W.dtype == np.float64 and W.shape == (n, m)
        assert rel(W, g[f"t{t}_W"]) < 1e-4
    assert state.iteration == 5


def test_resume_from_host_arrays_and_rebind_on_new_arguments():
    g, o, cfg = _config1()
    n, m = g["Y"].shape
    accel = sap.resolve_accel(cfg, n, 200)
    state = SolverState.zeros(n, m, accelerated=True)
    for _ in range(3):
        state, _, _ = adasap_step(o, state, g["Y"], cfg, accel)
    # a reference-style state built from plain arrays at iteration 3 resumes
    resumed = SolverState(state.W.copy(), state.V.copy(), state.Z.copy(), iteration=3)
    for t in (3, 4):
        resumed, eta, block = adasap_step(o, resumed, g["Y"], cfg, accel)
        assert np.array_equal(block, g[f"t{t}_block"])
    assert rel(resumed.W, g["t4_W"]) < 1e-4
    # a new Y object is read (the engine rebinds): a zero right-hand side from
    # a zero state stays at zero
    zero = SolverState.zeros(n, m, accelerated=True)
    Y0 = np.zeros_like(g["Y"])
    zero, _, _ = adasap_step(o, zero, g["Y"], cfg, accel)
    first = zero._e
    zero.W = np.zeros((n, m))
    zero.V = np.zeros((n, m))
    zero.Z = np.zeros((n, m))
    zero, _, _ = adasap_step(o, zero, Y0, cfg, accel)
    assert zero._e is not first
    assert np.abs(zero.W).max() == 0.0
    # assigning an array detaches the engine and resumes from the assignment
    state.W = state.W
    assert state._e is None


def test_identity_precond_and_no_acceleration_step_loop():
    """tests/test_solvers.py:221-239 through adasap_step: plain block
    coordinate descent with the power-iteration stepsize."""
    from oracle import sapgp_oracle as orc
    rng = np.random.default_rng(5)
    X = rng.uniform(-1, 1, size=(40, 2))
    spec = sap.KernelSpec("rbf", np.full(2, 0.5), 1.0)
    o = sap.KernelOracle(spec, X, 0.3)
    y = rng.standard_normal((40, 1))
    cfg = sap.RunConfig(lam=0.3, solver_id="adasap_i", blocksize=8, seed=11, residual_every=0)
    state = SolverState.zeros(40, 1)
    pts = orc.Points("rbf", np.full(2, 0.5), 1.0, X)
    K = orc.block_block(pts, np.arange(40))
    w = np.zeros((40, 1))
    for t in range(25):
        state, eta, block = adasap_step(o, state, y, cfg, sap.NO_ACCELERATION,
                                        identity_precond=True)
        ref_block = orc.uniform_block(11, t, 40, 8)
        assert np.array_equal(block, ref_block)
        grad = (K @ w)[block] + 0.3 * w[block] - y[block]
        w[block] -= eta * grad
    assert rel(state.W, w) < 1e-5


def test_budgeted_state_raises_contract_error_past_its_budget():
    g, o, cfg = _config1()
    n, m = g["Y"].shape
    accel = sap.resolve_accel(cfg, n, 200)
    Y = g["Y"]  # one array object: the budgeted engine stays bound
    st = sap.make_state(o, Y, cfg, accel, total=2)
    for _ in range(2):
        st, _, _ = adasap_step(o, st, Y, cfg, accel)
    with pytest.raises(sap.ContractError):
        adasap_step(o, st, Y, cfg, accel)
    st._e.close()


def test_prefaulted_readback_is_bitwise_the_plain_one(monkeypatch):
    """The W readback into the array pre-faulted at bind time
    (xfer.prefaulted, n*m >= 2^20 here) returns exactly what the plain
    readback returns, and a second read (no pre-faulted array left) too."""
    from paper_2505_13723_b200 import xfer
    rng = np.random.default_rng(5)
    n, d, m = 20000, 5, 65
    X = rng.standard_normal((n, d))
    Y = rng.standard_normal((n, m))
    o = sap.KernelOracle(sap.KernelSpec("matern32", np.full(d, 2.0), 1.0), X, 1e-2)
    cfg = sap.RunConfig(lam=1e-2, blocksize=500, nystrom_rank=50, residual_every=0, seed=3)
    accel = sap.resolve_accel(cfg, n, 500)
    out = []
    for threads in (4, 0):
        monkeypatch.setattr(xfer, "_PF_THREADS", threads)
        st = SolverState.zeros(n, m, accelerated=True)
        for _ in range(3):
            st, _, _ = adasap_step(o, st, Y, cfg, accel)
        if threads:
            assert st._e._readback is not None
        W = st.W
        assert W.shape == (n, m) and W.dtype == np.float64 and W.flags.c_contiguous
        st, _, _ = adasap_step(o, st, Y, cfg, accel)
        out.append((W, st.W))
        st.iteration = st.iteration  # detach: releases the engine
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])
    assert not np.array_equal(out[0][0], out[0][1])
