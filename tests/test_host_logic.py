"""Host-side logic of the drop-in API (no GPU): configuration parity with
the reference, partitioning, index checks, and the algebra of the lazy
two-array Nesterov state used by the engine."""

import math

import numpy as np
import pytest

import paper_2505_13723_b200 as sap
from oracle import sapgp_oracle as orc
from paper_2505_13723_b200 import dist, rng
from paper_2505_13723_b200.parallel import ShardInfo
from paper_2505_13723_b200.solvers import _basis, budget_iterations, resolve_blocksize


def test_runconfig_defaults_and_validation():
    c = sap.RunConfig()
    assert (c.lam, c.max_passes, c.residual_every, c.grad_eval_point) == (1e-3, 50.0, 1, "z")
    for bad in (dict(lam=0.0), dict(solver_id="x"), dict(grad_eval_point="q"), dict(seed=-1),
                dict(max_passes=None), dict(mu=-1.0), dict(blocksize=0), dict(residual_every=-1)):
        with pytest.raises(sap.ConfigError):
            sap.RunConfig(**bad)
    with pytest.raises(sap.ConfigError):
        sap.RunConfig.from_dict({"lam": 1.0, "bogus": 1})
    with pytest.raises(sap.ConfigError):
        sap.RunConfig(blocksize=10).validate_for(5)
    spec = sap.kernel_from_dict({"family": "matern32", "lengthscales": 2.0}, d=3)
    assert spec.lengthscales.tolist() == [2.0, 2.0, 2.0]


def test_budget_and_blocksize_defaults():
    c = sap.RunConfig()
    assert resolve_blocksize(c, 2000) == 20
    assert budget_iterations(c, 200 / 2000) == 500


def test_partition_matches_oracle():
    for size in (0, 1, 5, 17, 257, 1000):
        for parts in (1, 2, 3, 7):
            assert dist.partition(size, parts) == orc.partition(size, parts)
    assert dist.tile_ranges(1000) == orc.tile_ranges(1000)


def test_check_indices():
    for bad in ([], [0, 0], [-1], [10]):
        with pytest.raises(sap.ContractError):
            dist.check_indices(np.array(bad, dtype=np.int64), 10)


def test_block_draws_match_reference_fixture():
    from conftest import GOLDEN
    import os
    g = np.load(os.path.join(GOLDEN, "rng.npz"))
    for seed, n, b, t, crc, first, last in g["rows"]:
        blk = rng.uniform_block(seed, t, n, b)
        assert rng.block_hash(blk) == crc and blk[0] == first and blk[-1] == last


def _lazy_run(beta, gamma, alpha, steps=40, n=30, m=3, b=5, seed=0):
    """Replay the engine's basis algebra (M_t = [u1, s_t u2], scalar s) in fp64
    numpy and compare with the dense recurrence of solvers.py:76-85."""
    r = np.random.default_rng(seed)
    W = np.zeros((n, m)); V = W.copy(); Z = W.copy()
    P = np.zeros((n, m)); Q = np.zeros((n, m))
    u1, u2, lam2, dense = _basis(beta, alpha)
    assert not dense
    s = 1.0
    delta = np.array([-gamma, -(1 - alpha)])
    renorms = 0
    for _ in range(steps):
        B = np.sort(r.choice(n, b, replace=False))
        D = np.zeros((n, m)); D[B] = r.standard_normal((b, m))
        eta = r.uniform(0.1, 1.0)
        W, V, Z = orc.nesterov_update(W, V, Z, D, eta, beta, gamma, alpha)
        M = np.column_stack([u1, s * u2])
        Zt = M[1, 0] * P + M[1, 1] * Q
        WB = Zt[B] - eta * D[B]
        sn = lam2 * s
        e = np.linalg.solve(np.column_stack([u1, sn * u2]), delta)
        P[B] += e[0] * eta * D[B]
        Q[B] += e[1] * eta * D[B]
        Wl = M[1, 0] * P + M[1, 1] * Q
        Wl[B] = WB
        s = sn
        if abs(s) < 2.0 ** -20:
            Q *= s; s = 1.0; renorms += 1
        Mn = np.column_stack([u1, s * u2])
        Vl = Mn[0, 0] * P + Mn[0, 1] * Q
        Zl = Mn[1, 0] * P + Mn[1, 1] * Q
        sc = max(1.0, np.abs(Z).max())
        assert np.abs(Wl - W).max() <= 1e-9 * sc
        assert np.abs(Vl - V).max() <= 1e-9 * sc
        assert np.abs(Zl - Z).max() <= 1e-9 * sc
    return renorms


def test_lazy_nesterov_basis_reproduces_dense_update():
    co = orc.accel_coeffs(1e-2, 1_000_000, 2000)
    _lazy_run(*co)
    _lazy_run(*orc.accel_coeffs(0.3, 40, 8))
    assert _lazy_run(*orc.accel_coeffs(1e-3, 200, 2), steps=3000) > 0  # renormalisation
    assert _lazy_run(*orc.accel_coeffs(1.0, 200, 25), steps=400) > 10   # tests/test_solvers.py:242


def test_identity_accel_uses_trivial_basis():
    u1, u2, lam2, dense = _basis(1.0, 0.0)
    assert np.array_equal(np.column_stack([u1, u2]), np.eye(2)) and lam2 == 1.0 and not dense


def test_shard_info():
    for n in (1, 7, 1000):
        for world in (1, 2, 3, 8):
            shards = [ShardInfo.of(n, r, world) for r in range(world)]
            assert shards[0].lo == 0 and shards[-1].hi == n
            assert sum(s.size for s in shards) == n
            blk = np.arange(n)
            owners = sum((s.local_positions(blk) >= 0).astype(int) for s in shards)
            assert np.all(owners == 1)


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(sap.WorkerError):
        sap.KernelOracle(sap.KernelSpec("rbf", np.ones(2)), np.zeros((4, 2)), 0.1)


def test_batched_device_factor_matches_host_factor():
    """randnla.factor_gram_batch (the lookahead's batched factorisation; run here
    on CPU tensors with torch's eigh standing in for the device Jacobi solver,
    which tests/test_gpu_fused_step.py checks against numpy) equals the per-element host path factor_gram_retry +
    woodbury_core + rho + the P^{-1/2} coefficients, including an element that
    needs a shift escalation and one with pruned null modes."""
    import torch
    from paper_2505_13723_b200.randnla import (factor_gram_batch, factor_gram_retry,
                                               woodbury_core)
    rng = np.random.default_rng(4)
    b, r, lam = 300, 40, 1e-2
    trip = []
    for case in range(4):
        A = rng.standard_normal((b, b if case != 2 else 25))
        M = A @ A.T / b                      # case 2: rank 25 < r (null modes)
        Om = rng.standard_normal((b, r))
        Y = M @ Om
        if case == 3:                        # indefinite at the first shift
            Y = Y - 1e-9 * np.abs(Y).max() * Om
        trip.append((Y.T @ Y, Om.T @ Y, Om.T @ Om))
    G = [torch.as_tensor(np.stack([t[k] for t in trip])) for k in range(3)]

    def eig(H):  # the device Jacobi eigensolver's contract: descending, sweeps
        ev, V = torch.linalg.eigh(H)
        return ev.flip(-1), V.flip(-1), torch.zeros(H.shape[0], dtype=torch.int32)

    W, S, rho, Mc, E, flags = factor_gram_batch(G[0], G[1], G[2], r, lam, eig=eig)
    for i, (gyy, goy, goo) in enumerate(trip):
        Wh, Sh, UtU = factor_gram_retry(gyy, goy, goo, r)
        rho_h = float(Sh[-1]) + lam
        Mch = woodbury_core(Sh, UtU, rho_h)
        if i == 2:
            # rank-deficient sketch: its shifted Gram is PD only up to rounding, so
            # batched and unbatched LAPACK may settle on different shift levels;
            # the retained modes agree, the null tail (S ~ 1e-5, far below rho)
            # is rounding noise either way
            top = Sh > 1e-3 * Sh.max()
            np.testing.assert_allclose(S[i].numpy()[top], Sh[top], rtol=1e-6)
            continue
        np.testing.assert_allclose(S[i].numpy(), Sh, rtol=1e-9, atol=1e-12 * Sh.max())
        assert abs(float(rho[i]) - rho_h) <= 1e-9 * rho_h
        # eigenvectors are defined up to sign: compare the products that matter
        np.testing.assert_allclose((W[i] @ W[i].T).numpy(), Wh @ Wh.T, rtol=1e-7,
                                   atol=1e-9 * np.abs(Wh @ Wh.T).max())
        np.testing.assert_allclose((W[i] @ Mc[i] @ W[i].T).numpy(), Wh @ Mch @ Wh.T, rtol=1e-6,
                                   atol=1e-9 * np.abs(Wh @ Mch @ Wh.T).max())
        np.testing.assert_allclose(E[i].numpy(), 1.0 / np.sqrt(Sh + rho_h) - 1.0 / np.sqrt(rho_h),
                                   rtol=1e-8, atol=1e-12)
    assert not flags.any()


def test_prefaulted_readback_array(monkeypatch):
    """xfer.prefaulted: a C-contiguous float64 array of the asked shape whose
    pages the background threads have touched once the futures are done
    (every 512th element zeroed), page-aligned slices, and off with 0 threads."""
    from paper_2505_13723_b200 import xfer
    monkeypatch.setattr(xfer, "_PF_THREADS", 3)
    out, futs = xfer.prefaulted((1001, 7))
    for f in futs:
        f.result()
    assert out.shape == (1001, 7) and out.dtype == np.float64 and out.flags.c_contiguous
    assert len(futs) == 3
    assert np.all(out.reshape(-1)[::512] == 0.0)
    out0, futs0 = xfer.prefaulted((0, 5))
    assert out0.shape == (0, 5) and not futs0
    monkeypatch.setattr(xfer, "_PF_THREADS", 0)
    assert xfer.prefaulted((10, 10)) is None
