"""The lookahead's Nystrom factorisation on the device (randnla.factor_gram_batch
with the Jacobi eigensolver sap_sym_eig_batch): eigenpairs against numpy, and
the reference's failure semantics (rand_nystrom_retry, randnla.py:52-106:
shift ladder 1, 1e4, 1e8, then NumericalError; negative trace) against
outcomes the live reference produced (tests/golden/nystrom_failures.npz)."""

import os
import types

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

import paper_2505_13723_b200 as sap  # noqa: E402
from paper_2505_13723_b200 import randnla  # noqa: E402
from paper_2505_13723_b200.pipeline import Lookahead  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("backend", ["cusolver", "jacobi"])
@pytest.mark.parametrize("r,count", [(100, 6), (7, 3), (150, 2), (1, 2)])
def test_eigensolver_matches_numpy(r, count, backend, monkeypatch):
    monkeypatch.setenv("SAP_EIG", backend)
    rng = np.random.default_rng(r)
    mats = []
    for q in range(count):
        A = rng.standard_normal((r, r + 3))
        M = A @ A.T
        if q == 1 and r > 4:  # repeated eigenvalues and a null space
            ev, Q = np.linalg.eigh(M)
            ev[:3] = 0.0
            ev[3:5] = ev[5]
            M = Q @ np.diag(ev) @ Q.T
        mats.append(M)
    H = torch.as_tensor(np.stack(mats), device="cuda")
    ev, V, sweeps = randnla.sym_eig_batch(H.clone())
    assert bool((sweeps >= 0).all())
    for q, M in enumerate(mats):
        ref = np.linalg.eigvalsh(M)[::-1]
        got = ev[q].cpu().numpy()
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        Vq = V[q].cpu().numpy()
        assert np.abs(Vq.T @ Vq - np.eye(r)).max() < 1e-12
        assert np.abs(Vq @ np.diag(got) @ Vq.T - M).max() <= 1e-12 * np.abs(M).max()


def test_factor_failure_semantics_match_reference():
    g = np.load(os.path.join(GOLDEN, "nystrom_failures.npz"))
    names = [str(x) for x in g["names"]]
    trip = []
    for nm in names:
        sk, om = g[f"{nm}_sketch"], g[f"{nm}_omega"]
        trip.append((sk.T @ sk, om.T @ sk, om.T @ om))
    G = [torch.as_tensor(np.stack([t[k] for t in trip]), device="cuda") for k in range(3)]
    r = trip[0][0].shape[0]
    W, S, rho, Mc, E, flags = randnla.factor_gram_batch(G[0], G[1], G[2], r, 1e-2)
    flags = flags.cpu().numpy()
    for i, nm in enumerate(names):
        err = str(g[f"{nm}_error"])
        if "negative trace" in err:
            assert flags[i] & randnla.FLAG_NEG_TRACE
        elif err:
            assert flags[i] & randnla.FLAG_CHOLESKY
        else:
            assert flags[i] == 0
            ref = g[f"{nm}_S"]
            top = ref > 1e-6 * ref.max()
            np.testing.assert_allclose(S[i].cpu().numpy()[top], ref[top], rtol=1e-8)
    # the lookahead raises the reference's exceptions from the flags
    for bit, msg in ((randnla.FLAG_NEG_TRACE, "negative trace; M is not PSD"),
                     (randnla.FLAG_CHOLESKY, "Cholesky of the shifted Gram failed")):
        slot = types.SimpleNamespace(normals=None,
                                     bad=torch.tensor([0, bit], dtype=torch.int32, device="cuda"))
        with pytest.raises(sap.NumericalError, match=msg):
            Lookahead.check_flags(types.SimpleNamespace(slots=[slot]))
    slot = types.SimpleNamespace(normals=None, bad=torch.tensor([randnla.FLAG_PLAIN],
                                                                dtype=torch.int32, device="cuda"))
    with pytest.warns(RuntimeWarning):
        Lookahead.check_flags(types.SimpleNamespace(slots=[slot]))
