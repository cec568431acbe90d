"""Synthetic GP problems for parity tests and benchmarks.

All randomness comes from named substreams of one root seed, so the same
(n, d, family, m, seed) always yields the same arrays:

* X ~ N(0,1)^{(n+t) x d}, z-scored with the sample std (data.py:147-178);
  the first n rows train, the last t rows are the held-out test set
  (1% of n, capped at 10^4);
* kernel: ``family`` with ARD lengthscales sqrt(d) and variance 1;
* y = f(X) + eps, f one random-feature prior draw (q=2048 features,
  gp.py:49-70), eps ~ N(0, lam); targets z-scored on the train part;
* RHS: [y, y - f_s(X) - zeta_s] for s = m-1 prior draws, exactly the
  pathwise-conditioning layout of gp.py:215-221 (streams "prior", "zeta").

The feature products run chunked in float64 with torch, on the GPU when a
device is given (the n=10^6 bench problem), else on the host CPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .rng import standard_normal, substream


@dataclass
class Problem:
    X: np.ndarray          # (n, d) training inputs
    y: np.ndarray          # (n,)   standardised targets
    Y: np.ndarray          # (n, m) right-hand sides [y, y - f_s - zeta_s]
    Xtest: np.ndarray      # (t, d)
    ytest: np.ndarray      # (t,)
    f_test: np.ndarray     # (t, m-1) prior draws at the test points
    family: str
    lengthscales: np.ndarray
    variance: float
    lam: float

    @property
    def n(self):
        return self.X.shape[0]

    def spec(self):
        from .kernels import KernelSpec
        return KernelSpec(self.family, self.lengthscales, self.variance)


def _standardize_cols(A):
    mu = A.mean(axis=0)
    sd = A.std(axis=0, ddof=1) if A.shape[0] > 1 else np.ones(A.shape[1:])
    sd = np.where(sd > 0.0, sd, 1.0)
    return (A - mu) / sd


def feature_map(family, lengthscales, q, rng):
    """Random Fourier frequencies/phases for the family (gp.py:49-63)."""
    d = lengthscales.size
    normal = rng.standard_normal((q, d))
    if family == "rbf":
        freq = normal
    elif family == "matern32":
        freq = normal * np.sqrt(3.0 / rng.chisquare(3.0, size=(q, 1)))
    else:
        freq = normal * np.sqrt(5.0 / rng.chisquare(5.0, size=(q, 1)))
    freq = freq / lengthscales
    phases = rng.uniform(0.0, 2.0 * np.pi, size=q)
    return freq, phases


def features_times(freq, phases, variance, X, theta, device=None, chunk=65536):
    """phi(X) @ theta with phi = sqrt(2 var / q) cos(X F^T + p), never
    materialising phi for all rows (gp.py:65-70): on a CUDA device the fused
    tensor-core product (kernels.cos_features_times), else -- shapes outside
    it, or host-only data generation -- chunked fp64 torch."""
    if device is not None and torch.device(device).type == "cuda":
        from .kernels import cos_features_times
        out = cos_features_times(freq, phases, variance, np.asarray(X, dtype=np.float64),
                                 np.asarray(theta, dtype=np.float64), device)
        if out is not None:
            return out.double().cpu().numpy()
    dev = torch.device(device) if device is not None else torch.device("cpu")
    F = torch.as_tensor(freq, dtype=torch.float64, device=dev)
    P = torch.as_tensor(phases, dtype=torch.float64, device=dev)
    T = torch.as_tensor(theta, dtype=torch.float64, device=dev)
    scale = math.sqrt(2.0 * variance / F.shape[0])
    out = np.empty((X.shape[0], T.shape[1]))
    for lo in range(0, X.shape[0], chunk):
        xb = torch.as_tensor(X[lo:lo + chunk], dtype=torch.float64, device=dev)
        out[lo:lo + chunk] = (scale * torch.cos(xb @ F.T + P) @ T).cpu().numpy()
    return out


def _n_test(n, test_fraction=0.01, test_cap=10_000):
    return max(1, min(test_cap, int(n * test_fraction)))


def _all_inputs(n, d, seed, t):
    return _standardize_cols(substream(seed, "synthetic_x").standard_normal((n + t, d)))


def make_inputs(n, d, seed=0, test_fraction=0.01, test_cap=10_000):
    """Training inputs of ``make_problem`` alone (no targets)."""
    return np.ascontiguousarray(_all_inputs(n, d, seed, _n_test(n, test_fraction, test_cap))[:n])


def make_problem(n, d, family="rbf", m=9, seed=0, lam=1e-2, q=2048,
                 test_fraction=0.01, test_cap=10_000, device=None, rhs="pathwise"):
    """Build the synthetic problem of SURVEY.md §8d.

    ``rhs="noise"`` replaces the s sample columns by N(0,1) draws (allowed
    for throughput-only runs; timing does not depend on the data).
    """
    t = _n_test(n, test_fraction, test_cap)
    Xall = _all_inputs(n, d, seed, t)
    ls = np.full(d, math.sqrt(d))
    var = 1.0
    freq, ph = feature_map(family, ls, q, substream(seed, "features"))
    s = m - 1
    th = np.concatenate([substream(seed, "truth").standard_normal((q, 1)),
                         substream(seed, "prior").standard_normal((q, s))], axis=1)
    if rhs == "pathwise":
        vals = features_times(freq, ph, var, Xall, th, device)
    else:
        vals = features_times(freq, ph, var, Xall, th[:, :1], device)
    f_truth = vals[:, 0]
    yall = f_truth + math.sqrt(lam) * substream(seed, "noise").standard_normal(n + t)
    ymu, ysd = yall[:n].mean(), yall[:n].std(ddof=1)
    yall = (yall - ymu) / ysd
    y = yall[:n]
    if rhs == "pathwise":
        z = standard_normal(substream(seed, "zeta"), (n, s), device)
        zeta = math.sqrt(lam) * (z.cpu().numpy() if torch.is_tensor(z) else z)
        Y = np.concatenate([y[:, None], y[:, None] - vals[:n, 1:] - zeta], axis=1)
        f_test = vals[n:, 1:]
    else:
        Y = np.concatenate([y[:, None], substream(seed, "zeta").standard_normal((n, s))], axis=1)
        f_test = np.zeros((t, s))
    return Problem(np.ascontiguousarray(Xall[:n]), y, np.ascontiguousarray(Y),
                   np.ascontiguousarray(Xall[n:]), yall[n:], f_test,
                   family, ls, var, lam)


@dataclass
class DeviceProblem:
    """``make_problem``'s problem with the right-hand sides built on the device:
    ``Ycm`` is the (m x n) fp32 column-major buffer the solver adopts without a
    copy (pass ``Ycm.T``); X, y and the test set stay on the host."""
    X: np.ndarray
    y: np.ndarray
    Ycm: "torch.Tensor"
    Xtest: np.ndarray
    ytest: np.ndarray
    f_test: np.ndarray
    family: str
    lengthscales: np.ndarray
    variance: float
    lam: float

    @property
    def n(self):
        return self.X.shape[0]

    def spec(self):
        from .kernels import KernelSpec
        return KernelSpec(self.family, self.lengthscales, self.variance)


def make_problem_device(n, d, family="rbf", m=65, seed=0, lam=1e-2, q=2048, device="cuda",
                        chunk_rows=4_000_000, test_fraction=0.01, test_cap=10_000):
    """``make_problem`` (pathwise right-hand sides) for sizes whose n x m
    host arrays would not fit: the same named streams, the prior draws f_s(X)
    by the fused tensor-core cosine product, zeta by the device sampler in
    row chunks that continue the numpy stream exactly
    (``rng.standard_normal_chunks``), each chunk of [y, y - f_s - zeta]
    written straight into the solver's column-major fp32 layout. Equal to
    make_problem's arrays up to the fp32 cosine product (~5e-5)."""
    from .kernels import cos_features_times
    from .rng import standard_normal_chunks
    dev = torch.device(device)
    t = _n_test(n, test_fraction, test_cap)
    Xall = _all_inputs(n, d, seed, t)
    ls = np.full(d, math.sqrt(d))
    var = 1.0
    freq, ph = feature_map(family, ls, q, substream(seed, "features"))
    s = m - 1
    th = np.concatenate([substream(seed, "truth").standard_normal((q, 1)),
                         substream(seed, "prior").standard_normal((q, s))], axis=1)

    def feats(X, theta):
        out = cos_features_times(freq, ph, var, X, theta, dev)
        if out is None:
            out = torch.as_tensor(features_times(freq, ph, var, X, theta, dev), device=dev)
        return out

    f_truth = np.empty(n + t)
    for lo in range(0, n + t, chunk_rows):
        hi = min(n + t, lo + chunk_rows)
        f_truth[lo:hi] = feats(Xall[lo:hi], th[:, :1])[:, 0].double().cpu().numpy()
    yall = f_truth + math.sqrt(lam) * substream(seed, "noise").standard_normal(n + t)
    ymu, ysd = yall[:n].mean(), yall[:n].std(ddof=1)
    yall = (yall - ymu) / ysd
    y = yall[:n]
    Ycm = torch.empty((m, n), dtype=torch.float32, device=dev)
    sq = math.sqrt(lam)
    for lo, hi, z in standard_normal_chunks(substream(seed, "zeta"), n, s, dev, chunk_rows):
        yc = torch.as_tensor(y[lo:hi], device=dev)
        f = feats(Xall[lo:hi], th[:, 1:]).double()
        Ycm[0, lo:hi] = yc.float()
        Ycm[1:, lo:hi] = (yc[:, None] - f - sq * z).T.float()
    f_test = feats(Xall[n:], th[:, 1:]).double().cpu().numpy()
    return DeviceProblem(np.ascontiguousarray(Xall[:n]), y, Ycm, np.ascontiguousarray(Xall[n:]),
                         yall[n:], f_test, family, ls, var, lam)
