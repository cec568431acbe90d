"""CPU oracle for the ADASAP hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference algorithm (the
`sapgp` package, arXiv 2505.13723) for exactly the functions on the B200
hot path. It exists to *check* the CUDA path and to serve as the timed CPU
baseline in ``bench.py``. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
it. The product package ``paper_2505_13723_b200`` never imports it and
fails loudly when its CUDA library is missing.

Parity status: PINNED. ``tests/golden/make_golden.py`` runs the real
reference (imported from /root/reference in the build container) and writes
the fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks
this restatement against every one of them.

Every function cites the reference location it restates
(paths relative to /root/reference/pkg/src/sapgp/).
"""

from __future__ import annotations

import math
import os
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg

EPS64 = np.finfo(np.float64).eps
COL_TILE = 256  # dist.py:19 -- the fixed tile width of the ordered reduction


class OracleError(Exception):
    """Raised where the reference raises one of its SapgpError subclasses."""

    def __init__(self, kind, message):
        super().__init__(message)
        self.kind = kind  # "contract" | "numerical" | "config"


# ---------------------------------------------------------------------------
# random substreams  (rng.py:14-24)


def substream(seed, name, *idx):
    key = [int(seed), zlib.crc32(name.encode("utf-8"))] + [int(i) for i in idx]
    return np.random.default_rng(np.random.SeedSequence(key))


def uniform_block(seed, t, n, b):
    """solvers.py:260-262 -- sorted uniform block without replacement."""
    return np.sort(substream(seed, "block", t).choice(n, size=b, replace=False))


def block_crc(block):
    """solvers.py:250-251 -- crc32 of the int64 index bytes."""
    return zlib.crc32(np.ascontiguousarray(block).tobytes())


# ---------------------------------------------------------------------------
# kernel values  (kernels.py:45-66)


def scaled_points(X, lengthscales):
    """kernels.py:45-53 -- X / lengthscale (scalar or ARD)."""
    X = np.asarray(X, dtype=np.float64)
    ls = np.atleast_1d(np.asarray(lengthscales, dtype=np.float64))
    if ls.size not in (1, X.shape[1]):
        raise OracleError("contract", "lengthscale size mismatch")
    return X / ls


def family_values(family, variance, sq):
    """kernels.py:56-66 -- clamp at zero, then the family transform."""
    sq = np.maximum(sq, 0.0)
    if family == "rbf":
        return variance * np.exp(-0.5 * sq)
    r = np.sqrt(sq)
    if family == "matern32":
        a = math.sqrt(3.0) * r
        return variance * (1.0 + a) * np.exp(-a)
    if family == "matern52":
        a = math.sqrt(5.0) * r
        return variance * (1.0 + a + (5.0 / 3.0) * sq) * np.exp(-a)
    raise OracleError("contract", f"unknown family {family!r}")


class Points:
    """Pre-scaled points plus squared row norms (kernels.py:100-112)."""

    def __init__(self, family, lengthscales, variance, X):
        self.family = family
        self.variance = float(variance)
        self.Z = scaled_points(X, lengthscales)
        self.sqn = np.einsum("ij,ij->i", self.Z, self.Z)

    @property
    def n(self):
        return self.Z.shape[0]

    def tile(self, rows, cols):
        """kernels.py:118-127 -- expansion-form distances, exact diagonal."""
        rows = np.asarray(rows, dtype=np.intp)
        cols = np.asarray(cols, dtype=np.intp)
        sq = (self.sqn[rows][:, None] + self.sqn[cols][None, :]
              - 2.0 * self.Z[rows] @ self.Z[cols].T)
        sq[rows[:, None] == cols[None, :]] = 0.0
        return family_values(self.family, self.variance, sq)

    def cross_tile(self, Zs, sqs, start, stop):
        """kernels.py:170-175 -- external rows, no diagonal rule."""
        sq = sqs[:, None] + self.sqn[start:stop][None, :] - 2.0 * Zs @ self.Z[start:stop].T
        return family_values(self.family, self.variance, sq)


# ---------------------------------------------------------------------------
# partitioned products  (dist.py)


def partition(size, parts):
    """dist.py:22-35 -- contiguous ranges whose sizes differ by at most one."""
    parts = min(parts, max(size, 1))
    q, rem = divmod(size, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + q + (1 if i < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


def tile_ranges(size):
    """dist.py:38-40."""
    return partition(size, max(1, math.ceil(size / COL_TILE)))


def check_block(block, n):
    """dist.py:96-105."""
    block = np.asarray(block, dtype=np.intp).ravel()
    if block.size == 0:
        raise OracleError("contract", "empty index block")
    if block.min() < 0 or block.max() >= n:
        raise OracleError("contract", "block index out of range")
    if np.unique(block).size != block.size:
        raise OracleError("contract", "duplicate index in block")
    return block


def _ordered_map(fn, count, workers):
    if workers <= 1 or count <= 1:
        return [fn(i) for i in range(count)]
    groups = partition(count, min(workers, count))
    with ThreadPoolExecutor(max_workers=len(groups)) as ex:
        futs = [ex.submit(lambda g: [fn(i) for i in range(*g)], g) for g in groups]
        out = []
        for f in futs:
            out.extend(f.result())
    return out


def col_dist_matmul(pts, W, block, workers=1):
    """dist.py:108-127 -- K[block, :] @ W summed in ascending tile order."""
    block = check_block(block, pts.n)
    W = np.asarray(W, dtype=np.float64)
    vec = W.ndim == 1
    W2 = W[:, None] if vec else W
    tiles = tile_ranges(pts.n)
    parts = _ordered_map(
        lambda i: pts.tile(block, np.arange(*tiles[i])) @ W2[tiles[i][0]:tiles[i][1]],
        len(tiles), workers)
    acc = np.zeros((block.size, W2.shape[1]))
    for p in parts:
        acc += p
    return acc[:, 0] if vec else acc


def row_dist_matmul(pts, omega, block, workers=1):
    """dist.py:130-147 -- K[block, block] @ omega by row tiles."""
    block = check_block(block, pts.n)
    omega = np.asarray(omega, dtype=np.float64)
    vec = omega.ndim == 1
    om = omega[:, None] if vec else omega
    tiles = tile_ranges(block.size)
    parts = _ordered_map(
        lambda i: pts.tile(block[tiles[i][0]:tiles[i][1]], block) @ om,
        len(tiles), workers)
    out = np.vstack(parts)
    return out[:, 0] if vec else out


def block_block(pts, block):
    """kernels.py:129-136 -- exactly symmetric K[B,B] with diag = variance."""
    block = check_block(block, pts.n)
    t = pts.tile(block, block)
    up = np.triu(t, 1)
    out = up + up.T
    np.fill_diagonal(out, pts.variance)
    return out


def full_matmul(pts, M):
    """kernels.py:145-159 -- K @ M over 256x256 tiles."""
    M = np.asarray(M, dtype=np.float64)
    vec = M.ndim == 1
    M2 = M[:, None] if vec else M
    out = np.empty((pts.n, M2.shape[1]))
    for r0, r1 in tile_ranges(pts.n):
        rows = np.arange(r0, r1)
        acc = np.zeros((r1 - r0, M2.shape[1]))
        for c0, c1 in tile_ranges(pts.n):
            acc += pts.tile(rows, np.arange(c0, c1)) @ M2[c0:c1]
        out[r0:r1] = acc
    return out[:, 0] if vec else out


def cross_matmul(pts, lengthscales, Xstar, W):
    """kernels.py:161-176 -- k(Xstar, X) @ W tiled over training points."""
    W = np.asarray(W, dtype=np.float64)
    vec = W.ndim == 1
    W2 = W[:, None] if vec else W
    Zs = scaled_points(Xstar, lengthscales)
    sqs = np.einsum("ij,ij->i", Zs, Zs)
    out = np.zeros((Zs.shape[0], W2.shape[1]))
    for c0, c1 in tile_ranges(pts.n):
        out += pts.cross_tile(Zs, sqs, c0, c1) @ W2[c0:c1]
    return out[:, 0] if vec else out


# ---------------------------------------------------------------------------
# randomized NLA  (randnla.py)


def rand_nystrom(sketch, omega, rank, shift_scale=1.0):
    """randnla.py:52-94 -- shifted Gram, Cholesky, triangular solve, thin SVD."""
    sketch = np.asarray(sketch, dtype=np.float64)[:, :rank]
    omega = np.asarray(omega, dtype=np.float64)[:, :rank]
    gram = omega.T @ sketch
    gram = 0.5 * (gram + gram.T)
    shift = shift_scale * EPS64 * float(np.trace(gram))
    if shift < 0.0:
        raise OracleError("numerical", "negative Gram trace")
    shifted = gram + shift * (omega.T @ omega)
    if not shifted.any():
        half = np.zeros_like(sketch)
    else:
        try:
            C = scipy.linalg.cholesky(shifted)
        except scipy.linalg.LinAlgError as exc:
            if np.linalg.matrix_rank(omega) < rank:
                raise OracleError("contract", "rank deficient omega") from exc
            raise OracleError("numerical", "shifted Gram Cholesky failed") from exc
        half = scipy.linalg.solve_triangular(C, sketch.T, trans="T", lower=False).T
    U, sig, _ = np.linalg.svd(half, full_matrices=False)
    return U, np.maximum(sig * sig - shift, 0.0)


def rand_nystrom_retry(sketch, omega, rank, escalations=(1.0, 1e4, 1e8)):
    """randnla.py:97-106."""
    err = None
    for s in escalations:
        try:
            return rand_nystrom(sketch, omega, rank, s)
        except OracleError as exc:
            if exc.kind != "numerical":
                raise
            err = exc
    raise err


def apply_inv(U, S, rho, g):
    """randnla.py:109-134 -- Cholesky-stabilised Woodbury, zero modes pruned."""
    g = np.asarray(g, dtype=np.float64)
    keep = S > 0.0
    if not keep.any():
        return g / rho
    Uk, Sk = U[:, keep], S[keep]
    small = rho * np.diag(1.0 / Sk) + Uk.T @ Uk
    try:
        L = scipy.linalg.cho_factor(small, lower=True)
    except scipy.linalg.LinAlgError:
        return apply_inv_plain(U, S, rho, g)
    return (g - Uk @ scipy.linalg.cho_solve(L, Uk.T @ g)) / rho


def apply_inv_plain(U, S, rho, g):
    """randnla.py:137-148."""
    if S.size == 0:
        return g / rho
    Ut = U.T @ g
    sc = 1.0 / (S + rho)
    return U @ (Ut * (sc[:, None] if g.ndim == 2 else sc)) + (g - U @ Ut) / rho


def apply_inv_sqrt(U, S, rho, v):
    """randnla.py:151-162."""
    if S.size == 0:
        return v / math.sqrt(rho)
    Ut = U.T @ v
    sc = 1.0 / np.sqrt(S + rho)
    return U @ (Ut * (sc[:, None] if v.ndim == 2 else sc)) + (v - U @ Ut) / math.sqrt(rho)


def rand_power_stepsize(h_apply, U, S, rho, iters, rng):
    """randnla.py:165-196 -- 10-step normalised powering, eta = 1/Rayleigh."""
    v = rng.standard_normal(U.shape[0])
    nv = np.linalg.norm(v)
    if nv == 0.0:
        v = rng.standard_normal(U.shape[0])
        nv = np.linalg.norm(v)
    v = v / nv
    est = None
    for _ in range(iters):
        y = apply_inv_sqrt(U, S, rho, h_apply(apply_inv_sqrt(U, S, rho, v)))
        est = float(v @ y)
        ny = np.linalg.norm(y)
        if ny == 0.0:
            raise OracleError("numerical", "power iteration collapsed")
        v = y / ny
    if est is None or est <= 0.0:
        raise OracleError("numerical", "nonpositive Rayleigh estimate")
    return 1.0 / est


# ---------------------------------------------------------------------------
# ADASAP  (solvers.py)


def accel_coeffs(lam, n, b, mu="default", nu="default"):
    """solvers.py:32-53, :69-73 -- (beta, gamma, alpha) from (mu, nu)."""
    mu = lam if mu == "default" else float(mu)
    nu = n / b if nu == "default" else float(nu)
    gamma = 1.0 / math.sqrt(mu * nu)
    return 1.0 - math.sqrt(mu / nu), gamma, 1.0 / (1.0 + gamma * nu)


def nesterov_update(W, V, Z, D, eta, beta, gamma, alpha):
    """solvers.py:76-85 -- the Z blend uses the incoming V."""
    Wn = Z - eta * D
    Vn = beta * V + (1.0 - beta) * Z - (gamma * eta) * D
    Zn = alpha * V + (1.0 - alpha) * Wn
    return Wn, Vn, Zn


def adasap_step(pts, lam, Y, W, V, Z, t, seed, b, r, coeffs, workers=1,
                identity_precond=False, record=None):
    """solvers.py:361-403 -- one iteration; returns (W, V, Z, eta, block)."""
    n = pts.n
    block = uniform_block(seed, t, n, b)
    G = col_dist_matmul(pts, Z, block, workers)
    g = G + lam * Z[block] - Y[block]
    if identity_precond:
        U, S, rho = np.zeros((b, 0)), np.zeros(0), 1.0
    else:
        omega = substream(seed, "omega", t).standard_normal((b, r))
        sketch = row_dist_matmul(pts, omega, block, workers)
        U, S = rand_nystrom_retry(sketch, omega, r)
        rho = float(S[-1]) + lam
    Kbb = block_block(pts, block)
    eta = rand_power_stepsize(lambda v: Kbb @ v + lam * v, U, S, rho, 10,
                              substream(seed, "power", t))
    D = np.zeros_like(W)
    D[block] = apply_inv(U, S, rho, g)
    if record is not None:
        record.update(G=G, g=g, S=S, rho=rho, eta=eta, DB=D[block], block=block)
    W, V, Z = nesterov_update(W, V, Z, D, eta, *coeffs)
    return W, V, Z, eta, block


def adasap_solve(pts, lam, Y, iters, seed, b, r, coeffs=None, workers=1,
                 identity_precond=False, snapshots=()):
    """solvers.py:406-456 with residual_every=0 and no tail averaging.

    Returns the final W plus per-iteration (eta, crc32(block)) and the W
    iterates requested in ``snapshots`` (1-based iteration counts).
    """
    Y = np.asarray(Y, dtype=np.float64)
    vec = Y.ndim == 1
    Y2 = Y[:, None] if vec else Y
    if coeffs is None:
        coeffs = accel_coeffs(lam, pts.n, b)
    W = np.zeros_like(Y2)
    V, Z = W.copy(), W.copy()
    etas, crcs, snaps = [], [], {}
    for t in range(iters):
        W, V, Z, eta, block = adasap_step(pts, lam, Y2, W, V, Z, t, seed, b, r,
                                          coeffs, workers, identity_precond)
        etas.append(eta)
        crcs.append(block_crc(block))
        if t + 1 in snapshots:
            snaps[t + 1] = W.copy()
    return (W[:, 0] if vec else W), np.array(etas), np.array(crcs, dtype=np.int64), snaps


def relative_residual(pts, lam, W, Y):
    """solvers.py:254-257."""
    res = full_matmul(pts, W) + lam * W - Y
    return float(np.linalg.norm(res) / max(np.linalg.norm(Y), np.finfo(np.float64).tiny))


def rmse(pred, truth):
    """gp.py:240-245."""
    pred = np.asarray(pred, dtype=np.float64).ravel()
    truth = np.asarray(truth, dtype=np.float64).ravel()
    return float(np.sqrt(np.mean((pred - truth) ** 2)))


# ---------------------------------------------------------------------------
# baselines on the same operator  (solvers.py:463-584)

SDD_MOMENTUM = 0.9  # solvers.py:25


def _due(every, t, total):
    """solvers.py:351-354."""
    if every <= 0:
        return t == total - 1
    return (t + 1) % every == 0 or t == total - 1


def sap_solve(pts, lam, Y, iters, seed, b, residual_every=0, workers=1):
    """solvers.py:269-348 (uniform sampler, no tail averaging) -- exact projection
    steps: (K[B,B] + lam I) d = K[B,:] W + lam W[B] - Y[B] by one Cholesky,
    W[B] -= d. Returns (W, residual trace, crc32 per block)."""
    Y = np.asarray(Y, dtype=np.float64)
    Y2 = Y[:, None] if Y.ndim == 1 else Y
    W = np.zeros_like(Y2)
    res, crcs = [], []
    for t in range(iters):
        block = uniform_block(seed, t, pts.n, b)
        grad = col_dist_matmul(pts, W, block, workers) + lam * W[block] - Y2[block]
        H = block_block(pts, block)
        H[np.diag_indices_from(H)] += lam
        W[block] -= scipy.linalg.cho_solve(scipy.linalg.cho_factor(H, lower=True), grad)
        res.append(relative_residual(pts, lam, W, Y2) if _due(residual_every, t, iters)
                   else math.nan)
        crcs.append(block_crc(block))
    return (W[:, 0] if Y.ndim == 1 else W), np.array(res), np.array(crcs, dtype=np.int64)


def sdd_solve(pts, lam, Y, iters, seed, b, scale=10.0, residual_every=0, workers=1):
    """solvers.py:463-516 -- block stochastic dual descent: raw block gradient,
    stepsize scale/n, heavy-ball momentum 0.9, geometric averaging 100/T.
    Returns (estimate, residual trace (nan where not due), crc32 per block)."""
    Y = np.asarray(Y, dtype=np.float64)
    Y2 = Y[:, None] if Y.ndim == 1 else Y
    n = pts.n
    eta = scale / n
    avg = min(1.0, 100.0 / iters)
    w = np.zeros_like(Y2)
    vel = np.zeros_like(Y2)
    est = np.zeros_like(Y2)
    res, crcs = [], []
    for t in range(iters):
        block = uniform_block(seed, t, n, b)
        grad = col_dist_matmul(pts, w, block, workers) + lam * w[block] - Y2[block]
        vel *= SDD_MOMENTUM
        vel[block] -= eta * grad
        w += vel
        est += avg * (w - est)
        res.append(relative_residual(pts, lam, est, Y2) if _due(residual_every, t, iters)
                   else math.nan)
        crcs.append(block_crc(block))
    return (est[:, 0] if Y.ndim == 1 else est), np.array(res), np.array(crcs, dtype=np.int64)


def pcg_solve(pts, lam, Y, iters, seed, rank, tol=1e-6):
    """solvers.py:519-584 -- CG on (K + lam I) W = Y with a global rank-r
    Nystrom preconditioner (Omega from substream(seed, "omega"), sketch K Omega),
    per-column recurrences, columns frozen once below tol. Returns (X,
    residual trace, iterations)."""
    Y = np.asarray(Y, dtype=np.float64)
    Y2 = Y[:, None] if Y.ndim == 1 else Y
    n = pts.n
    if rank > 0:
        omega = substream(seed, "omega").standard_normal((n, rank))
        U, S = rand_nystrom_retry(full_matmul(pts, omega), omega, rank)
        rho = float(S[-1]) + lam
    else:
        U, S, rho = np.zeros((n, 0)), np.zeros(0), 1.0
    tiny = np.finfo(np.float64).tiny
    X = np.zeros_like(Y2)
    R = Y2.copy()
    Zp = apply_inv(U, S, rho, R)
    P = Zp.copy()
    rz = np.einsum("ij,ij->j", R, Zp)
    cn = np.maximum(np.linalg.norm(Y2, axis=0), tiny)
    yn = max(np.linalg.norm(Y2), tiny)
    res, done = [], 0
    for t in range(iters):
        active = np.linalg.norm(R, axis=0) / cn > tol
        if not np.any(active):
            break
        AP = full_matmul(pts, P) + lam * P
        pap = np.einsum("ij,ij->j", P, AP)
        if np.any(pap[active] <= 0.0):
            raise OracleError("numerical", "conjugate gradient breakdown")
        alpha = np.where(active, rz / np.where(pap > 0.0, pap, 1.0), 0.0)
        X += alpha * P
        R -= alpha * AP
        Zp = apply_inv(U, S, rho, R)
        rz_new = np.einsum("ij,ij->j", R, Zp)
        beta = np.where(active, rz_new / np.where(rz > 0.0, rz, 1.0), 0.0)
        P = Zp + beta * P
        rz = rz_new
        done = t + 1
        res.append(float(np.linalg.norm(R) / yn))
    return (X[:, 0] if Y.ndim == 1 else X), np.array(res), done


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
