"""The SDD and Nystrom-PCG baselines on the B200 block product (SURVEY.md
§8f, row 3; reference solvers.py:463-584).

Both reuse the hot path: SDD's gradient is the same K[B,:] w block product
(``sap_krows_tc`` / ``sap_krows_times``) as ADASAP's Phase I, and PCG's
K P is the same kernel with every point as a row (rows = the shard,
columns = all points). What is new here:

* ``sdd_solve`` -- heavy-ball momentum 0.9 and geometric iterate averaging
  (solvers.py:487-493) as ONE fused dense pass over (velocity, w, estimate)
  plus a block-row scatter (``sap_sdd_update``); state column-major fp32,
  sharded over ranks like ADASAP's, one all-reduce of the b x m gradient;
* ``pcg_solve`` -- per-column CG recurrences in fp64 on the device with the
  rank-r Nystrom preconditioner applied as (R - U Mc U^T R) / rho
  (randnla.py:109-134), the n x n product on the tensor cores. One device
  (PCG needs every point's P in every product; a sharded PCG is future work).

Deviations: block products fp32-accurate (split-precision tensor cores, as
everywhere in this package); SDD state fp32 (reference fp64); the PCG
Omega draw runs on the GPU at scale (numpy-exact but for 1-ulp ziggurat-tail
values, rng.py).
"""

from __future__ import annotations

import math
from collections import deque
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _native as nat
from .errors import ConfigError, ContractError, NumericalError
from .kernels import KernelOracle, ZOperand, krows_tc, krows_times, to_colmajor
from .parallel import allreduce_sum_, current_shard, gather_rows
from .randnla import rand_nystrom_retry, woodbury_core
from .rng import native_blocks, standard_normal, substream

SDD_MOMENTUM = 0.9          # solvers.py:25
DIVERGENCE_FACTOR = 1e6     # solvers.py:24


class BlockFeed:
    """Sorted uniform blocks (solvers.py:260-262) drawn ahead on host threads and
    copied to the device through a ring of pinned buffers."""

    def __init__(self, seed, n, b, total, device, ahead=8, ring=4):
        self.seed, self.n, self.b, self.total, self.dev = seed, n, b, total, device
        self.pool = ThreadPoolExecutor(max_workers=2, thread_name_prefix="sap-blocks")
        self.futs = deque()
        self.next_t = 0
        self.ahead = ahead
        pin = torch.cuda.is_available()
        self.h = [torch.empty(b, dtype=torch.int64, pin_memory=pin) for _ in range(ring)]
        self.d = [torch.empty(b, dtype=torch.int64, device=device) for _ in range(ring)]
        self.ev = [None] * ring
        self.k = 0
        self._fill()

    def _draw(self, t):
        blocks, crcs = native_blocks(self.seed, t, 1, self.n, self.b)
        return blocks[0], crcs[0]

    def _fill(self):
        while self.next_t < self.total and len(self.futs) < self.ahead:
            self.futs.append(self.pool.submit(self._draw, self.next_t))
            self.next_t += 1

    def get(self):
        blk, crc = self.futs.popleft().result()
        self._fill()
        k = self.k
        self.k = (k + 1) % len(self.h)
        if self.ev[k] is not None:
            self.ev[k].synchronize()  # the copy issued `ring` steps ago is done
        self.h[k].numpy()[:] = blk
        self.d[k].copy_(self.h[k], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.ev[k] = ev
        return blk, crc, self.d[k]

    def close(self):
        self.pool.shutdown(wait=True)


def _relres_cm(oracle, shard, Xcm, Ycm, lam, ynorm):
    """||K X + lam X - Y||_F / ||Y||_F for a sharded column-major (m x ld) X
    (solvers.py:254-257); rows of this shard against all points."""
    nl = shard.size
    Xloc = Xcm[:, :nl].T
    Xfull = gather_rows(Xloc, oracle.n, shard).T.contiguous()
    if nl == 0:
        part = torch.zeros(1, dtype=torch.float64, device=oracle.device)
    else:
        ids = torch.arange(shard.lo, shard.hi, device=oracle.device, dtype=torch.int64)
        KX = oracle.rows_times_device(ids, Xfull.to(torch.float32).contiguous())
        res = KX.double() + lam * Xloc.double() - Ycm[:, :nl].T.double()
        part = (res * res).sum().reshape(1)
    allreduce_sum_(part)
    return float(torch.sqrt(part)) / ynorm


class SddEngine:
    """Device-resident block SDD iteration (solvers.py:478-493)."""

    def __init__(self, oracle, Y, config, total, shard=None):
        if not isinstance(oracle, KernelOracle):
            raise ContractError("the B200 solver needs a device KernelOracle")
        from .solvers import resolve_blocksize
        self.o, self.cfg, self.dev = oracle, config, oracle.device
        n = oracle.n
        self.n = n
        self.shard = shard if shard is not None else current_shard(n)
        Ya = np.asarray(Y, dtype=np.float64)
        if Ya.shape[0] != n:
            raise ContractError("right-hand side must have n rows")
        self.vector = Ya.ndim == 1
        Yl = Ya[self.shard.lo:self.shard.hi]
        Yl = Yl[:, None] if Yl.ndim == 1 else Yl
        self.m = Yl.shape[1]
        self.b = resolve_blocksize(config, n)
        self.lam = oracle.lam
        self.total = total
        self.eta = float(config.stepsize_scale) / n
        self.avg = min(1.0, 100.0 / total)
        nl = self.shard.size
        self.ld = max(4, (nl + 3) // 4 * 4)
        f32, m, b = torch.float32, self.m, self.b
        self.V = torch.zeros((m, self.ld), dtype=f32, device=self.dev)
        self.W = torch.zeros((m, self.ld), dtype=f32, device=self.dev)
        self.E = torch.zeros((m, self.ld), dtype=f32, device=self.dev)
        self.Y = to_colmajor(Yl, nl, self.dev, self.ld) if nl > 0 else \
            torch.zeros((m, self.ld), dtype=f32, device=self.dev)
        self.G = torch.empty((b, m), dtype=f32, device=self.dev)
        self.g = torch.empty((b, m), dtype=torch.float64, device=self.dev)
        self.VB = torch.empty((b, m), dtype=f32, device=self.dev)
        self.pos = torch.full((self.ld,), -1, dtype=torch.int32, device=self.dev)
        self.use_tc = oracle.use_tc(m) and b >= 16 and nl > 0
        if self.use_tc:
            self.tcp = oracle.tc_points(self.shard.lo, self.shard.hi)
            self.zop = ZOperand(m, nl, self.dev)
            self.RAg = torch.empty(((b + 255) // 256 * 256, self.tcp.ka), dtype=self.tcp.dtype,
                                   device=self.dev)
            need = nat.load().sap_krows_tc_workspace(b, m, nl)
        else:
            need = nat.load().sap_krows_workspace(b, m, max(nl, 1))
        self.ws = torch.empty(max(need // 4 + 1, 1), dtype=f32, device=self.dev)
        self.feed = BlockFeed(config.seed, n, b, total, self.dev)
        self.t = 0

    def close(self):
        self.feed.close()

    def step(self):
        blk, crc, bd = self.feed.get()
        sh, b, m = self.shard, self.b, self.m
        loc = sh.local_positions(bd)
        if sh.size > 0 and self.use_tc:
            self.zop.fill(self.W)
            self.tcp.gather_rows(bd, out=self.RAg)
            krows_tc(self.o.spec, self.tcp, self.RAg, b, bd, self.zop, self.G, ws=self.ws)
        elif sh.size > 0:
            pts = self.o.points
            Xb, rsq = pts.gather(bd)
            krows_times(self.o.spec, pts, Xb, rsq, bd, self.W, self.G, col_base=sh.lo,
                        ws=self.ws, ncols=sh.size, col_offset=sh.lo)
        else:
            self.G.zero_()
        # grad = K[B,:] w + lam w[B] - Y[B] (solvers.py:486)
        nat.call("sap_grad_gather", nat.ptr(self.G), self.G.stride(0), nat.ptr(self.W), None,
                 nat.ptr(self.Y), self.ld, 1.0, 0.0, nat.ptr(loc), b, m, self.lam,
                 nat.ptr(self.g), self.g.stride(0), nat.stream_handle())
        allreduce_sum_(self.g)
        nat.call("sap_sdd_update", nat.ptr(self.V), nat.ptr(self.W), nat.ptr(self.E), self.ld,
                 self.ld, m, nat.ptr(loc), b, nat.ptr(self.g), self.g.stride(0), self.eta,
                 SDD_MOMENTUM, self.avg, nat.ptr(self.VB), nat.ptr(self.pos),
                 nat.stream_handle())
        self.t += 1
        return blk, crc

    def estimate_local(self):
        return self.E[:, :self.shard.size].T

    def relative_residual(self, ynorm):
        return _relres_cm(self.o, self.shard, self.E, self.Y, self.lam, ynorm)


def sdd_solve(oracle, Y, config, pool=None, on_iterate=None):
    """Block stochastic dual descent with heavy-ball momentum and geometric
    iterate averaging (solvers.py:463-516): stepsize scale/n, momentum 0.9,
    averaging weight min(1, 100/T); a residual above 1e6 or a non-finite
    iterate marks divergence."""
    from .solvers import (ConvergenceTrace, SolveResult, _due, _to_host64, _y_norm,
                          budget_iterations, resolve_blocksize)
    n = oracle.n
    b = resolve_blocksize(config, n)
    total = budget_iterations(config, b / n)
    eng = SddEngine(oracle, Y, config, total)
    try:
        ynorm = _y_norm(Y)
        trace = ConvergenceTrace()
        diverged, done = False, 0
        for t in range(total):
            blk, crc = eng.step()
            done = t + 1
            if on_iterate is not None:
                on_iterate(done, _to_host64(gather_rows(eng.estimate_local(), n, eng.shard)))
            relres = math.nan
            if _due(config.residual_every, t, total):
                if not bool(torch.isfinite(eng.W).all()):
                    relres = math.inf
                else:
                    relres = eng.relative_residual(ynorm)
            trace.record(done, done * b / n, relres, eng.eta, crc)
            if not math.isnan(relres):
                if not np.isfinite(relres) or relres > DIVERGENCE_FACTOR:
                    diverged = True
                    break
                if config.tol is not None and relres <= config.tol:
                    break
        est = _to_host64(gather_rows(eng.estimate_local(), n, eng.shard))
    finally:
        eng.close()
    return SolveResult(est[:, 0] if eng.vector else est, trace, diverged, done, done * b / n)


def _omega(seed, n, rank, device=None):
    """substream(seed, "omega").standard_normal((n, r)) (solvers.py:538), on the
    GPU at scale (rng.standard_normal)."""
    z = standard_normal(substream(seed, "omega"), (n, rank), device)
    return z.cpu().numpy() if torch.is_tensor(z) else z


def pcg_solve(oracle, Y, config, pool=None, on_iterate=None):
    """Conjugate gradient on (K + lam I) W = Y with a global rank-r Nystrom
    preconditioner, per-column recurrences (solvers.py:519-584). ``nystrom_rank``
    0 gives plain CG; stops when every column's relative residual is below
    tol (default 1e-6) or the budget (default n iterations) is spent."""
    from .solvers import ConvergenceTrace, SolveResult
    if current_shard(oracle.n).world > 1:
        raise ConfigError("pcg_solve runs on one device (the B200 build shards ADASAP and SDD)")
    n, lam, dev = oracle.n, oracle.lam, oracle.device
    Ya = np.asarray(Y, dtype=np.float64)
    vector = Ya.ndim == 1
    Y2 = Ya[:, None] if vector else Ya
    if Y2.shape[0] != n:
        raise ContractError("right-hand side must have n rows")
    rank = config.nystrom_rank if config.nystrom_rank is not None else min(100, n)
    rank = int(rank)
    if rank < 0 or rank > n:
        raise ConfigError("pcg rank outside [0, n]")
    f64 = torch.float64
    if rank > 0:
        omega = _omega(config.seed, n, rank, dev)
        sketch = oracle.matmul(omega)
        factor = rand_nystrom_retry(sketch, omega, rank)
        rho = float(factor.S[-1]) + lam
        U = torch.as_tensor(factor.U, dtype=f64, device=dev)
        Mc = torch.as_tensor(woodbury_core(factor.S, (U.T @ U).cpu().numpy(), rho),
                             dtype=f64, device=dev)

        def apply_inv(R):
            return (R - U @ (Mc @ (U.T @ R))) / rho
    else:
        def apply_inv(R):
            return R / 1.0

    tol = config.tol if config.tol is not None else 1e-6
    total = config.max_iters if config.max_iters is not None else n
    if config.max_iters is None and config.max_passes is not None:
        total = max(1, math.ceil(config.max_passes))
    tiny = np.finfo(np.float64).tiny
    Yd = torch.as_tensor(Y2, dtype=f64, device=dev)
    X = torch.zeros_like(Yd)
    R = Yd.clone()
    Zp = apply_inv(R)
    P = Zp.clone()
    rz = (R * Zp).sum(0)
    col_norms = torch.clamp(torch.linalg.vector_norm(Yd, dim=0), min=tiny)
    ynorm = max(float(torch.linalg.vector_norm(Yd)), tiny)
    ids = torch.arange(n, device=dev, dtype=torch.int64)
    trace = ConvergenceTrace()
    done = 0
    for t in range(total):
        active = torch.linalg.vector_norm(R, dim=0) / col_norms > tol
        if not bool(active.any()):
            break
        # AP = K P + lam P: the block-row kernel with every point as a row
        KP = oracle.rows_times_device(ids, P.T.to(torch.float32).contiguous())
        AP = KP.to(f64) + lam * P
        pap = (P * AP).sum(0)
        if bool((pap[active] <= 0.0).any()):
            raise NumericalError("conjugate gradient breakdown: p^T A p <= 0")
        alpha = torch.where(active, rz / torch.where(pap > 0.0, pap, torch.ones_like(pap)),
                            torch.zeros_like(pap))
        X += alpha * P
        R -= alpha * AP
        Zp = apply_inv(R)
        rz_new = (R * Zp).sum(0)
        beta = torch.where(active, rz_new / torch.where(rz > 0.0, rz, torch.ones_like(rz)),
                           torch.zeros_like(rz))
        P = Zp + beta * P
        rz = rz_new
        done = t + 1
        if on_iterate is not None:
            on_iterate(done, X.cpu().numpy())
        trace.record(done, float(done), float(torch.linalg.vector_norm(R)) / ynorm, math.nan, 0)
    Xh = X.cpu().numpy()
    return SolveResult(Xh[:, 0] if vector else Xh, trace, False, done, float(done))


class SapEngine(SddEngine):
    """Exact sketch-and-project (solvers.py:269-287): the block gradient on the
    same block product, then (K[B,B] + lam I) d = grad by one fp64 Cholesky of
    size b on the device (cuSOLVER through torch.linalg), W[B] -= d. K[B,B] is
    the fp64 tile (sap_ktile64, the reference's arithmetic)."""

    def __init__(self, oracle, Y, config, total, shard=None):
        super().__init__(oracle, Y, config, total, shard)
        if self.shard.world > 1:
            raise ConfigError("exact SAP runs on one device (its b x b solve is not sharded)")
        self.info = torch.zeros((), dtype=torch.int32, device=self.dev)
        # the iterate in fp64 (the exact projection is an fp64 solve, state.W of
        # the reference); self.W is its fp32 copy, the block product's operand
        self.W64 = torch.zeros((self.m, self.ld), dtype=torch.float64, device=self.dev)
        Ya = np.asarray(Y, dtype=np.float64)
        Yl = Ya[self.shard.lo:self.shard.hi]
        Yl = Yl[:, None] if Yl.ndim == 1 else Yl
        self.Y64 = torch.zeros((self.m, self.ld), dtype=torch.float64, device=self.dev)
        self.Y64[:, :Yl.shape[0]] = torch.as_tensor(Yl.T, device=self.dev)

    def step(self):
        blk, crc, bd = self.feed.get()
        b, m = self.b, self.m
        loc = self.shard.local_positions(bd)
        if self.use_tc:
            self.zop.fill(self.W)
            self.tcp.gather_rows(bd, out=self.RAg)
            krows_tc(self.o.spec, self.tcp, self.RAg, b, bd, self.zop, self.G, ws=self.ws)
        else:
            pts = self.o.points
            Xb, rsq = pts.gather(bd)
            krows_times(self.o.spec, pts, Xb, rsq, bd, self.W, self.G, col_base=self.shard.lo,
                        ws=self.ws, ncols=self.shard.size, col_offset=self.shard.lo)
        # grad = K[B,:] W + lam W[B] - Y[B], the last two terms from the fp64 iterate
        self.g.copy_(self.G)
        self.g += self.lam * self.W64[:, loc].T - self.Y64[:, loc].T
        H = self.o.block_device(bd)
        H.diagonal().add_(self.lam)
        L, info = torch.linalg.cholesky_ex(H)
        self.info = torch.maximum(self.info, info)  # checked at the end of the solve
        d = torch.cholesky_solve(self.g, L)
        self.W64[:, loc] -= d.T
        self.W[:, loc] = self.W64[:, loc].float()
        self.t += 1
        return blk, crc

    def iterate_local(self):
        return self.W64[:, :self.shard.size].T


def sap_solve(oracle, Y, config, sampler="uniform", dpp_model=None, pool=None, on_iterate=None):
    """Exact sketch-and-project from W0 = 0 with optional tail averaging
    (solvers.py:290-348). The k-DPP sampler (dpp.py) is outside the B200 build.
    A failed block Cholesky raises NumericalError at the end of the solve (the
    device flags are read once, not per step)."""
    from .solvers import (ConvergenceTrace, SolveResult, TailAverager, _due, _to_host64,
                          _y_norm, budget_iterations, resolve_blocksize)
    if sampler != "uniform":
        if sampler == "kdpp":
            raise ConfigError("k-DPP block sampling is outside the B200 build")
        raise ConfigError(f"unknown sampler {sampler!r}")
    n = oracle.n
    b = resolve_blocksize(config, n)
    total = budget_iterations(config, b / n)
    eng = SapEngine(oracle, Y, config, total)
    try:
        ynorm = _y_norm(Y)
        trace = ConvergenceTrace()
        averager = TailAverager(total, (n, eng.m)) if config.tail_average else None
        diverged, done = False, 0
        for t in range(total):
            blk, crc = eng.step()
            done = t + 1
            if averager is not None:
                averager.add(done, eng.iterate_local().clone())
            if on_iterate is not None:
                on_iterate(done, _to_host64(eng.iterate_local()))
            relres = math.nan
            if _due(config.residual_every, t, total):
                relres = _relres_cm(oracle, eng.shard, eng.W64, eng.Y64, eng.lam, ynorm)
            trace.record(done, done * b / n, relres, 1.0, crc)
            if np.isfinite(relres):
                if relres > DIVERGENCE_FACTOR or not bool(torch.isfinite(eng.W64).all()):
                    diverged = True
                    break
                if config.tol is not None and relres <= config.tol:
                    break
        if int(eng.info) != 0:
            raise NumericalError("block system factorization failed; lam may be too small "
                                 "for float64")
        W_loc = averager.average() if averager is not None and averager.count > 0 else \
            eng.iterate_local()
        W = _to_host64(W_loc)
    finally:
        eng.close()
    return SolveResult(W[:, 0] if eng.vector else W, trace, diverged, done, done * b / n)
