"""ADASAP on B200: drop-in mirror of ``sapgp.solvers`` (solvers.py:1-615).

Same public names and semantics (``AccelParams``, ``resolve_accel``,
``nesterov_update``, ``ConvergenceTrace``, ``SolverState``, ``SolveResult``,
``adasap_step``, ``adasap_solve``, ``solve``), with the iteration executed
by ``AdasapEngine``:

* Phase I  -- K[B,:] Z over this rank's shard on the tensor-core kernel
  (``sap_krows_tc``; ``sap_krows_times`` for shapes outside it), then the
  gradient gather g = K[B,:]Z + lam Z[B] - Y[B] (``sap_grad_gather``) and,
  with several GPUs, one float64 all-reduce of g (paper Alg. 6);
* Phases II/III -- produced ahead, batched, by ``pipeline.Lookahead``;
* Phase IV -- D_B = (g - U Mc U^T g) / rho with the r x r Cholesky-stabilised
  Woodbury core Mc (randnla.py:109-134; three small fp64 GEMMs) and the
  Nesterov update.

The Nesterov update never touches the n - b rows outside the block. Off
the block the recurrence (solvers.py:76-85) is the fixed linear map
T = [[beta, 1-beta], [alpha, 1-alpha]] on the row pair (V, Z), so the
engine stores two arrays (P, Q) and a 2 x 2 basis M with
[V; Z] = M [P; Q] row-wise: untouched rows follow M <- T M for free, and
the b block rows get an axpy (``sap_pq_update``). M is T's eigenbasis with
the decaying column scaled by a scalar recurrence s_t = (beta - alpha)^t,
renormalised by a rare dense rescale of Q. W is
materialised only when asked for (end of solve, residuals, tail averaging,
callbacks). DESIGN.md §4 has the derivation.

Deviations (documented, none changes the iterates beyond fp32 rounding):
arithmetic on the state and the block product is fp32 (reference fp64);
the per-iteration trace ``seconds`` is host enqueue time unless a residual
is due; errors inside the lookahead surface at the start of the batch that
contains the failing iteration.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from . import xfer
from .errors import ConfigError, ContractError
from .kernels import KernelOracle, ZOperand, krows_tc, krows_tc_partials, krows_times, to_colmajor
from .parallel import allreduce_sum_, current_shard, gather_rows
from .pipeline import Lookahead
from .rng import block_hash

DIVERGENCE_FACTOR = 1e6
SDD_MOMENTUM = 0.9
RENORM_LO, RENORM_HI = 2.0 ** -20, 2.0 ** 20


# ---------------------------------------------------------------------------
# acceleration parameters and the Nesterov recurrence (solvers.py:32-85)


@dataclass(frozen=True)
class AccelParams:
    mu: float
    nu: float

    def __post_init__(self):
        if not (self.mu > 0.0 and self.nu > 0.0):
            raise ContractError("acceleration parameters must be positive")

    @property
    def beta(self):
        return 1.0 - math.sqrt(self.mu / self.nu)

    @property
    def gamma(self):
        return 1.0 / math.sqrt(self.mu * self.nu)

    @property
    def alpha(self):
        return 1.0 / (1.0 + self.gamma * self.nu)


@dataclass(frozen=True)
class RawAccel:
    beta: float
    gamma: float
    alpha: float


NO_ACCELERATION = RawAccel(beta=1.0, gamma=0.0, alpha=0.0)


def resolve_accel(config, n, blocksize):
    """mu = lam, nu = n / blocksize by default (solvers.py:69-73)."""
    mu = config.lam if config.mu == "default" else float(config.mu)
    nu = n / blocksize if config.nu == "default" else float(config.nu)
    return AccelParams(mu, nu)


def nesterov_update(W, V, Z, direction, eta, beta, gamma, alpha):
    """W' = Z - eta D; V' = beta V + (1-beta) Z - gamma eta D; Z' = alpha V + (1-alpha) W'
    (solvers.py:76-85). Elementwise; runs on whatever device the inputs live on."""
    W_next = Z - eta * direction
    V_next = beta * V + (1.0 - beta) * Z - (gamma * eta) * direction
    Z_next = alpha * V + (1.0 - alpha) * W_next
    return W_next, V_next, Z_next


# ---------------------------------------------------------------------------
# traces, averaging, results (solvers.py:92-211)


@dataclass
class TraceRecord:
    iteration: int
    seconds: float
    passes: float
    residual: float
    stepsize: float
    block_hash: int
    subspace_err: float | None = None


class ConvergenceTrace:
    COLUMNS = ("iter", "seconds", "passes", "residual", "stepsize", "subspace_err_l")

    def __init__(self):
        self.records = []
        self._start = time.perf_counter()

    def record(self, iteration, passes, residual, stepsize, block_hash, subspace_err=None):
        self.records.append(TraceRecord(iteration, time.perf_counter() - self._start, passes,
                                        residual, stepsize, block_hash, subspace_err))

    def residuals(self):
        return np.array([r.residual for r in self.records])

    def passes(self):
        return np.array([r.passes for r in self.records])

    def final_residual(self):
        for rec in reversed(self.records):
            if np.isfinite(rec.residual):
                return rec.residual
        return math.nan

    def passes_to(self, tol):
        for rec in self.records:
            if np.isfinite(rec.residual) and rec.residual <= tol:
                return rec.passes
        return math.inf

    def to_csv(self, path):
        with open(path, "w") as fh:
            fh.write(",".join(self.COLUMNS) + "\n")
            for r in self.records:
                sub = "" if r.subspace_err is None else repr(r.subspace_err)
                fh.write(f"{r.iteration},{r.seconds!r},{r.passes!r},{r.residual!r},"
                         f"{r.stepsize!r},{sub}\n")


class TailAverager:
    """Streaming mean of iterates with indices in [ceil(T/2), T-1] (solvers.py:155-174)."""

    def __init__(self, total_iters, shape):
        if total_iters < 2:
            raise ContractError("tail averaging needs at least two iterations")
        self.start = math.ceil(total_iters / 2)
        self.stop = total_iters - 1
        self._sum = None
        self.shape = shape
        self.count = 0

    def add(self, index, iterate):
        """Accumulate in float64, in place (numpy iterates as in the reference,
        or device tensors: one preallocated fp64 accumulator, no per-add copy)."""
        if not self.start <= index <= self.stop:
            return
        if torch.is_tensor(iterate):
            if self._sum is None:
                self._sum = torch.zeros(iterate.shape, dtype=torch.float64, device=iterate.device)
            self._sum.add_(iterate.to(torch.float64))
        else:
            it = np.asarray(iterate, dtype=np.float64)
            if self._sum is None:
                self._sum = np.zeros(it.shape)
            self._sum += it
        self.count += 1

    def average(self):
        if self.count == 0:
            raise ContractError("empty tail-average window")
        return self._sum / self.count


def tail_average(iterates):
    items = list(iterates)
    if not items:
        raise ContractError("empty tail-average window")
    total = np.zeros_like(np.asarray(items[0], dtype=np.float64))
    for it in items:
        total += it
    return total / len(items)


@dataclass
class SolveResult:
    W: np.ndarray
    trace: ConvergenceTrace
    diverged: bool
    iterations: int
    passes: float


def resolve_blocksize(config, n):
    b = config.blocksize if config.blocksize is not None else max(1, n // 100)
    b = int(b)
    if not 1 <= b <= n:
        raise ConfigError(f"blocksize {b} outside [1, {n}]")
    return b


def resolve_rank(config, blocksize):
    r = config.nystrom_rank if config.nystrom_rank is not None else min(100, blocksize)
    r = int(r)
    if not 1 <= r <= blocksize:
        raise ConfigError(f"nystrom_rank {r} outside [1, {blocksize}]")
    return r


def budget_iterations(config, passes_per_iter):
    if config.max_iters is not None:
        return int(config.max_iters)
    passes = config.max_passes if config.max_passes is not None else 50.0
    return max(1, math.ceil(passes / passes_per_iter))


def _due(every, t, total):
    if every <= 0:
        return t == total - 1
    return (t + 1) % every == 0 or t == total - 1


# ---------------------------------------------------------------------------
# the engine


def _basis(beta, alpha):
    """Eigen-directions of T = [[beta, 1-beta], [alpha, 1-alpha]] for the lazy state.

    T has eigenvalue 1 on u1 = (1, 1)/sqrt(2) and lam2 = beta - alpha on
    u2 = (1-beta, -alpha)/|.|. The basis at iteration t is M_t = [u1, s_t u2]
    with the scalar recurrence s_{t+1} = lam2 s_t, so the directions never
    accumulate rounding (propagating M <- T M would let u2 drift into u1).
    Returns (u1, u2, lam2, dense); ``dense`` marks defective / degenerate T."""
    T = np.array([[beta, 1.0 - beta], [alpha, 1.0 - alpha]])
    if np.array_equal(T, np.eye(2)):
        return np.array([1.0, 0.0]), np.array([0.0, 1.0]), 1.0, False
    lam2 = beta - alpha
    e2 = np.array([1.0 - beta, -alpha])
    if abs(1.0 - beta + alpha) < 1e-12 or abs(lam2) < 1e-6:
        return np.array([1.0, 0.0]), np.array([0.0, 1.0]), 1.0, True
    return np.ones(2) / math.sqrt(2.0), e2 / np.linalg.norm(e2), lam2, False


class SolverState:
    """Iterate triple of ADASAP (solvers.py:189-202): ``W``, ``V``, ``Z`` (n x m)
    and ``iteration``; V and Z alias W when acceleration is off (``zeros``).

    Drop-in semantics: a state made by ``SolverState.zeros`` (or from any
    arrays) is stepped by ``adasap_step`` like the reference's. The first step
    binds a device engine to the state (the lazy two-array form of DESIGN.md
    §4, resumed from the state's arrays at ``iteration``); later steps reuse
    it while the oracle, Y, config, accel and identity_precond are the same.
    ``W``/``V``/``Z`` are written back lazily: reading one materialises the
    current iterate as a fresh float64 host array (the reference rebinds them
    to new arrays each step too, solvers.py:399-401). Assigning one, or
    ``iteration``, detaches the engine; the next step resumes from the
    assigned values."""

    def __init__(self, W=None, V=None, Z=None, iteration=0):
        self._zero = False  # known all-zero arrays (zeros()): no scan when binding
        if isinstance(W, AdasapEngine):  # bound to an engine (make_state)
            self._e, self._W, self._V, self._Z, self._it = W, None, None, None, W.t
            return
        self._e = None
        self._W, self._V, self._Z, self._it = W, V, Z, int(iteration)

    @classmethod
    def zeros(cls, n, m, accelerated=False):
        W = np.zeros((n, m))
        # three distinct zero arrays (np.zeros maps zero pages lazily; a copy
        # of W would touch all n*m*8 bytes twice)
        st = cls(W, np.zeros((n, m)), np.zeros((n, m))) if accelerated else cls(W, W, W)
        st._zero = True
        return st

    # -- engine binding ---------------------------------------------------------
    def _host(self, which):
        """The host array of W, V or Z, materialised from the bound engine's
        current iterate on first access after a step (one array at a time)."""
        cur = getattr(self, "_" + which)
        e = self._e
        if cur is None and e is not None:
            cur = _to_host64(e.gather_full(e.materialize(which)), out=e.take_readback())
            if e.vector:
                cur = cur[:, 0]
            setattr(self, "_" + which, cur)
        return cur

    def _sync(self):
        """All three host arrays <- the bound engine's current iterate."""
        for which in ("W", "V", "Z"):
            self._host(which)

    def _detach(self):
        self._sync()
        if self._e is not None:
            self._it = self._e.t
            self._e.release()
            self._e = None

    @property
    def iteration(self):
        return self._e.t if self._e is not None else self._it

    @iteration.setter
    def iteration(self, t):
        self._detach()
        self._it = int(t)

    @property
    def W(self):
        return self._host("W")

    @W.setter
    def W(self, v):
        self._detach()
        self._zero = False
        self._W = v

    @property
    def V(self):
        return self._host("V")

    @V.setter
    def V(self, v):
        self._detach()
        self._zero = False
        self._V = v

    @property
    def Z(self):
        return self._host("Z")

    @Z.setter
    def Z(self, v):
        self._detach()
        self._zero = False
        self._Z = v


def _as2d(A):
    if torch.is_tensor(A):
        return A if A.ndim == 2 else A[:, None]
    A = np.asarray(A, dtype=np.float64)
    return A if A.ndim == 2 else A[:, None]


_STAGE = {"buf": None}
_STAGE_CHUNK = int(os.environ.get("SAP_READBACK_CHUNK", str(1 << 23)))  # elements per chunk
_WIDEN_TASKS = int(os.environ.get("SAP_READBACK_TASKS", "0")) or xfer._TASKS


def _staging(elems):
    """Process-wide pinned fp32 staging buffer (two chunks), kept across calls
    (pinning 128 MB once costs more than a whole readback)."""
    buf = _STAGE["buf"]
    if buf is None or buf.numel() < 2 * elems:
        buf = torch.empty(2 * elems, dtype=torch.float32, pin_memory=True)
        _STAGE["buf"] = buf
    return buf


def _to_host64(t, out=None):
    """Device tensor -> fresh C-contiguous float64 numpy array (``out``: a
    pre-faulted array of the same shape to fill instead, xfer.prefaulted).

    fp32 state is copied as fp32 (half the bytes of a widened copy) through a
    pinned double buffer: the device->host copy of chunk k overlaps the host
    threads widening chunk k-1 into the output (numpy's casting copy releases
    the GIL), which also spreads the output's first-touch page faults."""
    src = t.contiguous()
    if out is None or out.shape != tuple(src.shape) or not out.flags.c_contiguous:
        out = np.empty(tuple(src.shape), dtype=np.float64)
    flat_out = out.reshape(-1)
    if src.dtype != torch.float32 or src.device.type != "cuda" or src.numel() < (1 << 20):
        torch.from_numpy(out).copy_(src.to(torch.float64))
        xfer.add("d2h", src.numel() * src.element_size())
        return out
    flat = src.reshape(-1)
    total = flat.numel()
    chunk = min(_STAGE_CHUNK, total)
    stage = _staging(chunk)
    stream = torch.cuda.current_stream(src.device)
    pend = [None, None]  # per staging half: futures of the widening of its last chunk

    def widen(c0, lo, hi, half, ev):  # output [lo, hi) of the chunk starting at c0
        ev.synchronize()
        base = half * chunk - c0
        np.copyto(flat_out[lo:hi], stage[base + lo: base + hi].numpy(), casting="same_kind")

    for k, lo in enumerate(range(0, total, chunk)):
        hi = min(total, lo + chunk)
        half = k & 1
        if pend[half] is not None:  # the half is free once its previous chunk is widened
            for f in pend[half]:
                f.result()
        stage[half * chunk: half * chunk + (hi - lo)].copy_(flat[lo:hi], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        step = (hi - lo + _WIDEN_TASKS - 1) // _WIDEN_TASKS
        # widening tasks per chunk, on disjoint slices of the output
        pend[half] = [xfer.host_pool().submit(widen, lo, s0, min(hi, s0 + step), half, ev)
                      for s0 in range(lo, hi, step)]
    for fs in pend:
        if fs is not None:
            for f in fs:
                f.result()
    xfer.add("d2h", total * 4)
    return out


class AdasapEngine:
    """Device-resident ADASAP iteration (solvers.py:361-456)."""

    def __init__(self, oracle, Y, config, accel, identity_precond=False, total=None, shard=None,
                 start=0, unbounded=False, state=None):
        """``total``: iteration budget (default from the config); ``unbounded``
        for the per-step API (adasap_step), which has no budget; ``start`` and
        ``state`` = (W, V, Z) (n x m, host or device) resume from an iterate
        triple at iteration ``start`` instead of zeros."""
        if not isinstance(oracle, KernelOracle):
            raise ContractError("the B200 solver needs a device KernelOracle")
        self.o = oracle
        self.cfg = config
        self.dev = oracle.device
        n = oracle.n
        self.n = n
        self.shard = shard if shard is not None else current_shard(n)
        Ya = Y if torch.is_tensor(Y) else np.asarray(Y, dtype=np.float64)
        self.vector = Ya.ndim == 1
        sh0 = self.shard
        # a CUDA tensor with exactly this shard's rows is taken as the local
        # part of a device-resident right-hand side (no full-n copy per rank)
        local_y = torch.is_tensor(Ya) and Ya.is_cuda and sh0.world > 1 and \
            Ya.shape[0] == sh0.size and sh0.size != n
        self.local_y = local_y
        if Ya.shape[0] != n and not local_y:
            raise ContractError("right-hand side must have n rows")
        Yl = Ya if local_y else Ya[self.shard.lo:self.shard.hi]
        if Yl.ndim == 1:
            Yl = Yl[:, None]
        self.m = int(Ya.shape[1]) if Ya.ndim == 2 else 1
        self.b = resolve_blocksize(config, n)
        self.r = 0 if identity_precond else resolve_rank(config, self.b)
        self.lam = oracle.lam
        self.start = int(start)
        self.total = None if unbounded else (total if total is not None else
                                             budget_iterations(config, self.b / n))
        self.accel_key = (accel.beta, accel.gamma, accel.alpha)
        self.identity_precond = identity_precond
        beta, gamma, alpha = accel.beta, accel.gamma, accel.alpha
        self.beta, self.gamma, self.alpha = beta, gamma, alpha
        self.u1, self.u2, self.lam2, self.dense = _basis(beta, alpha)
        self._u1x, self._u1y = float(self.u1[0]), float(self.u1[1])
        self._u2x, self._u2y = float(self.u2[0]), float(self.u2[1])
        self.s = self.s_prev = 1.0
        nl = self.shard.size
        self.ld = max(4, (nl + 3) // 4 * 4)
        f32 = torch.float32
        b, m = self.b, self.m
        xfer.mark("bind: start")
        self.use_tc = oracle.use_tc(m) and b >= 16 and nl > 0 and not self.dense
        self.tcp = oracle.tc_points(self.shard.lo, self.shard.hi) if self.use_tc else None
        # the lookahead first: its first plans (which need neither Y nor the
        # state) are produced while the rest of the engine is set up -- the
        # right-hand sides' upload alone takes ~20 ms at config 3
        self.t = self.start
        xfer.mark("bind: tc points")
        self.la = Lookahead(oracle, self.shard, config.seed, b, self.r, self.lam, self.total,
                            config.lookahead, identity_precond, tcp=self.tcp, start=self.start)
        xfer.mark("bind: lookahead")
        self.P = torch.zeros((self.m, self.ld), dtype=f32, device=self.dev)
        self.Q = torch.zeros((self.m, self.ld), dtype=f32, device=self.dev)
        self.Y = to_colmajor(Yl, nl, self.dev, self.ld) if nl > 0 else \
            torch.zeros((self.m, self.ld), dtype=f32, device=self.dev)
        xfer.mark("bind: Y upload")
        self.G = torch.empty((b, m), dtype=f32, device=self.dev)
        self.g = torch.empty((b, m), dtype=torch.float64, device=self.dev)
        self.WB = torch.zeros((b, m), dtype=f32, device=self.dev)
        self.last_loc = None
        self.etas = torch.zeros(max(self.total or 64, 1), dtype=torch.float64, device=self.dev)
        if self.use_tc:
            self.zop = ZOperand(m, nl, self.dev)
            self.Pb = torch.zeros(self.zop.nz, dtype=f32, device=self.dev)
            self.Qb = torch.zeros(self.zop.nz, dtype=f32, device=self.dev)
            need = nat.load().sap_krows_tc_workspace(b, m, nl)
        else:
            self.zop = self.Pb = self.Qb = None
            need = nat.load().sap_krows_workspace(b, m, max(nl, 1))
        self.ws = torch.empty(max(need // 4 + 1, 1), dtype=f32, device=self.dev)
        # Phase IV in one launch (sap_block_step, csrc/phase4.cu): gradient
        # gather + Woodbury apply + lazy update + the next operand's block rows;
        # SAP_FUSED_STEP=0 selects the unfused chain (grad_gather, two GEMMs,
        # pq_update, separate operand pass) for A/B runs
        lib = nat.load()
        self.fused = (os.environ.get("SAP_FUSED_STEP", "1") == "1" and not self.dense
                      and bool(lib.sap_block_step_supported(b, self.r, m)))
        self.p4ws = torch.zeros(lib.sap_block_step_workspace(b, self.r, m) // 8 + 1,
                                dtype=torch.float64, device=self.dev)
        self.zflag = torch.zeros(2, dtype=torch.int32, device=self.dev)
        self._fi = 0
        # the next iterate's operand buffer, filled inside the block-row kernel
        # (double buffering; skipped when the state would not fit beside it)
        self.zop_next = None
        if self.fused and self.use_tc:
            # room left for this process's allocations (the allocator's own
            # counters: cudaMemGetInfo, a driver call, cost up to ~40 ms per
            # bind next to the lookahead's producers)
            free = torch.cuda.get_device_properties(self.dev).total_memory - \
                torch.cuda.memory_allocated(self.dev)
            if free > 2 * self.zop.hi.numel() * 2 + (4 << 30):
                self.zop_next = ZOperand(m, nl, self.dev)
        xfer.mark("bind: buffers")
        self.z_stale = True  # zop does not hold Z_t yet (filled by the first step)
        self.W0 = None  # W at `start` when resuming from a nonzero state (until the first step)
        if state is not None:
            self._load_state(*state)
        self.crcs = []

    def _load_state(self, W, V, Z):
        """[V; Z] = M [P; Q] row-wise from a given iterate triple."""
        sh, nl = self.shard, self.shard.size
        if nl == 0:
            return
        cm = lambda A: to_colmajor(A[sh.lo:sh.hi] if A.ndim == 2 else A[sh.lo:sh.hi, None], nl,
                                   self.dev, self.ld)
        Vd, Zd = cm(_as2d(V)), cm(_as2d(Z))
        (a, b), (c, d) = self.M
        det = a * d - b * c
        # [P; Q] = M^-1 [V; Z], fp32 on the device
        self.P.copy_(Vd * (d / det) - Zd * (b / det))
        self.Q.copy_(Zd * (a / det) - Vd * (c / det))
        self.W0 = cm(_as2d(W))[:, :nl].T.contiguous()
        if self.Pb is not None:
            for A, bnd in ((self.P, self.Pb), (self.Q, self.Qb)):
                nat.call("sap_colabsmax", nat.ptr(A), A.stride(0), nl, self.m, nat.ptr(bnd),
                         nat.stream_handle())
        if self.dense:
            self.Wdense = self.W0.clone()

    def close(self):
        self.la.close()

    def prepare_readback(self):
        """Have host threads fault in the float64 array of the next full-iterate
        readback (n x m) while the device works (xfer.prefaulted); the first
        W/V/Z readback takes it."""
        self._readback = xfer.prefaulted((self.n, self.m)) if self.n * self.m >= (1 << 20) else None

    def take_readback(self):
        rb, self._readback = getattr(self, "_readback", None), None
        if rb is None:
            return None
        out, futs = rb
        for f in futs:
            f.result()
        return out

    def release(self):
        """close() and drop the device buffers (state, operands, workspaces)
        so the caching allocator can hand them to the next engine at once."""
        self._readback = None
        self.close()
        for name in ("P", "Q", "Y", "G", "g", "WB", "etas", "zop", "zop_next", "ws", "p4ws",
                     "Pb", "Qb", "W0", "tcp"):
            if hasattr(self, name):
                setattr(self, name, None)

    # -- one iteration ------------------------------------------------------------
    def step(self, point=None):
        """One ADASAP iteration; returns the host IterPlan (block, crc, rho)."""
        if point is None and self.fused:
            return self._step_fused()
        self.z_stale = True
        plan = self.la.get(self.t)
        sh = self.shard
        zp, zq = self._u1y, self.s * self._u2y
        if point is None:
            R, R2, ca, cb = self.P, self.Q, zp, zq
        else:
            R, R2, ca, cb = point, None, 1.0, 0.0
        # Phase I: K[B, shard] Z[shard]
        if sh.size > 0 and self.use_tc:
            if point is None:
                self.zop.fill(self.P, self.Q, zp, zq, self.Pb, self.Qb)
            else:
                self.zop.fill(point)
            krows_tc(self.o.spec, self.tcp, plan.RAg, self.b, plan.block_dev, self.zop, self.G,
                     ws=self.ws)
        elif sh.size > 0:
            krows_times(self.o.spec, self.o.points, plan.Xb, plan.rsq, plan.block_dev, R,
                        self.G, col_base=sh.lo, R2=R2, ca=ca, cb=cb, ws=self.ws, ncols=sh.size,
                        col_offset=sh.lo)
        else:
            self.G.zero_()
        gz = (zp, zq) if point is None else (1.0, 0.0)
        gpoint = (self.P, self.Q) if point is None else (point, None)
        nat.call("sap_grad_gather", nat.ptr(self.G), self.G.stride(0), nat.ptr(gpoint[0]),
                 nat.ptr(gpoint[1]), nat.ptr(self.Y), self.ld, gz[0], gz[1],
                 nat.ptr(plan.loc_dev), self.b, self.m, self.lam, nat.ptr(self.g),
                 self.g.stride(0), nat.stream_handle())
        allreduce_sum_(self.g)
        # Phase IV: D_B = (g - U Mc U^T g) / rho; the 1/rho rides on the
        # update's stepsize (every use of D in sap_pq_update is eta * D)
        if plan.U is not None:
            D = torch.addmm(self.g, plan.UMc, plan.U.T @ self.g, alpha=-1.0)
        else:
            D = self.g
        self._update(plan, D)
        if self.t == plan.batch_t0:  # the batch's stepsizes into the trace, once per batch
            self._record_etas(plan)
        self.last_loc = plan.loc_dev
        self.crcs.append(plan.crc)
        self.t += 1
        return plan

    def _step_fused(self):
        """Phase I on the block-row kernel (partials left unreduced; the next
        iterate's operand streamed by the same kernel), then Phases I(tail)-IV
        in one cooperative launch (sap_block_step): gradient gather, all-reduce
        (several ranks: between a GRAD and an APPLY launch), Woodbury apply
        D = g - U Mc U^T g (randnla.py:109-134), lazy Nesterov update of the
        block rows (solvers.py:76-85) and Z_{t+1} at those rows."""
        plan = self.la.get(self.t)
        sh, lib = self.shard, nat.load()
        zp, zq = self._u1y, self.s * self._u2y
        e0, e1, s_next = self._coeffs()
        zq1 = s_next * self._u2y
        a = nat.StepArgs()
        zn = self.zop_next
        if sh.size > 0 and self.use_tc:
            if self.z_stale:
                self.zop.fill(self.P, self.Q, zp, zq, self.Pb, self.Qb)
            nxt = (self.P, self.Q, zp, zq1, self.Pb, self.Qb, zn) if zn is not None else None
            a.splits = krows_tc_partials(self.o.spec, self.tcp, plan.RAg, self.b, plan.block_dev,
                                         self.zop, self.ws, nxt)
            a.part, a.variance, a.zscale = nat.ptr(self.ws), self.o.spec.variance, \
                nat.ptr(self.zop.scale)
        else:
            if sh.size > 0:
                krows_times(self.o.spec, self.o.points, plan.Xb, plan.rsq, plan.block_dev,
                            self.P, self.G, col_base=sh.lo, R2=self.Q, ca=zp, cb=zq, ws=self.ws,
                            ncols=sh.size, col_offset=sh.lo)
            else:
                self.G.zero_()
            a.G, a.ldg = nat.ptr(self.G), self.G.stride(0)
        a.P, a.Q, a.Y, a.ldp = nat.ptr(self.P), nat.ptr(self.Q), nat.ptr(self.Y), self.ld
        a.zp, a.zq, a.lam = zp, zq, self.lam
        a.loc, a.b, a.m = nat.ptr(plan.loc_dev), self.b, self.m
        a.g, a.ldgo = nat.ptr(self.g), self.g.stride(0)
        if plan.U is not None:
            a.U, a.UMc, a.ldu, a.r = nat.ptr(plan.U), nat.ptr(plan.UMc), plan.U.stride(0), self.r
        a.Pw, a.Qw, a.eta_dev, a.e0, a.e1 = nat.ptr(self.P), nat.ptr(self.Q), \
            nat.ptr(plan.eta_rho_dev), e0, e1
        a.WB, a.ldwb, a.Pb, a.Qb = nat.ptr(self.WB), self.WB.stride(0), nat.ptr(self.Pb), \
            nat.ptr(self.Qb)
        if zn is not None and sh.size > 0:
            a.Zhi_next, a.Zlo_next, a.ldz, a.zscale_next = nat.ptr(zn.hi), nat.ptr(zn.lo), \
                zn.ldz, nat.ptr(zn.scale)
            a.zp1, a.zq1, a.zflag, a.flag_idx = zp, zq1, nat.ptr(self.zflag), self._fi
            a.n_local = sh.size
            self._fi ^= 1
        ws, wsb, st = nat.ptr(self.p4ws), self.p4ws.numel() * 8, nat.stream_handle()
        if sh.world == 1:
            nat.check(lib.sap_block_step(ctypes.byref(a), nat.STEP_GRAD | nat.STEP_APPLY, ws, wsb,
                                         st))
        else:
            nat.check(lib.sap_block_step(ctypes.byref(a), nat.STEP_GRAD, ws, wsb, st))
            allreduce_sum_(self.g)
            nat.check(lib.sap_block_step(ctypes.byref(a), nat.STEP_APPLY, ws, wsb, st))
        if zn is not None and sh.size > 0:
            self.zop, self.zop_next = zn, self.zop
            self.z_stale = False
        else:
            self.z_stale = True
        self._advance(s_next)
        if self.t == plan.batch_t0:  # the batch's stepsizes into the trace, once per batch
            self._record_etas(plan)
        self.last_loc = plan.loc_dev
        self.crcs.append(plan.crc)
        self.t += 1
        return plan

    def eval_point(self, config):
        """The block-row product's point (solvers.py:376): None for Z (the
        engine's own operand), else W as a column-major (m x ld) array."""
        if config.grad_eval_point != "w" or (self.t == self.start and self.W0 is None):
            return None  # W = Z = 0 before the first step of a fresh solve
        W = self.materialize("W").T
        pt = torch.zeros((self.m, self.ld), dtype=torch.float32, device=self.dev)
        pt[:, :W.shape[1]] = W
        return pt

    def _record_etas(self, plan):
        k0, k1 = self.t - self.start, self.t - self.start + plan.batch_eta.numel()
        if k1 > self.etas.numel():
            grown = torch.zeros(max(k1, 2 * self.etas.numel()), dtype=torch.float64,
                                device=self.dev)
            grown[:self.etas.numel()].copy_(self.etas)
            self.etas = grown
        self.etas[k0:k1].copy_(plan.batch_eta)

    def _coeffs(self):
        """(e0, e1, s_next): the block rows' update of [P; Q] in the next basis,
        e = M_{t+1}^{-1} (-gamma, -(1 - alpha)) (2 x 2 closed form)."""
        delta = (-self.gamma, -(1.0 - self.alpha))
        s_next = self.lam2 * self.s
        a, c = self._u1x, self._u1y
        bb, dd = s_next * self._u2x, s_next * self._u2y
        det = a * dd - bb * c
        return (delta[0] * dd - bb * delta[1]) / det, (a * delta[1] - c * delta[0]) / det, s_next

    def _advance(self, s_next):
        self.s_prev, self.s = self.s, s_next
        if abs(s_next) < RENORM_LO or abs(s_next) > RENORM_HI:
            self.Q.mul_(s_next)
            if self.Qb is not None:
                self.Qb.mul_(abs(s_next))
            self.s_prev /= s_next
            self.s = 1.0

    @property
    def M(self):
        return np.column_stack([self.u1, self.s * self.u2])

    @property
    def M_prev(self):
        return np.column_stack([self.u1, self.s_prev * self.u2])

    def _update(self, plan, D):
        beta, gamma, alpha = self.beta, self.gamma, self.alpha
        delta = (-gamma, -(1.0 - alpha))
        M = ((self._u1x, self.s * self._u2x), (self._u1y, self.s * self._u2y))
        if self.dense:
            # degenerate T (repeated/zero second eigenvalue): apply T to every row
            self._pq(plan, D, M, 0.0, 0.0)
            self.Wdense = self.Q[:, :self.shard.size].T.clone()  # Z_t: W_{t+1} off the block
            P = self.P.clone()
            self.P.mul_(beta).add_(self.Q, alpha=1.0 - beta)
            self.Q.mul_(1.0 - alpha).add_(P, alpha=alpha)
            self._pq(plan, D, M, delta[0], delta[1], wb=False)
            return
        e0, e1, s_next = self._coeffs()
        self._pq(plan, D, M, e0, e1)
        self._advance(s_next)

    def _pq(self, plan, D, M, e0, e1, wb=True):
        nat.call("sap_pq_update", nat.ptr(self.P), nat.ptr(self.Q), self.ld,
                 nat.ptr(plan.loc_dev), self.b, self.m, nat.ptr(D), D.stride(0),
                 nat.ptr(plan.eta_rho_dev), M[1][0], M[1][1], e0, e1,
                 nat.ptr(self.WB) if wb else None, self.WB.stride(0), nat.ptr(self.Pb),
                 nat.ptr(self.Qb), nat.stream_handle())

    # -- materialisation ------------------------------------------------------------
    def materialize(self, which="W", col=None):
        """Local shard of W, V or Z as an (n_local x m) fp32 tensor; ``col``:
        only that right-hand side's column, (n_local x 1) (no n x m buffer)."""
        if col is not None:
            return self._materialize_col(which, int(col))
        nl = self.shard.size
        out = torch.empty((self.m, self.ld), dtype=torch.float32, device=self.dev)
        if which == "W":
            if self.t == self.start:
                if self.W0 is not None:
                    return self.W0.clone()
                return torch.zeros((nl, self.m), dtype=torch.float32, device=self.dev)
            a, c = self.M_prev[1, 0], self.M_prev[1, 1]
        elif which == "Z":
            a, c = self.M[1, 0], self.M[1, 1]
        else:
            a, c = self.M[0, 0], self.M[0, 1]
        if which == "W" and self.dense:
            W = self.Wdense
        else:
            if nl > 0:
                nat.call("sap_combine", nat.ptr(out), self.ld, nat.ptr(self.P), nat.ptr(self.Q),
                         self.ld, nl, self.m, a, c, nat.stream_handle())
            W = out[:, :nl].T
        if which == "W":
            loc = self.last_loc
            own = loc >= 0
            W = W.clone()
            W[loc[own]] = self.WB[own]
        return W

    def _materialize_col(self, which, c):
        nl = self.shard.size
        if which == "W" and self.t == self.start:
            return self.W0[:, c:c + 1].clone() if self.W0 is not None else \
                torch.zeros((nl, 1), dtype=torch.float32, device=self.dev)
        if which == "W" and self.dense:
            return self.Wdense[:, c:c + 1].clone()
        M = self.M_prev if which == "W" else self.M
        a, cc = (M[1, 0], M[1, 1]) if which in ("W", "Z") else (M[0, 0], M[0, 1])
        out = torch.empty((1, self.ld), dtype=torch.float32, device=self.dev)
        if nl > 0:
            nat.call("sap_combine", nat.ptr(out), self.ld, nat.ptr(self.P[c]), nat.ptr(self.Q[c]),
                     self.ld, nl, 1, a, cc, nat.stream_handle())
        W = out[:, :nl].T.clone()
        if which == "W":
            loc = self.last_loc
            own = loc >= 0
            W[loc[own], 0] = self.WB[own, c]
        return W

    def gather_full(self, local):
        """Concatenate shards (n x m) on every rank."""
        return gather_rows(local, self.n, self.shard)

    def y_norm(self):
        """||Y||_F over all ranks from the device-resident right-hand sides."""
        part = (self.Y[:, :self.shard.size].double() ** 2).sum().reshape(1)
        allreduce_sum_(part)
        return max(float(torch.sqrt(part)), np.finfo(np.float64).tiny)

    def relative_residual(self, W_local, ynorm):
        """||K W + lam W - Y||_F / ||Y||_F (solvers.py:254-257), shard-local:
        rank r forms (K W)[shard r] = sum_q K[shard r, shard q] W_q, the shards
        W_q arriving one at a time by broadcast (so no rank holds more than
        two n/P x m shards; no n x m all-gather), then one scalar all-reduce."""
        import torch.distributed as tdist
        from .kernels import range_product
        from .dist import partition
        sh = self.shard
        m = self.m
        Wcm = torch.zeros((m, self.ld), dtype=torch.float32, device=self.dev)
        if sh.size:
            Wcm[:, :sh.size] = W_local.T
        if sh.size == 0:
            part = torch.zeros(1, dtype=torch.float64, device=self.dev)
            KW = None
        else:
            ids = torch.arange(sh.lo, sh.hi, device=self.dev, dtype=torch.int64)
            if self.use_tc:
                rows = ("tc", self.tcp.gather_rows(ids))
            else:
                rows = ("pts",) + self.o.points.gather(ids)
            KW = torch.empty((sh.size, m), dtype=torch.float32, device=self.dev)
        ranges = [(0, self.n)] if sh.world == 1 else (
            partition(self.n, sh.world) if self.n >= sh.world else
            [(0, self.n) if q == 0 else (self.n, self.n) for q in range(sh.world)])
        for q, (lo, hi) in enumerate(ranges):
            if sh.world > 1:
                ldq = max(4, (hi - lo + 3) // 4 * 4)
                buf = Wcm if q == sh.rank else torch.empty((m, ldq), dtype=torch.float32,
                                                           device=self.dev)
                tdist.broadcast(buf, src=q)
            else:
                buf = Wcm
            if KW is not None:
                range_product(self.o, rows, ids, buf, lo, hi, KW, accumulate=q > 0,
                              tcp=self.tcp if q == sh.rank else None)
        if KW is not None:
            res = KW.double() + self.lam * W_local.double() - self.Y[:, :sh.size].T.double()
            part = (res * res).sum().reshape(1)
        allreduce_sum_(part)
        return float(torch.sqrt(part)) / ynorm


def _y_norm(Y):
    Ya = Y if torch.is_tensor(Y) else np.asarray(Y, dtype=np.float64)
    nrm = float(torch.linalg.vector_norm(Ya.double())) if torch.is_tensor(Ya) \
        else float(np.linalg.norm(Ya))
    return max(nrm, np.finfo(np.float64).tiny)


def _config_key(config):
    return (config.seed, config.blocksize, config.nystrom_rank, config.grad_eval_point,
            config.lookahead, config.lam)


def adasap_step(oracle, state, Y, config, accel, pool=None, identity_precond=False):
    """One iteration t = state.iteration (solvers.py:361-403); returns
    (state, eta, block) like the reference.

    ``state`` is a ``SolverState`` (e.g. ``SolverState.zeros(n, m, True)``).
    Y, config, accel and identity_precond are read on every call: the device
    engine bound to the state is reused only while they are the same (Y the
    same array object); otherwise the state is written back and a new engine
    resumes from it. ``pool`` is accepted for API compatibility (the device
    runs all tiles in one launch). eta is read back from the device (its
    lookahead batch is produced ahead, so this does not wait for the step's
    block product; read ``state.W`` or synchronise to wait for the iterate)."""
    if not isinstance(state, SolverState):
        raise ContractError("adasap_step needs a SolverState")
    e = state._e
    key = (id(oracle), id(Y), _config_key(config), (accel.beta, accel.gamma, accel.alpha),
           bool(identity_precond))
    if e is None or getattr(e, "bind_key", None) != key:
        state._detach()
        n = oracle.n
        if state._W is None:
            raise ContractError("state has no iterate arrays")
        for A in (state._W, state._V, state._Z):
            if _as2d(A).shape[0] != n:
                raise ContractError("state arrays must have n rows")
        zero = state._zero or all(
            not np.any(np.asarray(A)) if not torch.is_tensor(A) else not bool(A.any())
            for A in (state._W, state._V, state._Z))
        e = AdasapEngine(oracle, Y, config, accel, identity_precond, unbounded=True,
                         start=state._it,
                         state=None if zero else (state._W, state._V, state._Z))
        e.bind_key = key
        e.Y_src = Y  # keeps id(Y) valid while bound
        e.prepare_readback()  # the state's arrays are read back to the host later
        state._e = e
    plan = e.step(e.eval_point(config))
    state._W = state._V = state._Z = None  # written back lazily
    state._zero = False
    return state, plan.eta_host(), plan.block


def make_state(oracle, Y, config, accel=None, identity_precond=False, total=None):
    """Fresh zero state (solvers.py:197-202) bound to a device engine with an
    iteration budget (``total``, default from the config)."""
    n = oracle.n
    b = resolve_blocksize(config, n)
    if accel is None:
        accel = resolve_accel(config, n, b)
    eng = AdasapEngine(oracle, Y, config, accel, identity_precond, total)
    eng.bind_key = (id(oracle), id(Y), _config_key(config), (accel.beta, accel.gamma, accel.alpha),
                    bool(identity_precond))
    eng.Y_src = Y
    return SolverState(eng)


def adasap_solve(oracle, Y, config, identity_precond=False, pool=None, on_iterate=None,
                 accel=None):
    """Accelerated approximate sketch-and-project from W0 = 0 (solvers.py:406-456)."""
    n = oracle.n
    config.validate_for(n)
    b = resolve_blocksize(config, n)
    if accel is None:
        accel = resolve_accel(config, n, b)
    total = budget_iterations(config, b / n)
    eng = AdasapEngine(oracle, Y, config, accel, identity_precond, total)
    # a CUDA right-hand side keeps the solve on the device: W is returned as
    # this rank's shard (fp32 CUDA tensor), never gathered to n x m
    device_out = torch.is_tensor(Y) and Y.is_cuda
    if not device_out:
        eng.prepare_readback()
    try:
        ynorm = eng.y_norm() if device_out else _y_norm(Y)
        trace = ConvergenceTrace()
        averager = TailAverager(total, (n, eng.m)) if config.tail_average else None
        diverged = False
        done = 0
        pending = []  # (iteration, passes, relres, crc) -- stepsizes filled at the end
        for t in range(total):
            plan = eng.step(eng.eval_point(config))
            done = t + 1
            W_loc = None
            if averager is not None or on_iterate is not None:
                W_loc = eng.materialize("W")
                if averager is not None:
                    averager.add(done, W_loc)
                if on_iterate is not None:
                    on_iterate(done, _to_host64(eng.gather_full(W_loc)))
            relres = math.nan
            if _due(config.residual_every, t, total):
                W_loc = eng.materialize("W") if W_loc is None else W_loc
                relres = eng.relative_residual(W_loc, ynorm)
            trace.record(done, done * b / n, relres, math.nan, plan.crc)
            if np.isfinite(relres):
                finite = bool(torch.isfinite(W_loc).all())
                if relres > DIVERGENCE_FACTOR or not finite:
                    diverged = True
                    break
                if config.tol is not None and relres <= config.tol:
                    break
        eng.la.check_flags()
        etas = eng.etas[:done].cpu().numpy()
        xfer.add("d2h", etas.nbytes)
        for rec, eta in zip(trace.records, etas):
            rec.stepsize = float(eta)
        if averager is not None and averager.count > 0:
            W_loc = averager.average()
        else:
            W_loc = eng.materialize("W")
        W = W_loc if device_out else _to_host64(eng.gather_full(W_loc), out=eng.take_readback())
    finally:
        eng.release()
    return SolveResult(W[:, 0] if eng.vector else W, trace, diverged, done, done * b / n)


def solve(oracle, Y, config, dpp_model=None, pool=None, on_iterate=None):
    """Dispatch on ``config.solver_id`` (solvers.py:591-615).

    The B200 build implements the ADASAP hot path (``adasap``, ``adasap_i``)
    and the exact-SAP, SDD and Nystrom-PCG baselines on the same kernel
    (baselines.py)."""
    if config.solver_id == "adasap":
        return adasap_solve(oracle, Y, config, on_iterate=on_iterate)
    if config.solver_id == "adasap_i":
        return adasap_solve(oracle, Y, config, identity_precond=True, on_iterate=on_iterate)
    if config.solver_id == "sdd":
        from .baselines import sdd_solve
        return sdd_solve(oracle, Y, config, pool=pool, on_iterate=on_iterate)
    if config.solver_id == "pcg":
        from .baselines import pcg_solve
        return pcg_solve(oracle, Y, config, pool=pool, on_iterate=on_iterate)
    if config.solver_id == "sap":
        from .baselines import sap_solve
        return sap_solve(oracle, Y, config, sampler=config.sampler, dpp_model=dpp_model,
                         pool=pool, on_iterate=on_iterate)
    raise ConfigError(f"unknown solver {config.solver_id!r}")
