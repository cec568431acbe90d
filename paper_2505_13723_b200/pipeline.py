"""Lookahead producer of the iterate-independent ADASAP phases.

In one ADASAP iteration t (solvers.py:361-403) everything except the
block-row product and the update depends only on (seed, t) and X:

    B_t      = sort(substream(seed, "block", t).choice(n, b))    solvers.py:375
    Omega_t  = substream(seed, "omega", t).standard_normal((b, r)) :384
    sketch   = K[B,B] Omega_t                                     :385
    (U, S)   = rand_nystrom_retry(sketch, Omega_t, r)             :386
    rho      = S[-1] + lam                                         :387
    eta_t    = rand_power_stepsize(K[B,B] + lam I, (U, S), rho,
                                   10, substream(seed, "power", t)) :389-396

so they are produced in batches on a side CUDA stream and a host worker
thread, up to two batches ahead of the main stream's block-row products.
Batch sizes ramp 1, 2, 4, ... up to ``L = config.lookahead`` so the first
iteration waits for one plan only, not for a full batch. Per batch there is one device->host
round trip (three r x r matrices per iteration) for the host LAPACK part
(``randnla.factor_core_retry``); everything dimension-b runs on the GPU in
fp64 (QR of the sketch, U = Qs Ur, the batched power iteration). Buffers
live in three preallocated slots reused under CUDA events, so nothing is
allocated in steady state.
"""

from __future__ import annotations

import math
import os
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .errors import NumericalError
from .randnla import factor_gram_retry, woodbury_core
from .rng import block_hash, substream, uniform_block


@dataclass
class IterPlan:
    t: int
    block: np.ndarray          # host, sorted int64
    crc: int
    block_dev: torch.Tensor    # (b,) int64 global ids
    loc_dev: torch.Tensor      # (b,) int64 local row or -1
    Xb: torch.Tensor           # (b, ldx) fp32 gathered points
    rsq: torch.Tensor          # (b,) fp32
    U: torch.Tensor | None     # (b, r) fp64
    Mc: torch.Tensor | None    # (r, r) fp64 Woodbury core: D = (g - U Mc U^T g) / rho
    rho: float
    eta_dev: torch.Tensor      # (1,) fp64 view
    S: np.ndarray
    RAg: torch.Tensor | None = None  # (bpad, ka) gathered tensor-core row features


class _Slot:
    def __init__(self, L, b, r, ldx, dev, ka=0):
        f32, f64, i64 = torch.float32, torch.float64, torch.int64
        self.block_dev = torch.empty((L, b), dtype=i64, device=dev)
        self.loc_dev = torch.empty((L, b), dtype=i64, device=dev)
        self.Xb = torch.empty((L, b, ldx), dtype=f32, device=dev)
        self.rsq = torch.empty((L, b), dtype=f32, device=dev)
        self.U = torch.empty((L, b, r), dtype=f64, device=dev) if r else None
        self.Mc = torch.empty((L, r, r), dtype=f64, device=dev) if r else None
        self.E = torch.zeros((L, max(r, 1)), dtype=f64, device=dev)
        self.rho = torch.ones(L, dtype=f64, device=dev)
        self.v0 = torch.empty((L, b), dtype=f64, device=dev)
        self.Kbb = torch.empty((L, b, b), dtype=f64, device=dev)
        self.graph = None  # CUDA graph of the batched power iteration (full batches)
        self.eta = torch.empty(L, dtype=f64, device=dev)
        self.bad = torch.zeros(L, dtype=torch.int32, device=dev)
        bpad = (b + 255) // 256 * 256
        self.RAg = torch.empty((L, bpad, ka), dtype=f32, device=dev) if ka else None
        pin = torch.cuda.is_available()
        self.h_block = torch.empty((L, b), dtype=i64, pin_memory=pin)
        self.h_omega = torch.empty((L, b, max(r, 1)), dtype=f64, pin_memory=pin)
        self.h_v0 = torch.empty((L, b), dtype=f64, pin_memory=pin)
        self.h_small = torch.empty((L, 3, max(r, 1), max(r, 1)), dtype=f64, pin_memory=pin)
        self.h_w = torch.empty((L, 2, max(r, 1), max(r, 1)), dtype=f64, pin_memory=pin)
        self.h_coef = torch.empty((L, max(r, 1)), dtype=f64, pin_memory=pin)
        self.h_rho = torch.empty(L, dtype=f64, pin_memory=pin)
        self.free = None      # event on the main stream: last consumer enqueued
        self.h2d_done = None  # event on the side stream: pinned inputs consumed


@dataclass
class _Batch:
    slot: _Slot
    t0: int
    count: int
    blocks: list
    crcs: list
    rho: np.ndarray
    S: list
    ready: torch.cuda.Event = field(default=None)


class Lookahead:
    """Produces IterPlan(t) for t = 0..total-1 in batches of ``L``."""

    def __init__(self, oracle, shard, seed, b, r, lam, total, L, identity_precond, power_iters=10,
                 tcp=None):
        self.o, self.shard, self.seed = oracle, shard, seed
        self.n, self.b, self.r, self.lam = oracle.n, b, (0 if identity_precond else r), lam
        # three slots of L fp64 b x b blocks: keep them under ~3 GB
        cap = max(1, int(3e9 // (3 * 8 * b * b)))
        self.total, self.L = total, max(1, min(L, total, cap))
        self.iters = power_iters
        dev = oracle.device
        self.dev = dev
        # high priority: the side chain's short kernels run in the gaps between the
        # persistent block-row kernels instead of queueing behind the next one
        self.side = torch.cuda.Stream(device=dev, priority=-1)
        self.tcp = tcp
        ka = tcp.ka if tcp is not None else 0
        self.slots = [_Slot(self.L, b, self.r, oracle.points.ldx, dev, ka) for _ in range(3)]
        # side-stream scratch of the tensor-core sketch (used one plan at a time)
        # (only for blocks of >= 512 points: below that the 256-row tiles are
        # mostly padding and the FFMA sketch, ~4x more precise, costs little)
        self.sk_zop = None
        if tcp is not None and self.r and b >= 512 and oracle.use_tc(self.r):
            self.sk_zop = K.ZOperand(self.r, b, dev)
            self.sk_cols = torch.empty((b, ka), dtype=torch.float32, device=dev)
            self.sk_pos = torch.arange(b, dtype=torch.int64, device=dev)
            need = K.nat.load().sap_krows_tc_workspace(b, self.r, b)
            self.sk_ws = torch.empty(need // 4 + 1, dtype=torch.float32, device=dev)
        # batch k covers iterations [bounds[k], bounds[k+1])
        self.bounds = [0]
        c = 1
        while self.bounds[-1] < total:
            self.bounds.append(min(total, self.bounds[-1] + c))
            c = min(2 * c, self.L)
        self.pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="sap-lookahead")
        # host workers for the per-iteration numpy RNG and r x r LAPACK work (both
        # release the GIL in their kernels); sized to leave cores for the main thread
        try:
            cores = len(os.sched_getaffinity(0))
        except AttributeError:  # pragma: no cover
            cores = os.cpu_count() or 1
        self.hostpool = ThreadPoolExecutor(max_workers=max(1, min(self.L, cores - 2, 8)),
                                           thread_name_prefix="sap-host")
        self.timings = [] if os.environ.get("SAP_PROFILE") else None
        # r x r LAPACK calls from several host workers: one BLAS thread each (the
        # reference pins BLAS to one thread for the same reason, __init__.py:16-22)
        try:
            from threadpoolctl import threadpool_limits
            self._blas_limit = threadpool_limits(limits=1, user_api="blas")
        except Exception:  # pragma: no cover - threadpoolctl is optional
            self._blas_limit = None
        self.cur = None
        self.k = -1  # batch currently consumed
        # capture both slots' power-iteration graphs up front (static buffers; the
        # values are filled per batch), so no capture lands inside a timed solve
        if self.L > 1:
            with torch.cuda.device(dev), torch.cuda.stream(self.side):
                for slot in self.slots:
                    slot.v0.fill_(1.0)
                    slot.Kbb.zero_()
                    self._power(slot, self.L)  # warm-up (allocator, cuBLAS handles)
                    slot.graph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(slot.graph, stream=self.side,
                                          capture_error_mode="thread_local"):
                        self._power(slot, self.L)
                    slot.bad.zero_()
        self.futs = {}
        for k in range(min(2, len(self.bounds) - 1)):
            self._submit(k)

    def _submit(self, k):
        t0, t1 = self.bounds[k], self.bounds[k + 1]
        self.futs[k] = self.pool.submit(self._produce, self.slots[k % 3], t0, t1 - t0)

    def close(self):
        self.pool.shutdown(wait=True)
        self.hostpool.shutdown(wait=True)
        if self._blas_limit is not None:
            self._blas_limit.restore_original_limits()
            self._blas_limit = None

    # -- consumer side (main thread) ------------------------------------------
    def get(self, t):
        cur = self.cur
        if cur is None or t >= cur.t0 + cur.count:
            main = torch.cuda.current_stream(self.dev)
            if cur is not None:
                ev = torch.cuda.Event()
                ev.record(main)
                cur.slot.free = ev  # batch k+2 refills this slot after it
            self.k += 1
            cur = self.futs.pop(self.k).result()
            main.wait_event(cur.ready)
            self.cur = cur
            if self.k + 2 < len(self.bounds) - 1:
                self._submit(self.k + 2)
        i = t - cur.t0
        s = cur.slot
        return IterPlan(
            t=t, block=cur.blocks[i], crc=cur.crcs[i], block_dev=s.block_dev[i],
            loc_dev=s.loc_dev[i], Xb=s.Xb[i], rsq=s.rsq[i],
            U=None if s.U is None else s.U[i], Mc=None if s.Mc is None else s.Mc[i],
            rho=float(cur.rho[i]), eta_dev=s.eta[i:i + 1], S=cur.S[i],
            RAg=None if s.RAg is None else s.RAg[i])

    def check_flags(self):
        """Raise if any power iteration failed (checked once, at the end)."""
        for s in self.slots:
            if int(s.bad.max()) != 0:
                raise NumericalError("power iteration failed (collapsed or nonpositive Rayleigh "
                                     "estimate; H is not PSD)")

    # -- producer side (worker thread) ------------------------------------------
    def _produce(self, slot, t0, count):
        b, r, seed, n = self.b, self.r, self.seed, self.n
        if slot.h2d_done is not None:
            slot.h2d_done.synchronize()  # pinned inputs of the previous use consumed
        tm0 = time.perf_counter()

        def draw(i):
            t = t0 + i
            blk = uniform_block(seed, t, n, b).astype(np.int64)
            slot.h_block[i].numpy()[:] = blk
            if r:
                slot.h_omega[i].numpy()[:] = substream(seed, "omega", t).standard_normal((b, r))
            rng = substream(seed, "power", t)
            v = rng.standard_normal(b)
            nv = np.linalg.norm(v)
            if nv == 0.0:
                v = rng.standard_normal(b)
                nv = np.linalg.norm(v)
                if nv == 0.0:
                    raise NumericalError("power iteration start vector is zero")
            slot.h_v0[i].numpy()[:] = v / nv
            return blk, block_hash(blk)

        drawn = list(self.hostpool.map(draw, range(count)))
        blocks = [d[0] for d in drawn]
        crcs = [d[1] for d in drawn]
        tm1 = time.perf_counter()
        side = self.side
        pts = self.o.points
        with torch.cuda.device(self.dev), torch.cuda.stream(side):
            if slot.free is not None:
                side.wait_event(slot.free)
            slot.block_dev[:count].copy_(slot.h_block[:count], non_blocking=True)
            slot.v0[:count].copy_(slot.h_v0[:count], non_blocking=True)
            om = slot.h_omega[:count].to(self.dev, non_blocking=True) if r else None
            bd = slot.block_dev[:count]
            slot.loc_dev[:count].copy_(self.shard.local_positions(bd))
            sketch = torch.empty((count, b, max(r, 1)), dtype=torch.float32, device=self.dev)
            for i in range(count):
                Xb, rsq = pts.gather(bd[i], out=(slot.Xb[i], slot.rsq[i]))
                if self.tcp is not None:
                    self.tcp.gather_rows(bd[i], out=slot.RAg[i])
                if r:
                    omc = om[i].T.to(torch.float32).contiguous()  # (r, b) column-major RHS
                    if self.sk_zop is not None:
                        # K[B,B] Omega on the tensor cores: the block's own points
                        # as columns, rows matched to columns by block position
                        self.tcp.gather_cols(bd[i], out=self.sk_cols)
                        self.sk_zop.fill(omc)
                        K.krows_tc(self.o.spec, self.tcp, slot.RAg[i], b, self.sk_pos,
                                   self.sk_zop, sketch[i], ws=self.sk_ws, cols=(self.sk_cols, 0))
                    else:
                        K.krows_times(self.o.spec, _Cols(pts, Xb, rsq), Xb, rsq, bd[i], omc,
                                      sketch[i], col_ids=bd[i])
            if r:
                Y = sketch.to(torch.float64)
                omt = om.transpose(1, 2)
                small = torch.stack([Y.transpose(1, 2) @ Y, omt @ Y, omt @ om], dim=1)
                slot.h_small[:count].copy_(small, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        rho = np.empty(count)
        tm2 = time.perf_counter()
        if r:
            ev.synchronize()
            tm2 = time.perf_counter()
            hs = slot.h_small[:count].numpy()
            hom = slot.h_omega

            def factor(i):
                W, S, UtU = factor_gram_retry(hs[i, 0], hs[i, 1], hs[i, 2], r,
                                              omega_rank=lambda: np.linalg.matrix_rank(
                                                  hom[i].numpy()))
                rho_i = float(S[-1]) + self.lam
                slot.h_w[i, 0].numpy()[:] = W
                slot.h_w[i, 1].numpy()[:] = woodbury_core(S, UtU, rho_i)
                slot.h_coef[i].numpy()[:] = 1.0 / np.sqrt(S + rho_i) - 1.0 / math.sqrt(rho_i)
                return rho_i, S

            res = list(self.hostpool.map(factor, range(count)))
            rho[:] = [x[0] for x in res]
            Ss = [x[1] for x in res]
        else:
            ev.synchronize()  # pinned inputs consumed before the slot is refilled
            rho[:] = 1.0
            Ss = [np.zeros(0)] * count
        tm3 = time.perf_counter()
        slot.h_rho[:count].numpy()[:] = rho
        with torch.cuda.device(self.dev), torch.cuda.stream(side):
            for i in range(count):
                Xb, rsq = slot.Xb[i], slot.rsq[i]
                slot.Kbb[i] = K.ktile(self.o.spec, Xb, rsq, bd[i], Xb, rsq, bd[i], pts.ldx, pts.d)
            slot.rho[:count].copy_(slot.h_rho[:count], non_blocking=True)
            if r:
                w = slot.h_w[:count].to(self.dev, non_blocking=True)
                torch.bmm(Y, w[:, 0], out=slot.U[:count])
                slot.Mc[:count].copy_(w[:, 1])
                slot.E[:count].copy_(slot.h_coef[:count], non_blocking=True)
            if count == self.L and slot.graph is not None:
                slot.graph.replay()
            else:
                self._power(slot, count)
            ready = torch.cuda.Event()
            ready.record(side)
            slot.h2d_done = ready  # pinned host buffers reusable after this point
        if self.timings is not None:
            self.timings.append(dict(count=count, rng=tm1 - tm0, gpu_wait=tm2 - tm1,
                                     factor=tm3 - tm2, total=time.perf_counter() - tm0))
        return _Batch(slot, t0, count, blocks, crcs, rho, Ss, ready)

    def _power(self, slot, count):
        """Batched rand_power_stepsize (randnla.py:165-196) on P^{-1/2}(K+lam)P^{-1/2},
        P^{-1/2} x = x/sqrt(rho) + U diag((S+rho)^{-1/2} - rho^{-1/2}) U^T x,
        from the slot's static buffers (so full batches replay as one CUDA graph)."""
        Kbb, v, U, E = slot.Kbb[:count], slot.v0[:count], None, slot.E[:count]
        if self.r:
            U = slot.U[:count]
        isr = slot.rho[:count].rsqrt()[:, None]

        def pinv_sqrt(x):
            y = x * isr
            if U is not None:
                y = y + torch.bmm(U, (E * torch.bmm(U.transpose(1, 2), x[:, :, None])[:, :, 0])
                                  [:, :, None])[:, :, 0]
            return y

        bad = torch.zeros(count, dtype=torch.bool, device=self.dev)
        est = None
        for _ in range(self.iters):
            w = pinv_sqrt(v)
            z = torch.bmm(Kbb, w[:, :, None])[:, :, 0] + self.lam * w
            y = pinv_sqrt(z)
            est = (v * y).sum(dim=1)
            ny = torch.linalg.vector_norm(y, dim=1)
            bad |= ny == 0
            v = y / ny[:, None]
        bad |= est <= 0
        slot.eta[:count].copy_(1.0 / est)
        slot.bad[:count].bitwise_or_(bad.to(torch.int32))


class _Cols:
    """A gathered point subset viewed as a column point set."""

    def __init__(self, pts, Xs, sqn):
        self.Xs, self.sqn = Xs, sqn
        self.n, self.d, self.ldx, self.device = Xs.shape[0], pts.d, pts.ldx, pts.device
