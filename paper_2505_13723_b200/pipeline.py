"""Lookahead producer of the iterate-independent ADASAP phases.

In one ADASAP iteration t (solvers.py:361-403) everything except the
block-row product and the update depends only on (seed, t) and X:

    B_t      = sort(substream(seed, "block", t).choice(n, b))    solvers.py:375
    Omega_t  = substream(seed, "omega", t).standard_normal((b, r)) :384  (drawn on the GPU)
    sketch   = K[B,B] Omega_t                                     :385
    (U, S)   = rand_nystrom_retry(sketch, Omega_t, r)             :386
    rho      = S[-1] + lam                                         :387
    eta_t    = rand_power_stepsize(K[B,B] + lam I, (U, S), rho,
                                   10, substream(seed, "power", t)) :389-396

so they are produced in batches by ``depth`` (default 6) host producer
threads, up to ``depth`` batches ahead of the block-row products that
consume them; their GPU work is enqueued in order on the solver's stream
(see Lookahead.__init__). Batch sizes ramp 1, 4, 16, ... up to
``L = config.lookahead`` so the first iteration waits for one plan only, not
for a full batch. The host draws the blocks (numpy-exact, csrc/host_rng.cu)
and enqueues; everything else runs on the GPU with no device->host round
trip: Omega, the sketch, the Gram matrices, the whole r x r factorisation
(shift ladder, Jacobi eigensolves, Woodbury core, rho;
``randnla.factor_gram_batch``), U = Y W, K[B,B] and the batched power
iteration. Failures the reference raises at the failing step are flagged on
the device and raised by ``check_flags``. Buffers
live in depth + 1 preallocated slots reused under CUDA events, so nothing is
allocated in steady state.
"""

from __future__ import annotations

import os
import sys
import threading
import time
import warnings
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from . import xfer
from .errors import NumericalError
from .errors import ContractError
from .randnla import (FLAG_CHOLESKY, FLAG_EIGH, FLAG_EXTRA_SHIFT, FLAG_NEG_TRACE, FLAG_PLAIN,
                      FLAG_POWER, factor_gram_batch)
from .rng import DeviceNormals


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
    UMc: torch.Tensor | None   # (b, r) fp64 U Mc (precomputed, one GEMM less per step)
    rho: float                 # host value (nan on ranks that did not produce the batch)
    eta_dev: torch.Tensor      # (1,) fp64 view
    S: np.ndarray
    RAg: torch.Tensor | None = None  # (bpad, ka) gathered tensor-core row features
    eta_host: object = None          # () -> float: eta_t read back once its batch is produced
    rho_dev: torch.Tensor | None = None  # (1,) fp64 view of rho on the device
    eta_rho_dev: torch.Tensor | None = None  # (1,) eta / rho: the update of an unscaled D
    batch_t0: int = -1                   # first iteration of this plan's lookahead batch
    batch_eta: torch.Tensor | None = None  # the batch's stepsizes (device)


# One production stream per (device, priority) for the whole process, reused
# by every engine: the caching allocator keeps freed blocks in the pool of the
# stream they were allocated on, so a fresh stream per engine made every new
# engine's production allocate (cudaMalloc, ~15 segments) instead of reusing
# the previous engine's blocks, and stalled the first steps after each bind.
_FAST_STREAMS = {}
_FAST_LOCK = threading.Lock()


def _fast_stream(dev, priority):
    key = (torch.device(dev).index, priority)
    with _FAST_LOCK:
        st = _FAST_STREAMS.get(key)
        if st is None:
            st = _FAST_STREAMS[key] = torch.cuda.Stream(device=dev, priority=priority)
        return st


class _Slot:
    def __init__(self, L, b, r, ldx, dev, ka=0, fdtype=torch.float32):
        f32, f64, i64 = torch.float32, torch.float64, torch.int64
        self.block_dev = torch.empty((L, b), dtype=i64, device=dev)
        self.loc_dev = torch.empty((L, b), dtype=i64, device=dev)
        self.Xb = torch.empty((L, b, ldx), dtype=f32, device=dev)
        self.rsq = torch.empty((L, b), dtype=f32, device=dev)
        self.U = torch.empty((L, b, r), dtype=f64, device=dev) if r else None
        self.Mc = torch.empty((L, r, r), dtype=f64, device=dev) if r else None
        self.UMc = torch.empty((L, b, r), dtype=f64, device=dev) if r else None  # U Mc
        self.E = torch.zeros((L, max(r, 1)), dtype=f64, device=dev)
        self.rho = torch.ones(L, dtype=f64, device=dev)
        self.v0 = torch.empty((L, b), dtype=f64, device=dev)
        # K_BB in fp32: the values the tile kernel computes (fp32 arithmetic),
        # streamed once per power step by sap_power_stepsize
        # zeroed when rows are padded: the power kernel reads rows in 16-byte
        # chunks through the pad columns (times a zero w), and never-written
        # pad bits must not be NaN; with b % 4 == 0 there is no pad and the
        # tile kernel writes every entry a plan uses (no 512 MB memset per slot)
        alloc = torch.empty if b % 4 == 0 else torch.zeros
        self.Kbb = alloc((L, b, (b + 3) // 4 * 4), dtype=torch.float32, device=dev)
        self.eta = torch.empty(L, dtype=f64, device=dev)
        self.eta_rho = torch.empty(L, dtype=f64, device=dev)  # eta / rho (Phase IV's 1/rho folded)
        self.bad = torch.zeros(L, dtype=torch.int32, device=dev)
        # a batch's products, packed for the owner rank's broadcast (multi-GPU):
        # [U (b r), Mc (r r), E (r), rho, eta, bad] per iteration
        self.nprod = b * r + r * r + r + 3
        self.prod = torch.empty((L, self.nprod), dtype=f64, device=dev)
        bpad = (b + 255) // 256 * 256
        # pad rows b..bpad zero once (the batched gather writes rows < b only)
        self.RAg = torch.zeros((L, bpad, ka), dtype=fdtype, device=dev) if ka else None
        pin = torch.cuda.is_available()
        self.h_block = torch.empty((L, b), dtype=i64, pin_memory=pin)
        # Omega_t is drawn on the GPU from the omega stream's PCG64 state
        # (csrc/rng.cu, numpy-exact); the host only seeds the streams
        self.h_states = torch.empty((L, 4), dtype=i64, pin_memory=pin)
        self.states = torch.empty((L, 4), dtype=i64, device=dev)
        self.omega = torch.empty((L, b, r), dtype=f64, device=dev) if r else None
        self.normals = DeviceNormals(b * r, L, dev) if r else None
        self.h_v0 = torch.empty((L, b), dtype=f64, pin_memory=pin)
        self.h_eta = torch.empty(L, dtype=f64, pin_memory=pin)
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
    eta_ready: torch.cuda.Event = field(default=None)
    owner: int = 0


class Lookahead:
    """Produces IterPlan(t) for t = start..total-1 (total None: unbounded) in
    batches of up to ``L``."""

    _WIDTH = int(os.environ.get("SAP_PRODUCE_WIDTH", "2"))  # batches produced concurrently
    _RAMP = max(2, int(os.environ.get("SAP_RAMP", "4")))    # batch-size growth of the ramp
    # explicit leading batch sizes (SAP_RAMP_SIZES="1,4,8"), then growth by _RAMP
    _SIZES = tuple(int(x) for x in os.environ.get("SAP_RAMP_SIZES", "").split(",") if x.strip())

    def __init__(self, oracle, shard, seed, b, r, lam, total, L, identity_precond, power_iters=10,
                 tcp=None, start=0):
        self.o, self.shard, self.seed = oracle, shard, int(seed)
        if not 0 <= self.seed < 2**64:
            raise ContractError("seed must be a non-negative integer below 2**64")
        self.n, self.b, self.r, self.lam = oracle.n, b, (0 if identity_precond else r), lam
        # batches produced concurrently (one producer thread each, depth + 1
        # slots): a producer spends most of a batch waiting -- for its sketch,
        # queued behind the block products already enqueued, and on the host
        # factorisation -- so two producers left the solver host-bound at ~1.43
        # ms per RBF iteration against 1.25 with four (scripts/host_bound.py,
        # config 3); SAP_LOOKAHEAD_DEPTH overrides
        # (round 2: with the factorisation on the device a producer no longer
        # waits on the host; depth 6 keeps a fresh engine's ramp (batches of 1,
        # 2, 4, ...) from stalling the first steps -- 19 steps after a bind in
        # 30 ms instead of 42-390 ms at depth 4 -- at the same steady rate)
        self.depth = max(2, int(os.environ.get("SAP_LOOKAHEAD_DEPTH", "6")))
        # depth + 1 slots of L fp32 b x b blocks: keep them under ~4 GB
        # slots: depth in production + the one being consumed + SAP_SPARE_SLOTS
        # (default 1): a batch's production first waits until its slot's
        # previous batch has left the device; one spare slot makes that the
        # batch before last, not the last one
        self.nslots = self.depth + 1 + max(0, int(os.environ.get("SAP_SPARE_SLOTS", "1")))
        cap = max(1, int(4e9 // (self.nslots * 4 * b * b)))
        # total None: unbounded (the per-step API); batches are defined lazily
        self.total = total
        self.L = max(1, min(L, cap) if total is None else min(L, total, cap))
        self.iters = power_iters
        dev = oracle.device
        self.dev = dev
        # Production is enqueued in order on the solver's stream. The block-row
        # kernel is persistent (one CTA per SM, registers and shared memory
        # full), so nothing co-runs with it: a side-stream kernel that takes
        # the SMs a draining block-row kernel frees holds the next one back
        # (measured, config 3 on one B200: 380-430 iters/s with per-slot
        # high-priority side streams, krows up to 2.6 ms; 470-520 in order).
        # SAP_SIDE_STREAM=1 selects the side streams for experiments.
        self.main = torch.cuda.current_stream(dev)
        if os.environ.get("SAP_SIDE_STREAM", "0") == "1":
            self.sides = [torch.cuda.Stream(device=dev, priority=-1) for _ in range(self.nslots)]
        else:
            self.sides = [torch.cuda.current_stream(dev)] * self.nslots
        # the first production phase (Omega, gathers, sketch, Gram matrices --
        # what the producer waits for before its host factorisation) runs on a
        # high-priority stream: on the solver's stream it sat behind every
        # block product already queued (~7 ms of producer wait per iteration
        # at lookahead depth 4); its kernels are short, so they slip in between
        # two block products. SAP_FAST_STREAM=0 keeps it on the solver's stream.
        if os.environ.get("SAP_FAST_STREAM", "1") == "1":
            self.fast = _fast_stream(dev, int(os.environ.get("SAP_FAST_PRIORITY", "-1")))
        else:
            self.fast = None
        self.tcp = tcp
        ka = tcp.ka if tcp is not None else 0
        fdt = tcp.dtype if tcp is not None else torch.float32
        xfer.mark("lookahead: streams")
        self.slots = [_Slot(self.L, b, self.r, oracle.points.ldx, dev, ka, fdt)
                      for _ in range(self.nslots)]
        xfer.mark("lookahead: slots")
        # per-slot scratch of the tensor-core sketch (used one plan at a time by
        # the slot's producer)
        # (only for blocks of >= 512 points: below that the 256-row tiles are
        # mostly padding and the FFMA sketch, ~4x more precise, costs little)
        # the sketch K[B,B] Omega: by default a batched fp32 GEMM against the
        # K_BB tiles the power iteration needs anyway (SAP_SKETCH=tc: the
        # block-row kernel with the block's own points as columns, round 1)
        mode = os.environ.get("SAP_SKETCH", "gemm")
        self.sketch_gemm = mode in ("gemm", "gemm32")
        # the GEMM in three fp16 tensor-core passes (K_BB / variance and Omega
        # split hi + lo by the tile kernel / here, fp32 accumulation: 0.25 ms
        # against 0.63 ms for the fp32 SIMT GEMM per batch of 31 at b = 2000,
        # 3.2e-6 against 2.2e-6 relative error; scripts/sketch_probe.py); the
        # fp16 copies cost 2 b^2 bytes per slot iteration, so only up to
        # b = 4096 (SAP_SKETCH=gemm32: the fp32 GEMM)
        self.sketch_split = mode == "gemm" and bool(self.r) and b <= 4096
        if self.sketch_split:
            ldh = (b + 7) // 8 * 8
            for slot in self.slots:
                slot.Kh = torch.empty((self.L, b, ldh), dtype=torch.float16, device=dev)
                slot.Kl = torch.empty((self.L, b, ldh), dtype=torch.float16, device=dev)
        self.tc_sketch = (not self.sketch_gemm and tcp is not None and self.r and b >= 512
                          and oracle.use_tc(self.r))
        if self.tc_sketch:
            self.sk_pos = torch.arange(b, dtype=torch.int64, device=dev)
            need = K.nat.load().sap_krows_tc_workspace(b, self.r, b)
            for slot in self.slots:
                slot.sk_zop = K.ZOperand(self.r, b, dev)
                slot.sk_cols = torch.empty((self.L, b, ka), dtype=fdt, device=dev)
                slot.sk_bound = torch.empty(self.L * self.r, dtype=torch.float32, device=dev)
                slot.sk_ws = torch.empty(need // 4 + 1, dtype=torch.float32, device=dev)
        # torch.linalg's CUDA backends initialise lazily and not thread-safely:
        # touch the ones the producers use here, before any producer runs
        if self.r:
            with torch.cuda.device(dev):
                _a = torch.eye(2, dtype=torch.float64, device=dev)[None]
                _l, _ = torch.linalg.cholesky_ex(_a)
                torch.cholesky_inverse(_l)
                torch.linalg.solve_triangular(_l, _a, upper=False)
            xfer.mark("lookahead: linalg init")
        # batch k covers iterations [bounds[k], bounds[k+1]); sizes ramp 1, 4,
        # 16, ... up to L, extended on demand (_has_batch). Growth 4 rather
        # than 2: a batch's host-side cost is mostly per batch, not per
        # iteration, and fewer ramp batches kept a fresh engine's first 20
        # steps from waiting on production (34-36 ms against 38-41 ms with
        # 1, 2, 4, 8, 16; scripts/e2e_phases.py, SAP_RAMP)
        self.bounds = [int(start)]
        self._c = 1
        # depth producers: a batch's production (host RNG -> sketch on the GPU ->
        # host factorisation -> power iteration) takes longer than consuming
        # one, so depth batches are produced concurrently (slots k mod depth+1)
        self.pool = ThreadPoolExecutor(max_workers=self.depth, thread_name_prefix="sap-lookahead")
        # host threads of the native block draws (sap_host_draws, GIL released);
        # sized to leave cores for the main thread
        try:
            cores = len(os.sched_getaffinity(0))
        except AttributeError:  # pragma: no cover
            cores = os.cpu_count() or 1
        self.host_threads = max(1, min(self.L, cores - 2, 8))
        self.timings = [] if os.environ.get("SAP_PROFILE") else None
        # The solver thread enqueues its launches and must keep ahead of the
        # device while the producer threads run Python: with CPython's default 5 ms GIL
        # switch interval it can wait a whole interval for the GIL, longer than
        # an iteration's device time. 0.2 ms bounds that wait.
        swi = float(os.environ.get("SAP_SWITCH_INTERVAL", "2e-4"))
        if sys.getswitchinterval() > swi:
            sys.setswitchinterval(swi)
        self.cur = None
        self.k = -1  # batch currently consumed
        self.futs = {}
        self._gate = {}  # batch -> Event: its production has been enqueued
        for k in range(self.depth):
            if self._has_batch(k):
                self._submit(k)

    def _has_batch(self, k):
        """Define batches up to k (lazily); False past the iteration budget."""
        while len(self.bounds) <= k + 1 and (self.total is None or self.bounds[-1] < self.total):
            j = len(self.bounds) - 1  # index of the batch being defined
            c = min(self._SIZES[j], self.L) if j < len(self._SIZES) else self._c
            nxt = self.bounds[-1] + c
            self.bounds.append(nxt if self.total is None else min(self.total, nxt))
            self._c = min(self._RAMP * c, self.L)
        return len(self.bounds) > k + 1

    def _submit(self, k):
        t0, t1 = self.bounds[k], self.bounds[k + 1]
        ns = len(self.slots)
        owner = k % self.shard.world
        self._gate[k] = threading.Event()
        self.futs[k] = self.pool.submit(self._gated, k, self.slots[k % ns], t0, t1 - t0,
                                        self.sides[k % ns], owner)

    def _gated(self, k, *args):
        """Batch k's host-side production starts once batch k - _WIDTH has
        been enqueued: a fresh engine submits its first ``depth`` batches at
        once, and six producers sharing the GIL took ~35 ms to enqueue the
        one-iteration batch 0 that the first step waits for (~5 ms alone).
        In steady state the gate is long open when a batch is submitted."""
        prev = self._gate.get(k - self._WIDTH)
        if prev is not None:
            prev.wait()
            self._gate.pop(k - self._WIDTH, None)
        try:
            return self._produce(*args)
        finally:
            self._gate[k].set()

    def close(self):
        # batches not started yet are dropped; running producers finish their
        # enqueued device work before the slots can be released
        self.pool.shutdown(wait=True, cancel_futures=True)
        # hand the slot buffers (GBs at config 3) back to the caching allocator
        # now, not whenever the engine's reference cycles are collected: the
        # next engine reuses them instead of calling cudaMalloc
        self.futs.clear()
        self.cur = None
        self.slots = []

    # -- consumer side (main thread) ------------------------------------------
    def get(self, t):
        cur = self.cur
        if cur is None or t >= cur.t0 + cur.count:
            main = torch.cuda.current_stream(self.dev)
            if cur is not None:
                ev = torch.cuda.Event()
                ev.record(main)
                cur.slot.free = ev  # batch k+2 refills this slot after it
            if not self._has_batch(self.k + 1):
                raise ContractError(f"iteration {t} is past the solver's iteration budget "
                                    f"({self.total})")
            self.k += 1
            xfer.mark(f"get batch {self.k}")
            cur = self.futs.pop(self.k).result()
            xfer.mark(f"got batch {self.k}")
            main.wait_event(cur.ready)
            if self.shard.world > 1:
                self._share(cur)
            self.cur = cur
            if self._has_batch(self.k + self.depth):
                self._submit(self.k + self.depth)
        i = t - cur.t0
        s = cur.slot
        ev, h_eta = cur.eta_ready, s.h_eta

        def eta_host():
            ev.synchronize()
            return float(h_eta[i])

        return IterPlan(
            t=t, block=cur.blocks[i], crc=cur.crcs[i], block_dev=s.block_dev[i],
            loc_dev=s.loc_dev[i], Xb=s.Xb[i], rsq=s.rsq[i],
            U=None if s.U is None else s.U[i], Mc=None if s.Mc is None else s.Mc[i],
            UMc=None if s.UMc is None else s.UMc[i],
            rho=float(cur.rho[i]), eta_dev=s.eta[i:i + 1], S=cur.S[i],
            RAg=None if s.RAg is None else s.RAg[i], eta_host=eta_host,
            rho_dev=s.rho[i:i + 1], eta_rho_dev=s.eta_rho[i:i + 1], batch_t0=cur.t0,
            batch_eta=s.eta[:cur.count])

    def _share(self, cur):
        """Multi-GPU: batch k's Nystrom/stepsize products were computed by rank
        k % world only (Phases II-III round-robin); one NCCL
        broadcast of the packed products per batch, issued by every rank's main
        thread in batch order, so collective order is identical on all ranks."""
        s, n, b, r = cur.slot, cur.count, self.b, self.r
        P = s.prod[:n]
        owner = cur.owner == self.shard.rank
        if owner:
            o = 0
            if r:
                P[:, o:o + b * r].copy_(s.U[:n].reshape(n, b * r)); o += b * r
                P[:, o:o + r * r].copy_(s.Mc[:n].reshape(n, r * r)); o += r * r
                P[:, o:o + r].copy_(s.E[:n, :r]); o += r
            else:
                o = b * r + r * r + r
            P[:, o].copy_(s.rho[:n]); P[:, o + 1].copy_(s.eta[:n])
            P[:, o + 2].copy_(s.bad[:n].to(torch.float64))
        torch.distributed.broadcast(P, src=cur.owner)
        if not owner:
            o = 0
            if r:
                s.U[:n].copy_(P[:, o:o + b * r].reshape(n, b, r)); o += b * r
                s.Mc[:n].copy_(P[:, o:o + r * r].reshape(n, r, r)); o += r * r
                s.E[:n, :r].copy_(P[:, o:o + r]); o += r
            else:
                o = b * r + r * r + r
            s.rho[:n].copy_(P[:, o]); s.eta[:n].copy_(P[:, o + 1])
            torch.div(s.eta[:n], s.rho[:n], out=s.eta_rho[:n])
            s.bad[:n] |= P[:, o + 2].to(torch.int32)
            if r:
                torch.bmm(s.U[:n], s.Mc[:n], out=s.UMc[:n])
            s.h_eta[:n].copy_(s.eta[:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.dev))
            cur.eta_ready = ev

    def check_flags(self):
        """Raise the failures the reference raises at the failing step (device
        RNG, factorisation, power iteration), and warn for the fallbacks;
        checked once, at the end (flags are sticky per slot)."""
        bits = 0
        for s in self.slots:
            if s.normals is not None and int(s.normals.status()) != 0:
                raise NumericalError("device normal draw ran out of raw stream words")
            bits |= int(np.bitwise_or.reduce(s.bad.cpu().numpy()))
            xfer.add("d2h", s.bad.numel() * 4 + (4 if s.normals is not None else 0))
        if bits & FLAG_NEG_TRACE:
            raise NumericalError("sketch Gram has negative trace; M is not PSD")
        if bits & FLAG_CHOLESKY:
            raise NumericalError("Cholesky of the shifted Gram failed; retry with a larger shift")
        if bits & FLAG_EIGH:
            raise NumericalError("Jacobi eigensolver of the Nystrom Gram did not converge")
        if bits & FLAG_POWER:
            raise NumericalError("power iteration failed (collapsed or nonpositive Rayleigh "
                                 "estimate; H is not PSD)")
        if bits & FLAG_PLAIN:
            warnings.warn("stabilized Woodbury Cholesky failed; falling back to the plain "
                          "identity", RuntimeWarning)
        if bits & FLAG_EXTRA_SHIFT:
            warnings.warn("Nystrom Gram needed a shift beyond the reference ladder "
                          "(SAP_EXTRA_SHIFTS=1)", RuntimeWarning)

    # -- producer side (worker thread) ------------------------------------------
    def _host_draws(self, slot, t0, count, omega, v0):
        """Iterations t0..t0+count-1: blocks, crcs, omega PCG64 words and power
        start vectors written into the slot's pinned buffers by
        ``sap_host_draws`` (numpy-exact, csrc/host_rng.cu; GIL released, on
        the host workers' thread budget). Returns host copies of the blocks
        (the pinned rows are refilled when the slot is reused) and the crcs."""
        crcs = np.empty(count, dtype=np.uint32)
        K.nat.call("sap_host_draws", self.seed, t0, count, self.n, self.b,
                   slot.h_block.data_ptr(), crcs.ctypes.data,
                   slot.h_states.data_ptr() if omega else None,
                   slot.h_v0.data_ptr() if v0 else None, self.host_threads)
        blocks = slot.h_block[:count].numpy().copy()
        return list(blocks), [int(c) for c in crcs]

    def _produce(self, slot, t0, count, side, owner=0):
        if owner != self.shard.rank:
            return self._produce_blocks(slot, t0, count, side, owner)
        b, r = self.b, self.r
        if slot.h2d_done is not None:
            slot.h2d_done.synchronize()  # pinned inputs of the previous use consumed
        tm0 = time.perf_counter()
        xfer.mark(f"produce {t0}+{count} start")
        blocks, crcs = self._host_draws(slot, t0, count, omega=bool(r), v0=True)
        xfer.mark("draws")
        tm1 = time.perf_counter()
        pts = self.o.points
        fs = self.fast if self.fast is not None else side
        with torch.cuda.device(self.dev), torch.cuda.stream(fs):
            if slot.free is not None:
                fs.wait_event(slot.free)
            slot.block_dev[:count].copy_(slot.h_block[:count], non_blocking=True)
            slot.v0[:count].copy_(slot.h_v0[:count], non_blocking=True)
            xfer.add("h2d", count * b * 16 + (count * 32 if r else 0))
            om = None
            if r:
                slot.states[:count].copy_(slot.h_states[:count], non_blocking=True)
                om = slot.omega[:count]
                slot.normals.fill(slot.states, om.view(count, b * r), nstreams=count)
            xfer.mark("normals")
            bd = slot.block_dev[:count]
            slot.loc_dev[:count].copy_(self.shard.local_positions(bd))
            xfer.mark("loc")
            sketch = torch.empty((count, b, max(r, 1)), dtype=torch.float32, device=self.dev)
            xfer.mark("empty")
            # the batch's gathers, feature conversions and column bounds in one
            # launch each; per iteration only the sketch's Z operand and product
            flat = bd.reshape(-1)
            pts.gather(flat, out=(slot.Xb[:count].view(-1, pts.ldx), slot.rsq[:count].view(-1)))
            xfer.mark("gather")
            if self.tcp is not None:
                self.tcp.gather_rows_batch(bd, slot.RAg[:count])
                xfer.mark("gather rows")
            if r and self.sketch_split:
                # K_BB once per iteration (the power iteration's operand), and
                # K_BB / variance as fp16 hi + lo; the sketch K_BB Omega
                # (row_dist_matmul, dist.py:130-147) = variance (Kh Oh + Kh Ol +
                # Kl Oh) in two batched tensor-core GEMMs, fp32 accumulation
                K.ktile_f32_batch_split(self.o.spec, slot.Xb[:count], slot.rsq[:count], pts.d,
                                        slot.Kbb[:count], slot.Kh[:count], slot.Kl[:count])
                xfer.mark("kbb")
                oh = om.to(torch.float16)
                ohl = torch.cat([oh, (om - oh.to(torch.float64)).to(torch.float16)], dim=2)
                o1 = torch.bmm(slot.Kh[:count, :, :b], ohl, out_dtype=torch.float32)
                o2 = torch.bmm(slot.Kl[:count, :, :b], oh, out_dtype=torch.float32)
                torch.add(o1[:, :, :r], o1[:, :, r:], out=sketch)
                sketch.add_(o2).mul_(self.o.spec.variance)
                xfer.mark("sketch")
            elif r and self.sketch_gemm:
                # K_BB once per iteration (the power iteration's operand too),
                # then the sketch K_BB Omega as one batched fp32 GEMM
                # (row_dist_matmul, dist.py:130-147; 2 b^2 r flop per iteration)
                K.ktile_f32_batch(self.o.spec, slot.Xb[:count], slot.rsq[:count], pts.d,
                                  slot.Kbb[:count])
                xfer.mark("kbb")
                torch.bmm(slot.Kbb[:count, :, :b], om.to(torch.float32), out=sketch)
                xfer.mark("sketch")
            elif r:
                omc = om.transpose(1, 2).to(torch.float32).contiguous()  # (count, r, b) RHS
                if self.tc_sketch:
                    # K[B,B] Omega on the tensor cores: the block's own points as
                    # columns, rows matched to columns by block position
                    cols = slot.sk_cols[:count]
                    self.tcp.gather_cols(flat, out=cols.view(-1, cols.shape[2]))
                    bound = slot.sk_bound[:count * r]
                    K.nat.call("sap_colabsmax", K.nat.ptr(omc), b, b, count * r,
                               K.nat.ptr(bound), K.nat.stream_handle())
                for i in range(count):
                    if self.tc_sketch:
                        slot.sk_zop.fill(omc[i], Pb=bound[i * r:(i + 1) * r])
                        K.krows_tc(self.o.spec, self.tcp, slot.RAg[i], b, self.sk_pos,
                                   slot.sk_zop, sketch[i], ws=slot.sk_ws, cols=(cols[i], 0))
                    else:
                        Xb, rsq = slot.Xb[i], slot.rsq[i]
                        K.krows_times(self.o.spec, _Cols(pts, Xb, rsq), Xb, rsq, bd[i], omc[i],
                                      sketch[i], col_ids=bd[i])
            if r:
                # the three Gram matrices Y^T Y, Omega^T Y, Omega^T Omega as blocks
                # of ONE batched product [Y Omega]^T [Y Omega] (one wide GEMM
                # instead of three 100 x 100 ones)
                YO = torch.cat([sketch.to(torch.float64), om], dim=2)
                Y = YO[:, :, :r]
                G = YO.transpose(1, 2) @ YO
            ev = torch.cuda.Event()
            ev.record(fs)
        rho = np.full(count, np.nan)  # host copy not needed: the device holds rho
        tm2 = time.perf_counter()
        Ss = [None] * count
        if r:
            # the r x r factorisations, batched on the device (fast stream), the
            # eigensolves included (sap_sym_eig_batch): no host round trip;
            # failures and warnings ride on the plan flags (check_flags)
            with torch.cuda.device(self.dev), torch.cuda.stream(fs):
                xfer.mark("gram")
                W, S, rho_d, Mc, E, flags = factor_gram_batch(
                    G[:, :r, :r], G[:, r:, :r], G[:, r:, r:], r, self.lam)
                xfer.mark("factor")
                tm2 = time.perf_counter()
                torch.bmm(Y, W, out=slot.U[:count])
                slot.Mc[:count].copy_(Mc)
                torch.bmm(slot.U[:count], Mc, out=slot.UMc[:count])
                slot.E[:count, :r].copy_(E)
                slot.rho[:count].copy_(rho_d)
                slot.bad[:count] |= flags
                ev = torch.cuda.Event()
                ev.record(fs)
        else:
            ev.synchronize()  # pinned inputs consumed before the slot is refilled
            with torch.cuda.device(self.dev):
                slot.rho[:count].fill_(1.0)
        tm3 = time.perf_counter()
        with torch.cuda.device(self.dev), torch.cuda.stream(side):
            side.wait_event(ev)  # phase 1 (fast stream) done: Xb, rsq, U, Mc, E, rho
            if not (r and self.sketch_gemm):
                K.ktile_f32_batch(self.o.spec, slot.Xb[:count], slot.rsq[:count], pts.d,
                                  slot.Kbb[:count])
            inputs = torch.cuda.Event()
            inputs.record(side)
        # The power iteration is one long cluster kernel on 128 SMs: on the side
        # stream it would take the SMs a draining block-row kernel frees and hold
        # the next one back for its whole duration, so it is enqueued on the
        # solver's stream, between two block-row products.
        with torch.cuda.device(self.dev), torch.cuda.stream(self.main):
            self.main.wait_event(inputs)
            # SAP_POWER_L2=<bytes> splits the batch so each launch's K_BB blocks
            # fit that budget and stay in L2 across the 10 power steps (alone:
            # 71 us per iteration in launches of 4 against 86 us in one launch of
            # 8; inside the solver no difference beyond run-to-run noise, so
            # one launch by default)
            budget = float(os.environ.get("SAP_POWER_L2", "1e12"))
            step = max(1, min(count, int(budget // (4 * b * b))))
            for q0 in range(0, count, step):
                q1 = min(count, q0 + step)
                K.power_stepsize(slot.Kbb[q0:q1], slot.U[q0:q1] if r else None,
                                 slot.E[q0:q1], slot.rho[q0:q1], slot.v0[q0:q1], self.lam,
                                 self.iters, slot.eta[q0:q1], slot.bad[q0:q1])
            torch.div(slot.eta[:count], slot.rho[:count], out=slot.eta_rho[:count])
            xfer.mark("power")
            ready = torch.cuda.Event()
            ready.record(self.main)
            slot.h2d_done = ready  # pinned host buffers reusable after this point
            # the batch's stepsizes to the host as soon as they exist: a caller
            # that wants eta_t (adasap_step) waits for its batch's power
            # iteration, not for the block products queued after it
            slot.h_eta[:count].copy_(slot.eta[:count], non_blocking=True)
            xfer.add("d2h", count * 8)
            eta_ready = torch.cuda.Event()
            eta_ready.record(self.main)
        if self.timings is not None:
            self.timings.append(dict(count=count, rng=tm1 - tm0, gpu_wait=tm2 - tm1,
                                     factor=tm3 - tm2, total=time.perf_counter() - tm0,
                                     start=tm0, end=time.perf_counter()))
        return _Batch(slot, t0, count, blocks, crcs, rho, Ss, ready, eta_ready, owner)

    def _produce_blocks(self, slot, t0, count, side, owner):
        """A batch another rank produces: only what this rank's Phase I/IV needs
        locally (the blocks, their local rows and gathered features); the
        products arrive by broadcast in get()."""
        seed, n, b = self.seed, self.n, self.b
        if slot.h2d_done is not None:
            slot.h2d_done.synchronize()

        blocks, crcs = self._host_draws(slot, t0, count, omega=False, v0=False)
        pts = self.o.points
        fs = self.fast if self.fast is not None else side
        with torch.cuda.device(self.dev), torch.cuda.stream(fs):
            if slot.free is not None:
                fs.wait_event(slot.free)
            slot.block_dev[:count].copy_(slot.h_block[:count], non_blocking=True)
            xfer.add("h2d", count * b * 8)
            bd = slot.block_dev[:count]
            slot.loc_dev[:count].copy_(self.shard.local_positions(bd))
            for i in range(count):
                pts.gather(bd[i], out=(slot.Xb[i], slot.rsq[i]))
                if self.tcp is not None:
                    self.tcp.gather_rows(bd[i], out=slot.RAg[i])
            ready = torch.cuda.Event()
            ready.record(fs)
            slot.h2d_done = ready
        return _Batch(slot, t0, count, blocks, crcs,
                      np.full(count, np.nan), [None] * count, ready, None, owner)


class _Cols:
    """A gathered point subset viewed as a column point set."""

    def __init__(self, pts, Xs, sqn):
        self.Xs, self.sqn = Xs, sqn
        self.n, self.d, self.ldx, self.device = Xs.shape[0], pts.d, pts.ldx, pts.device
