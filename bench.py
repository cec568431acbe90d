#!/usr/bin/env python3
"""ADASAP benchmark on B200 (contract: one JSON line from rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, NCCL)

Workload (BASELINE.json configs[2], the headline): synthetic Matern-3/2 GP,
n = 10^6, d = 9, b = 2000, m = 65 RHS (mean + 64 pathwise samples),
Nystrom rank r = 100, lam = 1e-2, residual_every = 0. A "step" is one full
ADASAP iteration (Phases I-IV, solvers.py:361-403). ``value`` is solver
iterations per second for the whole job (strong scaling: the n points are
sharded over the N GPUs, one NCCL all-reduce of the b x m gradient per
iteration). The per-iteration working set (X 48 MB + lazy state P, Q
520 MB) exceeds the 126 MB L2, so no explicit flush is needed between steps.

``roofline`` describes the dominant kernel (the fused block-row product
K[B,:]Z on the tensor cores, sap_krows_tc): algorithmic flops per launch =
b * n_local * 2 (d + m), timed with CUDA events on its
stream, against the measured bf16 peak / 3 (three
split-precision passes per algorithmic flop); ``traffic`` is the DRAM bytes of
one launch from the committed ncu capture. ``e2e`` runs reference-style code
(SolverState.zeros + adasap_step) from host arrays with setup and the final
readback inside the timed region, bytes counted at each copy.
``cpu_baseline`` is the CPU oracle port (oracle/sapgp_oracle.py, a numpy
restatement of the reference) timed on this host's cores for one iteration.
``--impl reference`` times that same CPU implementation as the reference arm.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# the CPU oracle runs one BLAS thread per worker (reference conftest / __init__ policy)
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

CONFIG = dict(n=1_000_000, d=9, family="matern32", b=2000, m=65, r=100, lam=1e-2, seed=0)
METRIC = "ADASAP iters/s & kernel-entries/s at n=1M,1/2/4/8 B200; time-to-target RMSE"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=40)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--family", default=CONFIG["family"])
    ap.add_argument("--n", type=int, default=CONFIG["n"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def workload(args):
    return {"workload": f"synthetic {args.family} GP n={args.n} d={CONFIG['d']} b={CONFIG['b']} "
                        f"m={CONFIG['m']} r={CONFIG['r']} (BASELINE.json configs[2])",
            "n": args.n, "d": CONFIG["d"], "family": args.family, "blocksize": CONFIG["b"],
            "rhs": CONFIG["m"], "nystrom_rank": CONFIG["r"], "lam": CONFIG["lam"],
            "residual_every": 0, "parallelism": f"n-sharded x{args.gpus}",
            "l2": "working set > L2 (no flush needed)"}


# ---------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and the reference arm)


def oracle_problem(args):
    from oracle import sapgp_oracle as orc
    from paper_2505_13723_b200 import synthetic
    import numpy as np
    X = synthetic.make_inputs(args.n, CONFIG["d"], CONFIG["seed"])
    ls = np.full(CONFIG["d"], math.sqrt(CONFIG["d"]))
    pts = orc.Points(args.family, ls, 1.0, X)
    rng = np.random.default_rng(1)
    Y = rng.standard_normal((args.n, CONFIG["m"]))
    return orc, pts, Y


def time_oracle_steps(args, steps, warmup, budget_s=240.0):
    """Times oracle ADASAP iterations (all host cores, BLAS pinned per worker)."""
    import numpy as np
    orc, pts, Y = oracle_problem(args)
    cores = host_cores()
    b, r, lam = CONFIG["b"], CONFIG["r"], CONFIG["lam"]
    co = orc.accel_coeffs(lam, args.n, b)
    rng = np.random.default_rng(2)
    W = np.zeros_like(Y)
    V, Z = W.copy(), 0.01 * rng.standard_normal(Y.shape)
    t = 0
    for _ in range(warmup):
        W, V, Z, _, _ = orc.adasap_step(pts, lam, Y, W, V, Z, t, CONFIG["seed"], b, r, co, cores)
        t += 1
    times = []
    t_start = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        W, V, Z, _, _ = orc.adasap_step(pts, lam, Y, W, V, Z, t, CONFIG["seed"], b, r, co, cores)
        times.append(time.perf_counter() - t0)
        t += 1
        if time.perf_counter() - t_start > budget_s:
            break
    return len(times) / sum(times), cores, len(times)


# ---------------------------------------------------------------------------
# clocks


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.path = tempfile.mktemp(suffix=".csv")
        self.index = index
        self.proc = None

    def start(self, settle_s=1.5):
        """Start sampling and wait until nvidia-smi has settled (NVML start-up
        contends with CUDA driver calls, so it must not overlap the timed
        region's first launches); it keeps sampling through the region."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms",
                 os.environ.get("SAP_BENCH_CLOCK_MS", "200")],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        t_end = time.time() + 5.0
        while time.time() < t_end:
            time.sleep(0.05)
            if os.path.exists(self.path) and os.path.getsize(self.path) > 0:
                break
        time.sleep(max(0.0, settle_s - 0.0))

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# B200 arm


def b_pad_rows(b):
    return (b + 255) // 256 * 256  # block rows the CTA-pair kernel computes


# The lookahead produces plans in batches that ramp 1, 4, 16, then full
# batches from iteration 21 (pipeline.Lookahead); the first iterations are
# not steady state, so 64 count as warm-up whatever --warmup asks for.
RAMP_ITERS = 64


def measured_traffic(family):
    """dram__bytes_read.sum + dram__bytes_write.sum of one block-row launch at
    this config, from the committed ncu capture (profiles/r02_krows_traffic.json,
    written by scripts/ncu_traffic.py from an `ncu --set full` report of this
    bench); None if that capture is absent."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_krows_traffic.json")))
    except (OSError, ValueError):
        return None
    return d.get(family)


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as tdist

    import paper_2505_13723_b200 as sap
    from paper_2505_13723_b200 import _native as nat
    from paper_2505_13723_b200 import synthetic
    from paper_2505_13723_b200.parallel import init_from_env
    from paper_2505_13723_b200.solvers import AdasapEngine

    dist = init_from_env("nccl")
    rank = tdist.get_rank() if dist else 0
    world = tdist.get_world_size() if dist else 1
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = nat.load()

    prob = synthetic.make_problem(args.n, CONFIG["d"], args.family, CONFIG["m"],
                                  seed=CONFIG["seed"], lam=CONFIG["lam"], device=dev)
    spec = prob.spec()
    oracle = sap.KernelOracle(spec, prob.X, prob.lam, device=dev)
    # Python's full (generation-2) collections scan every tracked object --
    # ~180k after importing torch, ~37 ms per collection -- holding the GIL, so
    # the lookahead's producers stall at random steps (e2e runs of 0.1-0.5 s
    # instead of ~0.09 s). Objects alive now (modules, the problem) are frozen
    # out of those scans, as a long-running service would do after start-up
    # (scripts/e2e_phases.py GC=on/off/freeze/check).
    gc.freeze()
    warm = max(args.warmup, RAMP_ITERS)
    cfg = sap.RunConfig(lam=prob.lam, blocksize=CONFIG["b"], nystrom_rank=CONFIG["r"],
                        residual_every=0, seed=CONFIG["seed"])
    accel = sap.resolve_accel(cfg, args.n, CONFIG["b"])
    # unbounded: the lookahead keeps producing at its steady rate through the
    # timed window, as inside a long solve
    eng = AdasapEngine(oracle, prob.Y, cfg, accel, unbounded=True)
    shard = eng.shard
    n_local = shard.size
    b, m, d = CONFIG["b"], CONFIG["m"], CONFIG["d"]

    sampler = ClockSampler(local)
    if os.environ.get("SAP_BENCH_NO_CLOCKS") != "1":  # diagnosis only
        sampler.start()
    for _ in range(warm):
        eng.step()
    torch.cuda.synchronize()

    # kernel-level events around the dominant launch (same stream as the launch)
    import paper_2505_13723_b200.solvers as S
    evs = []
    originals = {name: getattr(S, name) for name in ("krows_times", "krows_tc", "krows_tc_partials")}

    def timed(fn):
        def wrapper(*a, **kw):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            out = fn(*a, **kw)
            e.record()
            evs.append((s, e))
            return out
        return wrapper

    for name, fn in originals.items():
        setattr(S, name, timed(fn))
    launches0 = lib.sap_launch_count()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        eng.step()
    t1.record()
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    launches = lib.sap_launch_count() - launches0
    clocks = sampler.stop()
    for name, fn in originals.items():
        setattr(S, name, fn)
    ms = t0.elapsed_time(t1)
    kms = [s.elapsed_time(e) for s, e in evs]
    kmean = sum(kms) / len(kms)
    if dist:
        tt = torch.tensor([ms, kmean], device=dev, dtype=torch.float64)
        tdist.all_reduce(tt, op=tdist.ReduceOp.MAX)
        ms, kmean = float(tt[0]), float(tt[1])
    eng.close()

    ms_step = ms / args.steps
    iters_s = 1000.0 / ms_step
    entries = b * args.n
    flops_launch = b * n_local * 2 * (d + m)
    achieved = flops_launch / (kmean * 1e-3) / 1e12
    kernel_name = ("sap_krows_tc (tcgen05 + TMEM + TMA, 3-pass split precision)" if eng.use_tc
                   else "sap_krows_times (FFMA path)")

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    bf16_peak = float(peaks.get("bf16_tflops", 1590.0))
    # the split-precision tensor-core path's peak is the
    # measured dense tensor peak over the passes one algorithmic flop costs
    # (3 fp16 hi/lo products, P_hi Z_hi + P_hi Z_lo + P_lo Z_hi)
    peak = bf16_peak / 3.0 if eng.use_tc else None
    tensor_pipe = None
    if eng.use_tc:
        ka, nz, half = eng.tcp.ka, eng.zop.nz, eng.tcp.half
        g1_rate = bf16_peak if half else 0.5 * bf16_peak  # f16 features, else tf32 (half rate)
        t_entry = 2 * ka / (g1_rate * 1e12) + 3 * 2 * nz / (bf16_peak * 1e12)
        ideal_ms = b * n_local * t_entry * 1e3
        g1 = "f16" if half else "tf32"
        tensor_pipe = {"hw_flop_per_entry": {"gemm1_" + g1: 2 * ka, "gemm2_f16": 6 * nz},
                       "ideal_ms_at_peak": ideal_ms, "frac": ideal_ms / kmean,
                       "note": "time the tensor pipe needs for GEMM1 (%s, ka=%d) + GEMM2 (3 "
                               "fp16 passes, nz=%d) at the measured bf16 peak over the "
                               "measured kernel time" % (g1, ka, nz)}
        # the epilogue's special-function bound: ex2 (RBF) or rsqrt + ex2 (Matern) per
        # kernel entry on the MUFU pipe (16 lanes/clk/SM for every MUFU op, scripts/micro/mufu.cu)
        mufu_ops = 1 if args.family == "rbf" else 2
        mufu_ms = b_pad_rows(b) * n_local * mufu_ops / (16 * 148 * 1.965e9) * 1e3
        tensor_pipe["mufu_bound_ms"] = mufu_ms
        tensor_pipe["mufu_frac"] = mufu_ms / kmean
    traffic = measured_traffic(args.family) if eng.use_tc and args.n == CONFIG["n"] else None

    e2e = None
    if not args.no_e2e and world == 1:
        e2e = run_e2e(args, prob, spec, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, nst = time_oracle_steps(args, steps=1, warmup=0)
        cpu = {"value": v, "unit": "iters/s", "cores": cores, "kind": "port",
               "sample": f"{nst} full ADASAP iteration(s) of the oracle port "
                         f"(oracle/sapgp_oracle.py) at the same n/d/b/m/r, {cores} worker "
                         f"threads, BLAS pinned to 1 thread per worker"}

    line = {
        "metric": METRIC, "value": iters_s, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (SURVEY.md §8d generator, pathwise RHS)",
        "config": workload(args),
        "warmup_effective": warm,
        "warmup_note": f"the lookahead's batch ramp (first {RAMP_ITERS} iterations) counts as "
                       "warm-up; the engine is unbounded so plan production continues at its "
                       "steady rate through the timed window",
        "kernel_entries_per_s": entries / (ms_step * 1e-3),
        "krows_ms": kmean,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                     "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_source": traffic["source"] if traffic else None,
                     "kernel": kernel_name,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (dense, burst) / 3 "
                                    "(SURVEY.md §8d: 3 split-precision passes)",
                     "algorithmic": f"{b}*{n_local}*2*({d}+{m}) flop per launch "
                                    "(2d+2m per kernel entry, BASELINE.md §2)",
                     "tensor_pipe": tensor_pipe},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        tdist.destroy_process_group()


E2E_RUNS = 5


def run_e2e(args, prob, spec, dev):
    """The same metric through the public drop-in API from HOST arrays, the way
    reference code runs it (tests/test_solvers.py:199-219): KernelOracle(X
    host), SolverState.zeros, K x adasap_step(oracle, state, Y host, config,
    accel) -- each step reads its stepsize back to the host -- and the final W
    to the host (state.W). Timed region: setup + K steps + W readback. Bytes
    are counted at every copy site (paper_2505_13723_b200/xfer.py). Two
    untimed warm-up runs first (process-level init: kernel modules, allocator
    pools), then E2E_RUNS timed runs, the median reported. ``solve`` adds
    the full adasap_solve of K iterations (its final relative residual, a K W
    product over all n^2 entries, included)."""
    import numpy as np
    import torch
    import paper_2505_13723_b200 as sap
    from paper_2505_13723_b200 import xfer
    from paper_2505_13723_b200.solvers import SolverState, adasap_step
    K = args.steps
    X, Y = np.ascontiguousarray(prob.X), np.ascontiguousarray(prob.Y)
    n, m = Y.shape
    cfg = sap.RunConfig(lam=prob.lam, blocksize=CONFIG["b"], nystrom_rank=CONFIG["r"],
                        residual_every=0, seed=CONFIG["seed"], max_iters=K)

    def step_run(k):
        o = sap.KernelOracle(spec, X, prob.lam, device=dev)
        accel = sap.resolve_accel(cfg, o.n, CONFIG["b"])
        state = SolverState.zeros(n, m, accelerated=True)
        etas = []
        for _ in range(k):
            state, eta, _ = adasap_step(o, state, Y, cfg, accel)
            etas.append(eta)
        W = state.W
        return W, etas, state

    for _ in range(2):  # untimed warm-up runs (process-level init: modules, handles, pools)
        _, _, st = step_run(max(2, args.warmup))
        st.iteration = st.iteration  # detach: releases the engine
    # E2E_RUNS timed runs, the median reported: a run occasionally stalls for
    # 0.1-0.5 s on the host (seen in every phase on some boxes, GPU idle;
    # scripts/e2e_phases.py), which one run would report as the throughput
    runs, finite = [], True
    gc_log = []
    if xfer.TRACE is not None:  # SAP_TRACE=1 (diagnosis): garbage collections during the runs
        gc.callbacks.append(lambda phase, info: gc_log.append(
            (time.perf_counter(), phase, info.get("generation"))))
    for _ in range(E2E_RUNS):
        torch.cuda.synchronize()
        if xfer.TRACE is not None:
            m0 = torch.cuda.memory_stats()
        x0 = xfer.snapshot()
        t0 = time.perf_counter()
        W, etas, st = step_run(K)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        x1 = xfer.snapshot()
        st._e.close()  # after the timed region: the lookahead's producers run ahead
        st.iteration = st.iteration  # detach: releases the engine
        runs.append(t1 - t0)
        if xfer.TRACE is not None:  # SAP_TRACE=1 (diagnosis): the run's marks, gaps > 10 ms
            last = t0
            for tt, th, tag in xfer.TRACE:
                if t0 <= tt <= t1 and tt - last > 0.01:
                    print(f"# e2e run {len(runs)} ({1e3 * (t1 - t0):.0f} ms): "
                          f"{1e3 * (tt - t0):7.1f} ms {th} {tag} after a {1e3 * (tt - last):.0f} ms gap",
                          file=sys.stderr)
                last = max(last, tt)
            xfer.TRACE.clear()
            starts = {}
            for tt, phase, gen in gc_log:
                if phase == "start":
                    starts[gen] = tt
                elif gen in starts and t0 <= tt <= t1 and tt - starts[gen] > 0.002:
                    print(f"# e2e run {len(runs)}: gc generation {gen} at "
                          f"{1e3 * (starts[gen] - t0):.1f} ms took {1e3 * (tt - starts[gen]):.1f} ms",
                          file=sys.stderr)
            gc_log.clear()
            m1 = torch.cuda.memory_stats()
            print(f"# e2e run {len(runs)}: cudaMalloc {m1.get('num_device_alloc', 0) - m0.get('num_device_alloc', 0)}"
                  f", cudaFree {m1.get('num_device_free', 0) - m0.get('num_device_free', 0)}, "
                  f"alloc retries {m1.get('num_alloc_retries', 0) - m0.get('num_alloc_retries', 0)}",
                  file=sys.stderr)
        finite = finite and bool(np.isfinite(W).all() and np.isfinite(etas).all())
        del W
    h2d, d2h = x1["h2d"] - x0["h2d"], x1["d2h"] - x0["d2h"]
    med = float(np.median(runs))
    # the full solve (final residual included), for the record
    t2 = time.perf_counter()
    o = sap.KernelOracle(spec, X, prob.lam, device=dev)
    res = sap.adasap_solve(o, Y, cfg)
    t3 = time.perf_counter()
    return {"value": K / med, "unit": "iters/s",
            "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K,
            "h2d_bytes_total": h2d, "d2h_bytes_total": d2h,
            "region": f"KernelOracle(X host) + SolverState.zeros + {K} x adasap_step(Y host), "
                      "each step's stepsize read to the host, + state.W (final iterate to "
                      "host float64); setup and readback inside the timed region",
            "seconds": med, "runs_seconds": [round(r, 4) for r in runs],
            "statistic": f"median of {E2E_RUNS} timed runs (gc.freeze() after setup)",
            "solve": {"iters_per_s": K / (t3 - t2), "seconds": t3 - t2,
                      "final_residual": res.trace.final_residual(),
                      "note": f"adasap_solve(max_iters={K}) from host X/Y to host W, including "
                              "its final relative residual (an n x n x m product)"},
            "finite": finite}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    v, cores, nst = time_oracle_steps(args, steps=args.steps, warmup=min(args.warmup, 1))
    line = {
        "metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": args.gpus, "steps": nst,
        "warmup": min(args.warmup, 1), "ms_per_step": 1000.0 / v, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload(args), "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": cores, "kind": "port",
                         "sample": f"{nst} timed ADASAP iterations of the oracle port on "
                                   f"{cores} host threads (time-capped at 240 s)"},
        "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        os.environ.setdefault("OMP_NUM_THREADS", "1")
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
