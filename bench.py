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
K[B,:]Z, sap_krows_times): algorithmic flops per launch = b * n_local *
2 (d + m), timed with CUDA events on its stream.
``cpu_baseline`` is the CPU oracle port (oracle/sapgp_oracle.py, a numpy
restatement of the reference) timed on this host's cores for one iteration.
``--impl reference`` times that same CPU implementation as the reference arm.
"""

from __future__ import annotations

import argparse
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

# dram__bytes_read.sum + dram__bytes_write.sum of one sap_krows_tc launch at this
# config, from the committed ncu capture (profiles/); re-capture when the kernel changes.
# dram__bytes_read.sum + dram__bytes_write.sum of one sap_krows_tc launch at config 3
# (profiles/r01e_krows_tc2_*_ncu_summary.txt, ncu --set full)
TRAFFIC_PER_LAUNCH = {"matern32": 416_395_008 + 21_179_392, "rbf": 416_449_280 + 19_812_352}

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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as tdist

    import paper_2505_13723_b200 as sap
    from paper_2505_13723_b200 import _native as nat
    from paper_2505_13723_b200 import synthetic
    from paper_2505_13723_b200.parallel import current_shard, init_from_env
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
    total = args.warmup + args.steps
    cfg = sap.RunConfig(lam=prob.lam, blocksize=CONFIG["b"], nystrom_rank=CONFIG["r"],
                        residual_every=0, seed=CONFIG["seed"], max_iters=total)
    accel = sap.resolve_accel(cfg, args.n, CONFIG["b"])
    eng = AdasapEngine(oracle, prob.Y, cfg, accel, total=total + 8)
    shard = eng.shard
    n_local = shard.size
    b, m, d = CONFIG["b"], CONFIG["m"], CONFIG["d"]

    sampler = ClockSampler(local)
    if os.environ.get("SAP_BENCH_NO_CLOCKS") != "1":  # diagnosis only
        sampler.start()
    for _ in range(args.warmup):
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
    kernel_name = ("sap_krows_tc (tcgen05 + TMEM + TMA, split-precision)" if eng.use_tc
                   else "sap_krows_times (FFMA path)")

    # FP32 FFMA peak of this GPU (the FFMA path's denominator)
    buf = torch.zeros(256, device=dev)
    iters = 1 << 16
    nat.call("sap_ffma_peak", nat.ptr(buf), iters, nat.stream_handle())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nat.call("sap_ffma_peak", nat.ptr(buf), iters, nat.stream_handle())
    e1.record()
    torch.cuda.synchronize()
    ffma_peak = 148 * 4 * 256 * 8 * iters * 2 / (e0.elapsed_time(e1) * 1e-3) / 1e12
    lib_launches_after = lib.sap_launch_count()

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass

    bf16_peak = float(peaks.get("bf16_tflops", 1590.0))
    # What the tensor pipe must execute per kernel entry in this formulation
    # (DESIGN.md §5): GEMM1 kind::tf32 over the ka augmented features, GEMM2
    # kind::f16 three split passes over nz padded right-hand sides. tf32 dense
    # peak taken as half the measured bf16 peak (no tf32 figure is measured).
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
                               "fp16 passes, nz=%d) at the measured bf16 peak (tf32 = half) "
                               "over the measured kernel time" % (g1, ka, nz)}
        # the epilogue's special-function bound: ex2 (RBF) or rsqrt + ex2 (Matern) per
        # kernel entry on the MUFU pipe (16 lanes/clk/SM, scripts/micro/pipes.cu)
        mufu_ops = 1 if args.family == "rbf" else 2
        mufu_ms = b_pad_rows(b) * n_local * mufu_ops / (16 * 148 * 1.965e9) * 1e3
        tensor_pipe["mufu_bound_ms"] = mufu_ms
        tensor_pipe["mufu_frac"] = mufu_ms / kmean
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
        "kernel_entries_per_s": entries / (ms_step * 1e-3),
        "krows_ms": kmean,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": bf16_peak,
                     "unit": "TFLOP/s", "frac": achieved / bf16_peak,
                     "traffic": TRAFFIC_PER_LAUNCH.get(args.family) if eng.use_tc else None,
                     "kernel": kernel_name,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops (dense, burst), of measured",
                     "algorithmic": f"{b}*{n_local}*2*({d}+{m}) flop per launch "
                                    "(2d+2m per kernel entry, BASELINE.md §2)",
                     "fp32_ffma_peak": ffma_peak,
                     "frac_of_fp32_ffma_roofline": achieved / ffma_peak,
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


def run_e2e(args, prob, spec, dev):
    """Same metric through the public API from host numpy arrays: KernelOracle(X
    host) + make_state(Y host) (setup, timed separately), W untimed warm-up
    steps, then K timed ``adasap_step`` calls -- each one generates the step's
    block indices, Gaussian sketch and power-iteration start on the host
    (numpy RNG, bit-exact with the reference), copies them host->device from
    pinned buffers and reads the step's stepsize back to the host -- and the
    final W to host (timed separately). ``value`` is K / (timed step loop);
    ``solve_iters_per_s`` also charges setup and the W readback to the K steps."""
    import numpy as np
    import torch
    import paper_2505_13723_b200 as sap
    K, Wu = args.steps, args.warmup
    X, Y = np.ascontiguousarray(prob.X), np.ascontiguousarray(prob.Y)
    cfg = sap.RunConfig(lam=prob.lam, blocksize=CONFIG["b"], nystrom_rank=CONFIG["r"],
                        residual_every=0, seed=CONFIG["seed"], max_iters=K + Wu)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o = sap.KernelOracle(spec, X, prob.lam, device=dev)
    accel = sap.resolve_accel(cfg, o.n, CONFIG["b"])
    state = sap.make_state(o, Y, cfg, accel)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    for _ in range(Wu):
        state, eta, block = sap.adasap_step(o, state, Y, cfg, accel)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    etas = []
    for _ in range(K):
        state, eta, block = sap.adasap_step(o, state, Y, cfg, accel)
        etas.append(eta)  # a host float: the per-step device->host read
    torch.cuda.synchronize()  # every step's device work is inside the timed region
    t2 = time.perf_counter()
    W = state.W
    t3 = time.perf_counter()
    state._e.close()
    b, r, m = CONFIG["b"], CONFIG["r"], CONFIG["m"]
    # pinned host->device per step: block ids, the omega stream's PCG64 state (the
    # sketch Omega is drawn on the GPU), power start, W and Woodbury factors,
    # coefficients, rho; device->host: 3 r x r Gram blocks + eta
    per_iter_h2d = b * 8 + 4 * 8 + b * 8 + 2 * r * r * 8 + 2 * r * 8 + 8
    per_iter_d2h = 3 * r * r * 8 + 8
    return {"value": K / (t2 - t1), "unit": "iters/s",
            "h2d_bytes_per_step": int(per_iter_h2d), "d2h_bytes_per_step": int(per_iter_d2h),
            "region": f"{K} x adasap_step through the public API after {Wu} warm-up steps "
                      "(host RNG seeding + block draw, pinned H2D of the step inputs, the step's "
                      "stepsize read to the host each step) and a final device synchronize; "
                      "setup (X, Y host->device) and the final W readback are timed separately",
            "seconds": t2 - t1, "setup_s": t_setup, "w_readback_s": t3 - t2,
            "solve_iters_per_s": K / (t_setup + (t2 - t1) + (t3 - t2)),
            "finite": bool(np.isfinite(W).all() and np.isfinite(etas).all())}


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
