"""ADASAP throughput at the other BASELINE.json configs on ONE B200:

  config 2  houseelec-shaped RBF, n=1e5, d=11, b=1000, m=65 (fp32 features, ka=64)
  config 4  RBF n=1e7, d=9, b=5000, m=65 (the 8-GPU config; here one GPU)
  config 5  taxi-shaped RBF n=1e8, d=9, b=10000, m=65 (the 8-GPU config sized for
            180 GB of HBM per GPU; here ALL of it on one GPU)

Throughput-only runs (SURVEY.md §8d allows noise RHS at n >= 1e7): X ~ N(0,1)
and Y ~ N(0,1) drawn on the device with torch's generator (seeded), not the
numpy synthetic generator, so the data are synthetic but not the reference's.
Prints one JSON object per config: iterations/s (device events), kernel
entries/s, the block product's share, and device memory in use.

    python scripts/scale_configs.py [2 4 5]
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_13723_b200 as sap  # noqa: E402
import paper_2505_13723_b200.solvers as S  # noqa: E402
from paper_2505_13723_b200.solvers import AdasapEngine  # noqa: E402

CONFIGS = {2: dict(n=100_000, d=11, b=1000, warm=200, steps=2000),
           4: dict(n=10_000_000, d=9, b=5000, warm=70, steps=40),
           5: dict(n=100_000_000, d=9, b=10000, warm=8, steps=8)}
m, r, lam = 65, 100, 1e-2
dev = torch.device("cuda", 0)


def run(cfg_id):
    c = CONFIGS[cfg_id]
    n, d, b = c["n"], c["d"], c["b"]
    g = torch.Generator(device=dev).manual_seed(cfg_id)
    X = torch.randn((n, d), generator=g, device=dev, dtype=torch.float64)
    Y = torch.randn((n, m), generator=g, device=dev, dtype=torch.float32)
    spec = sap.KernelSpec("rbf", np.full(d, math.sqrt(d)), 1.0)
    o = sap.KernelOracle(spec, X, lam, device=dev)
    del X
    cfg = sap.RunConfig(lam=lam, blocksize=b, nystrom_rank=r, residual_every=0, seed=0)
    # unbounded: plans keep being produced at the steady rate through the window
    eng = AdasapEngine(o, Y, cfg, sap.resolve_accel(cfg, n, b), unbounded=True)
    del Y
    for _ in range(c["warm"]):
        eng.step()
    torch.cuda.synchronize()
    evs = []
    origs = {k: getattr(S, k) for k in ("krows_tc", "krows_tc_partials")}

    def timed(fn):
        def w(*a, **kw):
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            out = fn(*a, **kw)
            e_.record()
            evs.append((s_, e_))
            return out
        return w

    for k, fn in origs.items():
        setattr(S, k, timed(fn))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(c["steps"]):
        eng.step()
    e.record()
    torch.cuda.synchronize()
    for k, fn in origs.items():
        setattr(S, k, fn)
    eng.la.check_flags()
    ms = s.elapsed_time(e) / c["steps"]
    kms = float(np.mean([a.elapsed_time(z) for a, z in evs]))
    free, totalmem = torch.cuda.mem_get_info()
    out = {"config": cfg_id, "workload": f"synthetic RBF GP n={n} d={d} b={b} m={m} r={r}",
           "data": "synthetic on-device N(0,1) inputs and noise RHS (throughput run)",
           "features": "fp16" if eng.tcp.half else "fp32", "iters_per_s": 1000.0 / ms,
           "ms_per_iter": ms, "krows_ms": kms, "krows_share": kms / ms,
           "kernel_entries_per_s": b * n / (ms * 1e-3),
           "krows_tflops_algorithmic": b * n * 2 * (d + m) / (kms * 1e-3) / 1e12,
           "device_mem_used_gb": (totalmem - free) / 1e9, "device_mem_total_gb": totalmem / 1e9,
           "next_operand_overlapped": eng.zop_next is not None,
           "passes_per_s": b / n * 1000.0 / ms}
    eng.close()
    del eng, o
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    ids = [int(a) for a in sys.argv[1:]] or [2, 4, 5]
    for i in ids:
        try:
            print(json.dumps(run(i)), flush=True)
        except torch.cuda.OutOfMemoryError as exc:  # report, then try a smaller n
            print(json.dumps({"config": i, "oom": str(exc)[:200]}), flush=True)
            torch.cuda.empty_cache()
            if i == 5:
                CONFIGS[5]["n"] = 60_000_000
                print(json.dumps(run(5)), flush=True)
