"""Measure SURVEY.md §8(f)'s rows at config-3 scale on one B200 (n=1e6, d=9,
m=65, Matern-3/2 unless --family): the products and solvers around the
ADASAP hot path, each on the same tensor-core kernel.

    python scripts/scale_bench.py [--family rbf] [--n 1000000] > profiles/...json

Prints one JSON object:
  sdd            block SDD (solvers.py:463-516): iterations/s, and the fused
                 momentum/averaging pass against the HBM roofline
  full_product   K @ P with every point a row (PCG's operator, the residual
                 solvers.py:254-257): ms, kernel entries/s
  cross_product  k(X*, X) W for 10^4 test points (PosteriorMean, gp.py:151-159)
  prior_rhs      phi(X) theta for the pathwise right-hand sides (gp.py:99-114)
All times are CUDA-event times on the launching stream after warm-up.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_13723_b200 as sap  # noqa: E402
from paper_2505_13723_b200 import synthetic  # noqa: E402
from paper_2505_13723_b200 import _native as nat  # noqa: E402
from paper_2505_13723_b200.baselines import SddEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="matern32")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--sdd-steps", type=int, default=40)
a = ap.parse_args()
n, d, b, m = a.n, 9, 2000, 65
dev = torch.device("cuda", 0)
peaks = {}
try:
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
except (OSError, ValueError):
    pass
hbm = float(peaks.get("hbm_gbs", 6547.8))


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e))
    return min(out)


res = {"workload": f"synthetic {a.family} GP n={n} d={d} m={m}", "gpu": torch.cuda.get_device_name(0)}
t0 = time.perf_counter()
prob = synthetic.make_problem(n, d, a.family, m, seed=0, lam=1e-2, device=dev)
res["prior_rhs"] = {"make_problem_seconds_host_timed": time.perf_counter() - t0,
                    "what": "make_problem: phi(X) theta for n + 10^4 points, q=2048 cosine "
                            "features, 65 columns (fused tensor-core product), zeta (n x 64) drawn "
                            "on the GPU, host numpy X and noise; first CUDA use in the process"}
from paper_2505_13723_b200.kernels import cos_features_times  # noqa: E402
from paper_2505_13723_b200.synthetic import feature_map  # noqa: E402
from paper_2505_13723_b200.rng import substream  # noqa: E402
_fr, _ph = feature_map(a.family, np.full(d, np.sqrt(d)), 2048, substream(0, "features"))
_th = np.random.default_rng(1).standard_normal((2048, m))
_Xd = torch.as_tensor(prob.X, device=dev)
res["prior_rhs"]["fused_product_ms"] = timed(
    lambda: cos_features_times(_fr, _ph, 1.0, _Xd, _th, dev), reps=3)
res["prior_rhs"]["entries_per_s"] = n * 2048 / (res["prior_rhs"]["fused_product_ms"] * 1e-3)
spec = prob.spec()
o = sap.KernelOracle(spec, prob.X, prob.lam, device=dev)

# -- SDD ---------------------------------------------------------------------
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, solver_id="sdd", max_iters=a.sdd_steps + 5,
                    residual_every=0, seed=0)
eng = SddEngine(o, prob.Y, cfg, a.sdd_steps + 5)
for _ in range(5):
    eng.step()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.sdd_steps):
    eng.step()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / a.sdd_steps
loc = torch.full((b,), -1, dtype=torch.int64, device=dev)


def dense_pass():
    nat.call("sap_sdd_update", nat.ptr(eng.V), nat.ptr(eng.W), nat.ptr(eng.E), eng.ld, eng.ld, m,
             nat.ptr(loc), 0, nat.ptr(eng.g), eng.g.stride(0), eng.eta, 0.9, eng.avg,
             nat.ptr(eng.VB), nat.ptr(eng.pos), nat.stream_handle())


dms = timed(dense_pass, reps=5)
nbytes = 6 * 4 * m * eng.ld + 4 * eng.ld  # read V W E pos, write V W E
res["sdd"] = {"iters_per_s": 1000.0 / ms, "ms_per_iter": ms, "blocksize": b,
              "dense_pass_ms": dms, "dense_pass_gbs": nbytes / dms * 1e-6,
              "dense_pass_frac_hbm": nbytes / dms * 1e-6 / hbm,
              "dense_pass_bytes": nbytes}
eng.close()

# -- full product (PCG operator / residual) ----------------------------------
ids = torch.arange(n, device=dev, dtype=torch.int64)
P = torch.randn((m, n), device=dev, dtype=torch.float32)
out = torch.empty((n, m), device=dev, dtype=torch.float32)
fms = timed(lambda: o.rows_times_device(ids, P, out=out), reps=2)
res["full_product"] = {"ms": fms, "entries_per_s": n * n / (fms * 1e-3),
                       "tflops_algorithmic": n * n * 2 * (d + m) / (fms * 1e-3) / 1e12}

# -- cross product (posterior mean / samples at the test points) ---------------
Xs = prob.Xtest
W = np.random.default_rng(0).standard_normal((n, m))
Wd = torch.as_tensor(W, device=dev, dtype=torch.float32)
cms = timed(lambda: o.cross_matmul(Xs, Wd), reps=3)
t = Xs.shape[0]
res["cross_product"] = {"test_points": t, "ms_incl_feature_prep": cms,
                        "entries_per_s": t * n / (cms * 1e-3)}
print(json.dumps(res))
