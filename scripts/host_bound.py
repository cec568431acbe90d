"""Is the ADASAP iteration host-bound? Times the main thread's enqueue per step
(eng.step() wall time) against the device time per step, plus the lookahead
producers' per-batch phases (SAP_PROFILE=1 timings), at config 3.

    python scripts/host_bound.py [--family rbf] [--steps 120]
"""
import argparse, os, sys, time
os.environ.setdefault("SAP_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="matern32")
ap.add_argument("--steps", type=int, default=120)
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=9)
ap.add_argument("--b", type=int, default=2000)
ap.add_argument("--L", type=int, default=32)
a = ap.parse_args()
n, d, b, m, r = a.n, a.d, a.b, 65, 100
prob = synthetic.make_problem(n, d, a.family, m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0,
                    max_iters=a.steps + 20, lookahead=a.L)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=a.steps + 20)
for _ in range(20):
    eng.step()
torch.cuda.synchronize()
host = []
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
t0 = time.perf_counter()
bnd = []
for _ in range(a.steps):
    k0 = eng.la.k
    h0 = time.perf_counter()
    eng.step()
    host.append(time.perf_counter() - h0)
    bnd.append(eng.la.k != k0)
t1 = time.perf_counter()
e.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
dev_ms = s.elapsed_time(e) / a.steps
host = np.array(host) * 1e3
print(f"device ms/step {dev_ms:.3f}  host enqueue ms/step mean {host.mean():.3f} "
      f"median {np.median(host):.3f} p90 {np.percentile(host, 90):.3f} max {host.max():.3f}; "
      f"enqueue loop {1e3 * (t1 - t0) / a.steps:.3f} ms/step, drain after loop {1e3 * (t2 - t1):.1f} ms")
bnd = np.array(bnd)
print(f"  batch-boundary steps {bnd.sum()} (L={eng.la.L}): host ms mean {host[bnd].mean():.3f}, "
      f"sum {host[bnd].sum():.1f}; other steps mean {host[~bnd].mean():.3f} "
      f"median {np.median(host[~bnd]):.3f} p90 {np.percentile(host[~bnd], 90):.3f}")
tm = eng.la.timings or []
if tm:
    for k in ("rng", "gpu_wait", "factor", "total"):
        v = [x[k] / x["count"] * 1e3 for x in tm[2:]]
        print(f"  producer {k:8s} per iteration: mean {np.mean(v):.3f} ms")
eng.close()
