"""Steady-state ADASAP iterations bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists (config 3 unless overridden)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine
ap = argparse.ArgumentParser()
ap.add_argument("--family", default="matern32")
ap.add_argument("--iters", type=int, default=8)
ap.add_argument("--warm", type=int, default=16)
ap.add_argument("--total", type=int, default=64)
a = ap.parse_args()
n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, a.family, m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=a.total)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=a.total)
for _ in range(a.warm): eng.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.iters): eng.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
eng.close()
print("ok")
