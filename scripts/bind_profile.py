"""Cost of binding a fresh engine (the step API's first call): engine
construction pieces and the first plan."""
import os, sys, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine
n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, "matern32", m, seed=0, lam=1e-2, device="cuda")
X, Y = np.ascontiguousarray(prob.X), np.ascontiguousarray(prob.Y)
cfg = sap.RunConfig(lam=1e-2, blocksize=b, nystrom_rank=r, residual_every=0, seed=0)
o = sap.KernelOracle(prob.spec(), X, 1e-2, device="cuda")
accel = sap.resolve_accel(cfg, n, b)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr = cProfile.Profile() if rep == 2 else None
    if pr: pr.enable()
    e = AdasapEngine(o, Y, cfg, accel, unbounded=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    e.step(); torch.cuda.synchronize(); t2 = time.perf_counter()
    for _ in range(19): e.step()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    if pr: pr.disable()
    print(rep, f"engine {1e3*(t1-t0):.1f} ms  step0 {1e3*(t2-t1):.1f} ms  19 steps {1e3*(t3-t2):.1f} ms", flush=True)
    if pr:
        pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
    e.close()
