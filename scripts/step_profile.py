"""Per-phase timing of ADASAP iterations at config 3 (lookahead host/GPU split)."""
import os, sys, time
os.environ["SAP_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine
n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, "matern32", m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=60)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=60)
for _ in range(8): eng.step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(40): eng.step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0)/40:.3f} ms/iter, wall {1e3*(t2-t0)/40:.3f} ms/iter")
for tm in eng.la.timings[:2] + eng.la.timings[-2:]:
    print({k: (round(v*1e3, 2) if isinstance(v, float) else v) for k, v in tm.items()})
eng.close()
