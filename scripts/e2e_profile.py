"""Where the public-API solve spends its fixed time (config 3 shapes)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine
n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, "matern32", m, seed=0, lam=1e-2, device="cuda", rhs="noise")
X, Y = prob.X, prob.Y
for rep in range(2):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    o = sap.KernelOracle(prob.spec(), X, prob.lam); torch.cuda.synchronize(); t.append(time.perf_counter())
    cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=30)
    eng = AdasapEngine(o, Y, cfg, sap.resolve_accel(cfg, n, b), total=30); torch.cuda.synchronize(); t.append(time.perf_counter())
    for _ in range(30): eng.step()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    W = eng.materialize("W").cpu().numpy().astype(np.float64); t.append(time.perf_counter())
    eng.close(); t.append(time.perf_counter())
    print(f"rep {rep}: oracle {t[1]-t[0]:.3f}s engine {t[2]-t[1]:.3f}s 30 steps {t[3]-t[2]:.3f}s W->host {t[4]-t[3]:.3f}s close {t[5]-t[4]:.3f}s", flush=True)
t0 = time.perf_counter(); o = sap.KernelOracle(prob.spec(), X, prob.lam)
res = sap.adasap_solve(o, Y, sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=30))
print(f"adasap_solve end-to-end {time.perf_counter()-t0:.3f}s")
