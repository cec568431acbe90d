import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200.solvers import AdasapEngine
rng = np.random.default_rng(6)
X = rng.uniform(-1, 1, size=(200, 2))
o = sap.KernelOracle(sap.KernelSpec("rbf", np.full(2, 0.4), 1.0), X, 1.0)
ones = np.ones(200)
y = o.matmul(ones) + ones
print("y finite", np.isfinite(y).all(), y[:3])
cfg = sap.RunConfig(lam=1.0, solver_id="adasap", blocksize=25, nystrom_rank=25, max_iters=200, residual_every=0)
acc = sap.resolve_accel(cfg, 200, 25)
eng = AdasapEngine(o, y, cfg, acc, total=200)
for t in range(40):
    plan = eng.step()
    torch.cuda.synchronize()
    W = eng.materialize("W")
    print(t, "rho", plan.rho, "S", plan.S[:3], plan.S[-3:], "eta", float(eng.etas[t]), "g", float(eng.g.abs().max()),
          "W", float(W.abs().max()), "P", float(eng.P.abs().max()), "Q", float(eng.Q.abs().max()), "M", eng.M.ravel())
    if not torch.isfinite(W).all():
        break
eng.close()
