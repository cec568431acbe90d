"""Per-role cycle timers of the block-row kernel INSIDE the solver (config 3):
needs a -DSAP_TC_TIMERS=1 build (scripts/build_variant.sh tm
"-DSAP_TC_TIMERS=1", then SAP_LIB_PATH=.../_lib_tm/libsapgp_b200.so). Runs to
steady state, then profiles two launches (the library prints the per-CTA
averages to stderr)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine

# config 3 by default; N=100000 D=11 B=1000 FAM=rbf for config 2
n, d, b = int(os.environ.get("N", "1000000")), int(os.environ.get("D", "9")), int(os.environ.get("B", "2000"))
m, r = 65, 100
prob = synthetic.make_problem(n, d, os.environ.get("FAM", "matern32"), m, seed=0, lam=1e-2,
                              device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), unbounded=True)
for _ in range(80):
    eng.step()
torch.cuda.synchronize()
os.environ["SAP_TC_PROF"] = "1"
for _ in range(2):
    eng.step()
torch.cuda.synchronize()
del os.environ["SAP_TC_PROF"]
eng.close()
