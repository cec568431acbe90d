"""cProfile of the solver's main thread over steady-state ADASAP steps (config 3):
where the per-step host time goes (launch wrappers, numpy, torch ops)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine
# python scripts/step_cprofile.py [n d b family]
args = sys.argv[1:]
n, d, b = (int(args[0]), int(args[1]), int(args[2])) if len(args) >= 3 else (1_000_000, 9, 2000)
fam = args[3] if len(args) >= 4 else "matern32"
m, r = 65, 100
prob = synthetic.make_problem(n, d, fam, m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=400)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=400)
for _ in range(40):
    eng.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    eng.step()
pr.disable()
torch.cuda.synchronize()
eng.close()
st = pstats.Stats(pr).sort_stats("tottime")
st.print_stats(25)
st.sort_stats("cumulative").print_callees("step")
st.sort_stats("cumulative").print_callees("krows_tc")
