"""Wall-clock trace of the lookahead producers against the solver steps:
when each batch is submitted, when its phases are enqueued, when the solver
consumes it (steady state, config 3)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic, pipeline
from paper_2505_13723_b200.solvers import AdasapEngine
T0 = time.perf_counter()
log = []
orig = pipeline.Lookahead._produce
def traced(self, slot, t0, count, side, owner=0):
    log.append((time.perf_counter() - T0, "produce-start", t0, count, threading.get_ident() % 1000))
    out = orig(self, slot, t0, count, side, owner)
    log.append((time.perf_counter() - T0, "produce-end", t0, count, threading.get_ident() % 1000))
    return out
pipeline.Lookahead._produce = traced
origp = pipeline.K.power_stepsize
def tp(*a, **k):
    log.append((time.perf_counter() - T0, "power-enqueue", None, None, threading.get_ident() % 1000))
    return origp(*a, **k)
pipeline.K.power_stepsize = tp
n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, "matern32", m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=2000)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=2000)
for t in range(400):
    if t % 32 == 31 or t < 70:
        torch.cuda.synchronize()
        log.append((time.perf_counter() - T0, "step", t, None, 0))
    eng.step()
torch.cuda.synchronize()
log.append((time.perf_counter() - T0, "end", None, None, 0))
for e in sorted(log):
    print(f"{e[0]*1e3:10.2f} ms  {e[1]:15s} t0={e[2]} count={e[3]} thr={e[4]}")
eng.close()
