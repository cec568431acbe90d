"""Per-step device time of the first iterations of a fresh engine (the driver's
--steps 20 --warmup 5 window sits in the lookahead ramp): prints each step's
CUDA-event duration on the solver stream and the host time spent in step()."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine

n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
fam = os.environ.get("FAM", "matern32")
prob = synthetic.make_problem(n, d, fam, m, seed=0, lam=1e-2, device="cuda")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
steps = int(os.environ.get("STEPS", "25"))
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=steps)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=steps + 8)
torch.cuda.synchronize()
evs, host = [], []
for t in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    eng.step()
    e1.record()
    host.append(time.perf_counter() - h0)
    evs.append((e0, e1))
torch.cuda.synchronize()
for t, ((e0, e1), h) in enumerate(zip(evs, host)):
    print(f"t={t:3d} device {e0.elapsed_time(e1):8.3f} ms  host {h * 1e3:8.3f} ms")
eng.close()
