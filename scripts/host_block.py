"""Which host call of an ADASAP step blocks (steady state, config 3)."""
import collections, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic, solvers, _native as nat
from paper_2505_13723_b200.solvers import AdasapEngine
n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, "matern32", m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=80)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=80)
for _ in range(8): eng.step()
torch.cuda.synchronize()
acc = collections.defaultdict(float)
cnt = collections.defaultdict(int)
def wrap(obj, name, label):
    f = getattr(obj, name)
    def w(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            acc[label] += time.perf_counter() - t
            cnt[label] += 1
    setattr(obj, name, w)
wrap(eng.la, "get", "la.get")
wrap(eng.zop, "fill", "zop.fill")
wrap(solvers, "krows_tc", "krows_tc")
wrap(eng, "_update", "_update")
orig_call = nat.call
def call(name, *a):
    t = time.perf_counter()
    try:
        return orig_call(name, *a)
    finally:
        acc["nat." + name] += time.perf_counter() - t
        cnt["nat." + name] += 1
nat.call = call
solvers.nat.call = call
t0 = time.perf_counter()
for _ in range(40): eng.step()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host {1e3*(t1-t0)/40:.3f} ms/iter")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:28s} {1e3*v/40:8.3f} ms/iter  ({cnt[k]} calls)")
eng.close()
