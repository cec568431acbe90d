"""Run the config-3 block-row product a few times (profiling target).

    python scripts/krows_once.py [--family matern32] [--reps 3]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic

ap = argparse.ArgumentParser()
ap.add_argument("--family", default="matern32")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--b", type=int, default=2000)
ap.add_argument("--m", type=int, default=65)
ap.add_argument("--d", type=int, default=9)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--backend", default="tc")
a = ap.parse_args()
X = synthetic.make_inputs(a.n, a.d, 0)
o = sap.KernelOracle(sap.KernelSpec(a.family, np.full(a.d, np.sqrt(a.d)), 1.0), X, 1e-2)
o.backend = a.backend
Z = torch.randn(a.m, a.n, device="cuda")
B = torch.as_tensor(np.sort(np.random.default_rng(0).choice(a.n, a.b, replace=False)), device="cuda")
out = torch.empty(a.b, a.m, device="cuda")
times = []
for _ in range(a.reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); o.rows_times_device(B, Z, out=out); e.record(); torch.cuda.synchronize()
    times.append(s.elapsed_time(e))
ent = a.b * a.n
print(f"krows {a.family} n={a.n} b={a.b} m={a.m}: ms={times} entries/s={ent/min(times)*1e3:.3e} "
      f"TFLOP/s={ent*2*(a.d+a.m)/min(times)*1e-9:.2f}")
