"""Time-to-target test RMSE with the device-resident pathwise problem
(synthetic.make_problem_device): one solve of the m = 65 right-hand sides,
the test RMSE of the posterior mean (column 0) evaluated on the device every
``--every`` iterations from a single materialised column (no n x m buffer).
Config 5 (taxi-shaped, n = 10^8, b = 10^4) fits one B200:

    python scripts/time_to_rmse_device.py --n 100000000 --b 10000 --passes 1
"""
import argparse, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--d", type=int, default=9)
ap.add_argument("--b", type=int, default=2000)
ap.add_argument("--family", default="rbf")
ap.add_argument("--passes", type=float, default=1.0)
ap.add_argument("--every", type=int, default=500)
ap.add_argument("--out", default=None)
a = ap.parse_args()
dev = torch.device("cuda", 0)
t0 = time.perf_counter()
prob = synthetic.make_problem_device(a.n, a.d, a.family, 65, seed=0, lam=1e-2, device=dev)
t_gen = time.perf_counter() - t0
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam, device=dev)
total = max(1, math.ceil(a.passes * a.n / a.b))
cfg = sap.RunConfig(lam=prob.lam, blocksize=a.b, nystrom_rank=100, residual_every=0, seed=0)
torch.cuda.synchronize()
t1 = time.perf_counter()
eng = AdasapEngine(o, prob.Ycm.T, cfg, sap.resolve_accel(cfg, a.n, a.b), total=total)
rows = []
out = open(a.out, "w") if a.out else None


def record(it):
    el = time.perf_counter() - t1
    w0 = eng.materialize("W", col=0)
    pred = o.cross_matmul(prob.Xtest, w0)[:, 0].double().cpu().numpy()
    rm = sap.rmse(pred, prob.ytest)
    row = {"iteration": it, "passes": it * a.b / a.n, "solve_seconds": el, "test_rmse": rm,
           "eval_seconds": time.perf_counter() - t1 - el}
    rows.append(row)
    line = json.dumps(row)
    print(line, flush=True)
    if out:
        out.write(line + "\n")
        out.flush()


eval_s = 0.0
for it in range(1, total + 1):
    eng.step()
    if it % a.every == 0 or it == total:
        torch.cuda.synchronize()  # the steps so far are solve time
        e0 = time.perf_counter()
        record(it)
        eval_s += time.perf_counter() - e0
        t1 += time.perf_counter() - e0  # evaluations are not solve time
eng.la.check_flags()
eng.close()
final = rows[-1]["test_rmse"]
summary = {"workload": f"synthetic {a.family} GP n={a.n} d={a.d} b={a.b} m=65 r=100, pathwise "
                       "RHS built on the device (make_problem_device)",
           "problem_generation_s": t_gen, "iterations": total, "passes": total * a.b / a.n,
           "solve_seconds": rows[-1]["solve_seconds"], "final_test_rmse": final,
           "time_to_within_1pct_s": next((r["solve_seconds"] for r in rows
                                          if r["test_rmse"] <= 1.01 * final), None),
           "evaluation_seconds_excluded": eval_s,
           "device_mem_gb": (torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9}
print(json.dumps(summary), flush=True)
if out:
    out.write(json.dumps(summary) + "\n")
