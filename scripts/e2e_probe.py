"""Per-step wall times of the public-API loop (bench.py run_e2e) to locate host stalls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
import bench

K = int(sys.argv[1]) if len(sys.argv) > 1 else 40
C = bench.CONFIG
prob = synthetic.make_problem(C["n"], C["d"], C["family"], C["m"], seed=C["seed"], lam=C["lam"],
                              device=torch.device("cuda"))
spec = prob.spec()
X, Y = np.ascontiguousarray(prob.X), np.ascontiguousarray(prob.Y)
for read_eta in (True, False, True):
    cfg = sap.RunConfig(lam=prob.lam, blocksize=C["b"], nystrom_rank=C["r"], residual_every=0,
                        seed=C["seed"], max_iters=K)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o = sap.KernelOracle(spec, X, prob.lam, device=torch.device("cuda"))
    accel = sap.resolve_accel(cfg, o.n, C["b"])
    st = sap.make_state(o, Y, cfg, accel)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ts = []
    for _ in range(K):
        a = time.perf_counter()
        if read_eta:
            st, eta, blk = sap.adasap_step(o, st, Y, cfg, accel)
        else:
            st._e.step()
        ts.append(time.perf_counter() - a)
    W = st.W
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st._e.close()
    print(f"read_eta={read_eta} setup {t1-t0:.3f}s steps {t2-t1:.3f}s ({(t2-t1)/K*1e3:.2f} ms/step) "
          f"per-step ms: " + " ".join(f"{x*1e3:.1f}" for x in ts[:12]) + " ... " +
          " ".join(f"{x*1e3:.1f}" for x in ts[-6:]), flush=True)
