"""Quick tensor-core path check: tc vs FFMA vs oracle on a few shapes, then timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from oracle import sapgp_oracle as orc

def run(n, d, b, m, fam, ls=None, seed=0, check_oracle=True):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    ls = np.full(d, np.sqrt(d)) if ls is None else ls
    o = sap.KernelOracle(sap.KernelSpec(fam, ls, 1.3), X, 1e-2)
    B = np.sort(rng.choice(n, b, replace=False))
    W = rng.standard_normal((n, m))
    o.backend = "tc"; t = sap.col_dist_matmul(o, W, B)
    o.backend = "ffma"; f = sap.col_dist_matmul(o, W, B)
    msg = f"n={n} d={d} b={b} m={m} {fam}: tc-vs-ffma {np.abs(t-f).max()/np.abs(f).max():.2e}"
    if check_oracle:
        r = orc.col_dist_matmul(orc.Points(fam, ls, 1.3, X), W, B, workers=8)
        msg += f" tc-vs-oracle {np.abs(t-r).max()/np.abs(r).max():.2e} ffma-vs-oracle {np.abs(f-r).max()/np.abs(r).max():.2e}"
    print(msg, flush=True)

run(300, 3, 20, 4, "rbf")
run(1000, 9, 200, 9, "rbf")
run(1000, 9, 200, 9, "matern32")
run(5000, 11, 300, 65, "matern52")
run(20000, 9, 1000, 65, "matern32")
run(100000, 9, 1000, 65, "rbf", check_oracle=False)
# timing at config 3
from paper_2505_13723_b200 import synthetic
n, d, b, m = 1_000_000, 9, 2000, 65
X = synthetic.make_inputs(n, d, 0)
for fam in ("matern32", "rbf"):
    o = sap.KernelOracle(sap.KernelSpec(fam, np.full(d, 3.0), 1.0), X, 1e-2)
    Z = torch.randn(m, n, device="cuda")
    B = torch.as_tensor(np.sort(np.random.default_rng(0).choice(n, b, replace=False)), device="cuda")
    for be in ("tc", "ffma"):
        o.backend = be
        out = torch.empty(b, m, device="cuda")
        ts = []
        for _ in range(4):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); o.rows_times_device(B, Z, out=out); e.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ref = out.clone() if be == "tc" else ref
        print(f"config3 {fam} {be}: ms {[round(x,3) for x in ts]}  TFLOP/s {b*n*2*(d+m)/min(ts)*1e-9:.1f}", flush=True)
    print("tc vs ffma at config3:", float((ref - out).abs().max() / out.abs().max()))
