"""Relative error of the config-3 block product (n=1e6, d=9, b=2000, m=65)
against the live reference's fixture (tests/golden/config3.npz), per family:
the accuracy side of a kernel variant (SAP_LIB_PATH) next to its timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.rng import substream

g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "config3.npz"))
n, d, m = 1_000_000, 9, 65
X = synthetic.make_inputs(n, d, 0)
Z = substream(0, "golden_z3").standard_normal((n, m))
for fam in ("matern32", "rbf"):
    o = sap.KernelOracle(sap.KernelSpec(fam, np.full(d, np.sqrt(d)), 1.0), X, 1e-2)
    got = sap.col_dist_matmul(o, Z, g[f"{fam}_B"])
    ref = g[f"{fam}_G"]
    print(f"{fam}: max rel err {np.abs(got - ref).max() / np.abs(ref).max():.3e}", flush=True)
