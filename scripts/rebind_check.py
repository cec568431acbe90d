"""INTEGRATION.md §2 check: the UNMODIFIED reference solver loop (installed in
baseline/_ref) running on the B200 block product via rebinding."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import numpy as np
import sapgp, sapgp.solvers as ref_solvers
import paper_2505_13723_b200 as b2
g = np.load(os.path.join(ROOT, "tests", "golden", "config1.npz"))
oracle = b2.KernelOracle(b2.KernelSpec("rbf", g["ls"], 1.0), g["X"], 1e-2)
ref_solvers.col_dist_matmul = b2.col_dist_matmul
ref_solvers.row_dist_matmul = b2.row_dist_matmul
cfg = sapgp.RunConfig(lam=1e-2, blocksize=200, nystrom_rank=100, residual_every=0, max_iters=100)
res = ref_solvers.adasap_solve(oracle, g["Y"], cfg)
crc = np.array([rec.block_hash for rec in res.trace.records])
print("blocks equal:", np.array_equal(crc, g["crc"][:100]))
ref = np.load(os.path.join(ROOT, "tests", "golden", "config1.npz"))
print("stepsize rel diff:", np.abs(np.array([r.stepsize for r in res.trace.records]) - ref["eta"][:100]).max() / ref["eta"].max())
