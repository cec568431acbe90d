"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container only (it imports the read-only reference package
from /root/reference/pkg/src). The GPU box never runs this script; it only
reads the committed .npz files.

    python tests/golden/make_golden.py

Fixtures (all float64, reference arithmetic):
  kernels_small.npz  block products / blocks / cross products, 3 families
                     (mirrors tests/test_kernels.py:66-142, test_dist.py)
  config1.npz        config 1 problem (n=2000 d=8 b=200 m=9 r=100 RBF):
                     inputs, per-iteration records for t=0..4, the full
                     500-iteration adasap_solve (block crc32s, stepsizes,
                     final W), posterior mean and RMSE on the test points
  config2.npz        one K[B,:]Z block product at config 2 / config 3 shape
                     (n=1e5, b=1000, m=65; RBF d=11 and Matern-3/2 d=9);
                     inputs are regenerated from seeds by the tests
  randnla.npz        Nystrom factor, Woodbury applies, power stepsize
  rng.npz            block crc32s / first draws for several (seed, t, n, b)
  config3.npz        config 3 (n=1e6, d=9, b=2000, m=65): one block product per
                     family (Matern-3/2, RBF) and a 5-iteration Matern-3/2
                     trajectory (block crc32s, stepsizes, sampled rows of W)
  config2_traj.npz   config 2 (n=1e5, d=11 RBF, b=1000, m=65, pathwise RHS) for
                     one pass (100 iterations): crc32s, stepsizes, sampled rows
                     of W, posterior mean and test RMSE
  nystrom_failures.npz  rand_nystrom_retry outcomes (S, or the NumericalError
                     message) on sketches of PSD, negative, indefinite and
                     low-rank matrices
  baselines.npz      the exact-SAP, SDD and Nystrom-PCG solvers (solvers.py:269-584) on
                     the config 1 problem: final estimates, residual traces,
                     block crc32s
"""

import os
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import sapgp  # noqa: E402  (the reference)
from sapgp import dist as rdist  # noqa: E402
from sapgp import randnla as rrand  # noqa: E402
from sapgp import solvers as rsol  # noqa: E402
from sapgp.rng import substream  # noqa: E402

from paper_2505_13723_b200 import synthetic  # noqa: E402


def kernels_small():
    out = {}
    rng = np.random.default_rng(1)
    X = rng.standard_normal((60, 3))
    M = rng.standard_normal((60, 4))
    B = np.sort(rng.choice(60, 17, replace=False))
    B = np.union1d(B, [0])  # the block contains index 0 (diagonal rule)
    Xs = rng.standard_normal((7, 3))
    omega = rng.standard_normal((B.size, 5))
    X300 = rng.standard_normal((300, 3))
    M300 = rng.standard_normal((300, 3))
    out.update(X=X, M=M, B=B, Xs=Xs, omega=omega, X300=X300, M300=M300,
               ls=np.array([0.9, 1.4, 0.6]), var=np.array(1.3))
    for fam in ("rbf", "matern32", "matern52"):
        spec = sapgp.KernelSpec(fam, np.array([0.9, 1.4, 0.6]), 1.3)
        orc = sapgp.KernelOracle(spec, X, 0.1)
        out[f"{fam}_KBM"] = rdist.col_dist_matmul(orc, M, B)
        out[f"{fam}_KBB"] = orc.block(B)
        out[f"{fam}_KBBom"] = rdist.row_dist_matmul(orc, omega, B)
        out[f"{fam}_cross"] = orc.cross_matmul(Xs, M)
        orc300 = sapgp.KernelOracle(spec, X300, 0.1)
        out[f"{fam}_matmul300"] = orc300.matmul(M300)
    np.savez_compressed(os.path.join(HERE, "kernels_small.npz"), **out)


def config1():
    n, d, b, m, r, lam, seed = 2000, 8, 200, 9, 100, 1e-2, 0
    prob = synthetic.make_problem(n, d, "rbf", m, seed=seed, lam=lam)
    spec = sapgp.KernelSpec("rbf", prob.lengthscales, prob.variance)
    orc = sapgp.KernelOracle(spec, prob.X, lam)
    cfg = sapgp.RunConfig(lam=lam, blocksize=b, nystrom_rank=r, residual_every=0,
                          seed=seed)
    accel = rsol.resolve_accel(cfg, n, b)
    out = dict(X=prob.X, Y=prob.Y, Xtest=prob.Xtest, ytest=prob.ytest,
               f_test=prob.f_test, ls=prob.lengthscales)
    # per-iteration detail for the first iterations, through the reference's
    # own step function (the Z passed to col_dist_matmul is the state's Z)
    state = rsol.SolverState.zeros(n, m, accelerated=True)
    for t in range(5):
        Zt = state.Z.copy()
        block = rsol._uniform_block(seed, t, n, b)
        G = rdist.col_dist_matmul(orc, Zt, block)
        omega = substream(seed, "omega", t).standard_normal((b, r))
        sketch = rdist.row_dist_matmul(orc, omega, block)
        fac = rrand.rand_nystrom_retry(sketch, omega, r)
        state, eta, blk = rsol.adasap_step(orc, state, prob.Y, cfg, accel)
        assert np.array_equal(blk, block)
        out[f"t{t}_Z"] = Zt
        out[f"t{t}_block"] = block
        out[f"t{t}_G"] = G
        out[f"t{t}_S"] = fac.S
        out[f"t{t}_eta"] = np.array(eta)
        out[f"t{t}_W"] = state.W.copy()
    res = rsol.adasap_solve(orc, prob.Y, cfg)
    out["final_W"] = res.W
    out["iters"] = np.array(res.iterations)
    out["crc"] = np.array([rec.block_hash for rec in res.trace.records], dtype=np.int64)
    out["eta"] = np.array([rec.stepsize for rec in res.trace.records])
    out["resid"] = np.array(res.trace.final_residual())
    pm = orc.cross_matmul(prob.Xtest, res.W)
    out["test_mean"] = pm
    out["test_rmse"] = np.array(sapgp.rmse(pm[:, 0], prob.ytest))
    np.savez_compressed(os.path.join(HERE, "config1.npz"), **out)


def config2():
    out = {}
    for tag, fam, d in (("rbf_d11", "rbf", 11), ("m32_d9", "matern32", 9)):
        n, b, m, seed = 100_000, 1000, 65, 0
        X = synthetic.make_inputs(n, d, seed)
        spec = sapgp.KernelSpec(fam, np.full(d, np.sqrt(d)), 1.0)
        orc = sapgp.KernelOracle(spec, X, 1e-2)
        Z = substream(seed, "golden_z").standard_normal((n, m))
        B = rsol._uniform_block(seed, 0, n, b)
        out[f"{tag}_B"] = B
        out[f"{tag}_G"] = rdist.col_dist_matmul(orc, Z, B, sapgp.WorkerPool(8))
    np.savez_compressed(os.path.join(HERE, "config2.npz"), **out)


def randnla():
    c1 = np.load(os.path.join(HERE, "config1.npz"))
    X, ls = c1["X"], c1["ls"]
    spec = sapgp.KernelSpec("rbf", ls, 1.0)
    orc = sapgp.KernelOracle(spec, X, 1e-2)
    B = c1["t1_block"]
    Kbb = orc.block(B)
    omega = substream(0, "omega", 1).standard_normal((B.size, 100))
    sketch = Kbb @ omega
    fac = rrand.rand_nystrom_retry(sketch, omega, 100)
    rho = float(fac.S[-1]) + 1e-2
    g = np.random.default_rng(3).standard_normal((B.size, 9))
    eta = rrand.rand_power_stepsize(lambda v: Kbb @ v + 1e-2 * v, fac, rho, 10,
                                    substream(0, "power", 1))
    np.savez_compressed(
        os.path.join(HERE, "randnla.npz"), Kbb=Kbb, omega=omega, S=fac.S,
        P=fac.U @ fac.U.T, rho=np.array(rho), g=g,
        inv=rrand.apply_inv(fac, rho, g), inv_sqrt=rrand.apply_inv_sqrt(fac, rho, g),
        eta=np.array(eta))


def baselines():
    """sdd_solve and pcg_solve of the reference on the config 1 problem."""
    n, d, b, m, lam, seed = 2000, 8, 200, 9, 1e-2, 0
    prob = synthetic.make_problem(n, d, "rbf", m, seed=seed, lam=lam)
    spec = sapgp.KernelSpec("rbf", prob.lengthscales, prob.variance)
    orc = sapgp.KernelOracle(spec, prob.X, lam)
    out = {}
    cfg = sapgp.RunConfig(lam=lam, blocksize=b, solver_id="sdd", max_iters=400,
                          residual_every=50, seed=seed, stepsize_scale=10.0)
    res = rsol.solve(orc, prob.Y, cfg)
    out["sdd_W"] = res.W
    out["sdd_res"] = np.array([r.residual for r in res.trace.records])
    out["sdd_crc"] = np.array([r.block_hash for r in res.trace.records], dtype=np.int64)
    out["sdd_eta"] = np.array([r.stepsize for r in res.trace.records])
    cfg = sapgp.RunConfig(lam=lam, blocksize=b, solver_id="sap", max_iters=60,
                          residual_every=10, seed=seed)
    res = rsol.solve(orc, prob.Y, cfg)
    out["sap_W"] = res.W
    out["sap_res"] = np.array([r.residual for r in res.trace.records])
    out["sap_crc"] = np.array([r.block_hash for r in res.trace.records], dtype=np.int64)
    for tag, rank in (("pcg", 100), ("cg", 0)):
        cfg = sapgp.RunConfig(lam=lam, solver_id="pcg", nystrom_rank=rank, max_iters=40,
                              seed=seed, tol=1e-6)
        res = rsol.solve(orc, prob.Y, cfg)
        out[f"{tag}_W"] = res.W
        out[f"{tag}_res"] = np.array([r.residual for r in res.trace.records])
        out[f"{tag}_iters"] = np.array(res.iterations)
    np.savez_compressed(os.path.join(HERE, "baselines.npz"), **out)


def rng_fixture():
    rows = []
    for seed, n, b in ((0, 2000, 200), (0, 100_000, 1000), (0, 1_000_000, 2000),
                       (7, 10_000_000, 5000)):
        for t in (0, 1, 2, 17, 499):
            blk = rsol._uniform_block(seed, t, n, b)
            rows.append((seed, n, b, t, zlib.crc32(blk.tobytes()), int(blk[0]), int(blk[-1])))
    om = substream(0, "omega", 3).standard_normal((5, 4))
    pw = substream(0, "power", 3).standard_normal(6)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), rows=np.array(rows, dtype=np.int64),
                        omega=om, power=pw)


# rows of W kept in the trajectory fixtures (a deterministic sample: the full
# n x m iterate does not fit a fixture)
def sample_rows(n, k=4096):
    return np.sort(substream(0, "golden_rows", n).choice(n, min(k, n), replace=False))


def config3():
    """Config 3 (the headline shape: n=1e6, d=9, b=2000, m=65) from the live
    reference: one block product per family (Matern-3/2 and RBF) and a
    5-iteration ADASAP trajectory (Matern-3/2, r=100, noise right-hand sides
    regenerated from a named substream)."""
    out = {}
    n, d, b, m, seed = 1_000_000, 9, 2000, 65, 0
    X = synthetic.make_inputs(n, d, seed)
    Z = substream(seed, "golden_z3").standard_normal((n, m))
    pool = sapgp.WorkerPool(8)
    for fam in ("matern32", "rbf"):
        spec = sapgp.KernelSpec(fam, np.full(d, np.sqrt(d)), 1.0)
        orc = sapgp.KernelOracle(spec, X, 1e-2)
        B = rsol._uniform_block(seed, 0, n, b)
        out[f"{fam}_B"] = B
        out[f"{fam}_G"] = rdist.col_dist_matmul(orc, Z, B, pool)
    del Z
    # 5 iterations of the reference solver, through its own step function
    # (adasap_solve would end with the relative residual, an n x n x m
    # product: hours at n = 1e6 in numpy)
    spec = sapgp.KernelSpec("matern32", np.full(d, np.sqrt(d)), 1.0)
    orc = sapgp.KernelOracle(spec, X, 1e-2)
    Y = substream(seed, "golden_y3").standard_normal((n, m))
    cfg = sapgp.RunConfig(lam=1e-2, blocksize=b, nystrom_rank=100, residual_every=0, seed=seed,
                          max_iters=5)
    accel = rsol.resolve_accel(cfg, n, b)
    state = rsol.SolverState.zeros(n, m, accelerated=True)
    crcs, etas = [], []
    for _ in range(5):
        state, eta, block = rsol.adasap_step(orc, state, Y, cfg, accel, pool)
        crcs.append(rsol._block_hash(block))
        etas.append(eta)
    rows = sample_rows(n)
    out["traj_rows"] = rows
    out["traj_W_rows"] = state.W[rows]
    out["traj_W_colnorm"] = np.linalg.norm(state.W, axis=0)
    out["traj_crc"] = np.array(crcs, dtype=np.int64)
    out["traj_eta"] = np.array(etas)
    pool.close()
    np.savez_compressed(os.path.join(HERE, "config3.npz"), **out)


def config2_trajectory():
    """Config 2 (houseelec-shaped: n=1e5, d=11, RBF, b=1000, m=65, pathwise
    right-hand sides built on the host) for one pass (100 iterations) of the
    live reference: block crc32s, stepsizes, sampled rows of W, the posterior
    mean at the test points and its test RMSE."""
    n, d, b, m, seed, lam = 100_000, 11, 1000, 65, 0, 1e-2
    prob = synthetic.make_problem(n, d, "rbf", m, seed=seed, lam=lam)
    spec = sapgp.KernelSpec("rbf", prob.lengthscales, prob.variance)
    orc = sapgp.KernelOracle(spec, prob.X, lam)
    cfg = sapgp.RunConfig(lam=lam, blocksize=b, nystrom_rank=100, residual_every=0, seed=seed,
                          max_passes=1.0)
    pool = sapgp.WorkerPool(8)
    res = rsol.adasap_solve(orc, prob.Y, cfg, pool=pool)
    pool.close()
    rows = sample_rows(n)
    pm = orc.cross_matmul(prob.Xtest, res.W)
    out = dict(rows=rows, W_rows=res.W[rows], W_colnorm=np.linalg.norm(res.W, axis=0),
               crc=np.array([rec.block_hash for rec in res.trace.records], dtype=np.int64),
               eta=np.array([rec.stepsize for rec in res.trace.records]),
               iters=np.array(res.iterations), test_mean=pm,
               test_rmse=np.array(sapgp.rmse(pm[:, 0], prob.ytest)),
               Y_colnorm=np.linalg.norm(prob.Y, axis=0))
    np.savez_compressed(os.path.join(HERE, "config2_traj.npz"), **out)


def nystrom_failures():
    """rand_nystrom_retry (randnla.py:97-106) on sketches of indefinite /
    negative matrices: which raise NumericalError (and which message), which
    succeed after escalating, and their S."""
    rng = np.random.default_rng(17)
    b, r = 120, 20
    out = {}
    cases = []
    A = rng.standard_normal((b, b))
    psd = A @ A.T / b
    ev, Q = np.linalg.eigh(psd)
    cases.append(("psd", psd))
    cases.append(("negdef", -psd))                                   # negative trace
    ind = Q @ np.diag(np.where(np.arange(b) % 3 == 0, -ev, ev)) @ Q.T  # indefinite, tr > 0
    cases.append(("indefinite", ind))
    low = Q[:, -10:] @ np.diag(ev[-10:]) @ Q[:, -10:].T                # rank 10 < r
    cases.append(("lowrank", low))
    names = []
    for k, (name, M) in enumerate(cases):
        om = rng.standard_normal((b, r))
        sk = M @ om
        out[f"{name}_sketch"], out[f"{name}_omega"] = sk, om
        try:
            fac = rrand.rand_nystrom_retry(sk, om, r)
            out[f"{name}_S"] = fac.S
            out[f"{name}_error"] = np.array("")
        except sapgp.NumericalError as exc:
            out[f"{name}_error"] = np.array(str(exc))
        names.append(name)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "nystrom_failures.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate only the named fixtures
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    kernels_small()
    config1()
    baselines()
    config2()
    randnla()
    rng_fixture()
    config3()
    config2_trajectory()
    nystrom_failures()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
