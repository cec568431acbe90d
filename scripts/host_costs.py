"""Host (enqueue) cost of each part of one ADASAP step at config 2, measured
on a warmed engine with the lookahead idle: wall time per call of the solver
thread's pieces (device work queues asynchronously; a synchronize every 50
calls keeps the launch queue short)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200 import _native as nat
from paper_2505_13723_b200.kernels import krows_tc
from paper_2505_13723_b200.solvers import AdasapEngine

n, d, b, m, r = 100_000, 11, 1000, 65, 100
prob = synthetic.make_problem(n, d, "rbf", m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=2000)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=2000)
for _ in range(64):
    eng.step()
torch.cuda.synchronize()
time.sleep(2.0)  # let the producers finish their batches
plan = eng.la.get(eng.t)
zp, zq = eng._u1y, eng.s * eng._u2y
parts = {
    "la.get": lambda: eng.la.get(eng.t),
    "zop.fill": lambda: eng.zop.fill(eng.P, eng.Q, zp, zq, eng.Pb, eng.Qb),
    "krows_tc": lambda: krows_tc(o.spec, eng.tcp, plan.RAg, eng.b, plan.block_dev, eng.zop, eng.G,
                                 ws=eng.ws),
    "grad_gather": lambda: nat.call("sap_grad_gather", nat.ptr(eng.G), eng.G.stride(0),
                                    nat.ptr(eng.P), nat.ptr(eng.Q), nat.ptr(eng.Y), eng.ld, zp, zq,
                                    nat.ptr(plan.loc_dev), eng.b, eng.m, eng.lam, nat.ptr(eng.g),
                                    eng.g.stride(0), nat.stream_handle()),
    "phase4": lambda: torch.addmm(eng.g, plan.UMc, plan.U.T @ eng.g, alpha=-1.0),
    "empty ctypes call": lambda: nat.load().sap_abi_version(),
}
for name, fn in parts.items():
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    ts = []
    for k in range(400):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if k % 50 == 49:
            torch.cuda.synchronize()
    ts.sort()
    print(f"{name:16s} median {ts[len(ts) // 2] * 1e6:7.1f} us  p10 {ts[len(ts) // 10] * 1e6:7.1f} us")
t0 = time.perf_counter()
for _ in range(200):
    eng.step()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"full step (host, producers active) {(t1 - t0) / 200 * 1e6:.1f} us")
eng.close()
