"""Phase IV probe: how often the fused launch rebuilds the next operand, and
the launch's time by mode (GRAD / APPLY / both, with and without the next
operand) at config 3 (b=2000, m=65, r=100)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic, _native as nat
from paper_2505_13723_b200.solvers import AdasapEngine

# config 3 by default; N=100000 D=11 B=1000 FAM=rbf for config 2
n, d, b = int(os.environ.get("N", "1000000")), int(os.environ.get("D", "9")), int(os.environ.get("B", "2000"))
m, r = 65, 100
prob = synthetic.make_problem(n, d, os.environ.get("FAM", "matern32"), m, seed=0, lam=1e-2,
                              device="cuda", rhs=os.environ.get("RHS", "noise"))
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
TOTAL = 200
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0, max_iters=TOTAL)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=TOTAL)
flags = []
for t in range(TOTAL - 8):
    fi = eng._fi
    eng.step()
    torch.cuda.synchronize()
    flags.append(int(eng.zflag[fi]))
print("rebuilds:", sum(flags), "of", len(flags), "first at", [i for i, f in enumerate(flags) if f][:20])

# isolated timing of the launch (state of the last step, repeated)
lib = nat.load()
plan = eng.la.get(eng.t)
a = nat.StepArgs()
a.part, a.splits, a.variance, a.zscale = nat.ptr(eng.ws), 37, 1.0, nat.ptr(eng.zop.scale)
a.P, a.Q, a.Y, a.ldp, a.zp, a.zq, a.lam = nat.ptr(eng.P), nat.ptr(eng.Q), nat.ptr(eng.Y), eng.ld, \
    0.7, 0.1, 1e-2
a.loc, a.b, a.m, a.g, a.ldgo = nat.ptr(plan.loc_dev), b, m, nat.ptr(eng.g), m
a.U, a.UMc, a.ldu, a.r = nat.ptr(plan.U), nat.ptr(plan.UMc), r, r
a.Pw, a.Qw, a.eta_dev, a.e0, a.e1 = nat.ptr(eng.P), nat.ptr(eng.Q), nat.ptr(plan.eta_rho_dev), 0.0, 0.0
Pb = eng.Pb.clone()
Qb = eng.Qb.clone()
a.WB, a.ldwb, a.Pb, a.Qb = nat.ptr(eng.WB), m, nat.ptr(Pb), nat.ptr(Qb)
ws = eng.p4ws
st = nat.stream_handle()


def timeit(mode, nxt, reps=50):
    if nxt:
        zn = eng.zop_next
        a.Zhi_next, a.Zlo_next, a.ldz, a.zscale_next = nat.ptr(zn.hi), nat.ptr(zn.lo), zn.ldz, nat.ptr(zn.scale)
        a.zp1, a.zq1, a.zflag, a.flag_idx, a.n_local = 0.7, 0.1, nat.ptr(eng.zflag), 0, n
    else:
        a.Zhi_next = None
    for _ in range(3):
        nat.check(lib.sap_block_step(ctypes.byref(a), mode, nat.ptr(ws), ws.numel() * 8, st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        nat.check(lib.sap_block_step(ctypes.byref(a), mode, nat.ptr(ws), ws.numel() * 8, st))
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for dbg in ("5", "6", "7", "0"):
    os.environ["SAP_P4_DEBUG"] = dbg
    print("GRAD|APPLY dbg %s (5: no B product, 6: no D product, 7: no update): %.1f us"
          % (dbg, timeit(3, False)))
for dbg in ("8", "9"):
    os.environ["SAP_P4_DEBUG"] = dbg
    print("GRAD|APPLY + next dbg %s (8: no rebuild check, 9: no operand rows): %.1f us"
          % (dbg, timeit(3, True)))
os.environ["SAP_P4_DEBUG"] = "0"
print("GRAD        %.1f us" % timeit(1, False))
print("GRAD|APPLY + next %.1f us" % timeit(3, True))
os.environ["SAP_P4_NO_PDL"] = "1"
print("GRAD|APPLY + next, no PDL %.1f us" % timeit(3, True))
del os.environ["SAP_P4_NO_PDL"]
print("APPLY       %.1f us" % timeit(2, False))
print("GRAD|APPLY  %.1f us" % timeit(3, False))
a.Pw = None
print("APPLY no update %.1f us" % timeit(2, False))
a.r = 0
print("APPLY r=0 no update %.1f us" % timeit(2, False))
eng.close()
