"""Cost of the lookahead's GPU phases for one batch of L=8 iterations, GPU otherwise idle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic, kernels as K
from paper_2505_13723_b200.pipeline import _Cols
n, d, b, r, L = 1_000_000, 9, 2000, 100, 8
X = synthetic.make_inputs(n, d, 0)
o = sap.KernelOracle(sap.KernelSpec("matern32", np.full(d, 3.0), 1.0), X, 1e-2)
pts = o.points
rng = np.random.default_rng(0)
bd = torch.as_tensor(np.stack([np.sort(rng.choice(n, b, replace=False)) for _ in range(L)]), device="cuda")
om = torch.randn(L, b, r, dtype=torch.float64, device="cuda")
def T(name, fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): out = fn()
    torch.cuda.synchronize()
    print(f"{name:30s} {1e3*(time.perf_counter()-t0)/reps:8.3f} ms", flush=True)
    return out
Xb = torch.empty(L, b, pts.ldx, device="cuda"); rsq = torch.empty(L, b, device="cuda")
def gathers():
    for i in range(L): pts.gather(bd[i], out=(Xb[i], rsq[i]))
T("gather x8", gathers)
Kbb = torch.empty(L, b, b, dtype=torch.float64, device="cuda")
def kt():
    for i in range(L): Kbb[i] = K.ktile(o.spec, Xb[i], rsq[i], bd[i], Xb[i], rsq[i], bd[i], pts.ldx, pts.d)
T("ktile x8", kt)
sk = torch.empty(L, b, r, device="cuda")
def sketch():
    for i in range(L):
        omc = om[i].T.to(torch.float32).contiguous()
        K.krows_times(o.spec, _Cols(pts, Xb[i], rsq[i]), Xb[i], rsq[i], bd[i], omc, sk[i], col_ids=bd[i])
T("sketch x8 (ffma)", sketch)
Y = sk.double()
from paper_2505_13723_b200.pipeline import chol_qr3
badf = torch.zeros(L, dtype=torch.int32, device="cuda")
T("qr batched (cusolver)", lambda: torch.linalg.qr(Y))
Q, R = T("chol_qr3 batched", lambda: chol_qr3(Y, badf))
T("grams", lambda: torch.stack([R, om.transpose(1,2) @ Y, om.transpose(1,2) @ om], dim=1))
U = Q
E = torch.rand(L, r, dtype=torch.float64, device="cuda")
v = torch.randn(L, b, dtype=torch.float64, device="cuda")
rho = torch.rand(L, dtype=torch.float64, device="cuda") + 0.1
def power():
    isr = rho.rsqrt()[:, None]; vv = v
    for _ in range(10):
        w = vv * isr + torch.bmm(U, (E * torch.bmm(U.transpose(1, 2), vv[:, :, None])[:, :, 0])[:, :, None])[:, :, 0]
        z = torch.bmm(Kbb, w[:, :, None])[:, :, 0] + 0.01 * w
        y = z * isr + torch.bmm(U, (E * torch.bmm(U.transpose(1, 2), z[:, :, None])[:, :, 0])[:, :, None])[:, :, 0]
        est = (vv * y).sum(1); ny = torch.linalg.vector_norm(y, dim=1); vv = y / ny[:, None]
    return est
T("power x10 batched", power)
