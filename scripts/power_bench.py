"""Time sap_power_stepsize on a config-3 sized batch (8 x b=2000, r=100)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_13723_b200 import kernels as K
L, b, r = int(os.environ.get("PL", "8")), int(os.environ.get("B", "2000")), 100
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
A = torch.randn(L, b, b, device=dev, generator=g) / b
Kbb = (A @ A.transpose(1, 2)).float().contiguous()
U = torch.linalg.qr(torch.randn(L, b, r, device=dev, dtype=torch.float64))[0].contiguous()
S = torch.rand(L, r, device=dev, dtype=torch.float64) * 10
rho = torch.full((L,), 0.5, device=dev, dtype=torch.float64)
E = (1 / torch.sqrt(S + rho[:, None]) - 1 / torch.sqrt(rho[:, None])).contiguous()
v0 = torch.randn(L, b, device=dev, dtype=torch.float64)
v0 /= v0.norm(dim=1, keepdim=True)
eta = torch.empty(L, device=dev, dtype=torch.float64)
bad = torch.zeros(L, device=dev, dtype=torch.int32)
for rep in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); K.power_stepsize(Kbb, U, E, rho, v0, 1e-2, 10, eta, bad); e.record()
    torch.cuda.synchronize()
    print(f"power batch of {L}: {s.elapsed_time(e):.3f} ms")
# reference: torch fp64
Pd = lambda x: x * rho.rsqrt()[:, None] + torch.bmm(U, (E * torch.bmm(U.transpose(1, 2), x[:, :, None])[:, :, 0])[:, :, None])[:, :, 0]
v = v0.clone(); Kd = Kbb.double()
for _ in range(10):
    y = Pd(torch.bmm(Kd, Pd(v)[:, :, None])[:, :, 0] + 1e-2 * Pd(v))
    est = (v * y).sum(1); v = y / y.norm(dim=1, keepdim=True)
print("max rel eta err", ((eta - 1 / est).abs() / (1 / est).abs()).max().item(), "bad", bad.tolist())
