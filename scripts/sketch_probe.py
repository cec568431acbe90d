import torch, time
d = torch.device("cuda")
c, b, r = 31, 2000, 100
K = torch.rand(c, b, b, device=d)
K = 0.5 * (K + K.transpose(1, 2))
Om = torch.randn(c, b, r, device=d, dtype=torch.float64)
def t(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): f()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e) / n
om32 = Om.float()
out = torch.empty(c, b, r, device=d)
print("fp32 bmm  %.3f ms" % t(lambda: torch.bmm(K, om32, out=out)))
Kh = K.half(); Kl = (K - Kh.float()).half()
Oh = Om.half(); Ol = (Om - Oh.double()).half()
OO = torch.cat([Oh, Ol], dim=2).contiguous()
def split3():
    o1 = torch.bmm(Kh, OO, out_dtype=torch.float32)
    o2 = torch.bmm(Kl, Oh, out_dtype=torch.float32)
    return o1[:, :, :r] + o1[:, :, r:] + o2
print("3-pass fp16 bmm (2 GEMMs + adds)  %.3f ms" % t(split3))
def splitK():
    Kh2 = K.half(); Kl2 = (K - Kh2.float()).half()
print("K split (torch)  %.3f ms" % t(splitK))
ref = torch.bmm(K.double(), Om)
print("err fp32", ((torch.bmm(K, om32) - ref).abs().max() / ref.abs().max()).item(),
      "err 3-pass", ((split3() - ref).abs().max() / ref.abs().max()).item())
