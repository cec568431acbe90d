"""Wall-time pieces of the public-API setup and W readback (bench e2e fixed costs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
import bench

C = bench.CONFIG
dev = torch.device("cuda")
prob = synthetic.make_problem(C["n"], C["d"], C["family"], C["m"], seed=C["seed"], lam=C["lam"], device=dev)
spec = prob.spec()
X, Y = np.ascontiguousarray(prob.X), np.ascontiguousarray(prob.Y)
def tick(label, f):
    torch.cuda.synchronize(); a = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print(f"{label:28s} {1e3*(time.perf_counter()-a):8.1f} ms", flush=True); return r
for rep in range(2):
    cfg = sap.RunConfig(lam=prob.lam, blocksize=C["b"], nystrom_rank=C["r"], residual_every=0, seed=0, max_iters=20)
    o = tick("KernelOracle", lambda: sap.KernelOracle(spec, X, prob.lam, device=dev))
    tick("tc_points", lambda: o.tc_points())
    accel = sap.resolve_accel(cfg, o.n, C["b"])
    st = tick("make_state", lambda: sap.make_state(o, Y, cfg, accel))
    tick("5 steps", lambda: [sap.adasap_step(o, st, Y, cfg, accel) for _ in range(5)])
    Wd = tick("materialize W", lambda: st._e.materialize("W"))
    W64 = tick("to f64 contiguous", lambda: Wd.to(torch.float64).contiguous())
    tick("cpu()", lambda: W64.cpu())
    tick("state.W total", lambda: st.W)
    def pinned():
        h = torch.empty(W64.shape, dtype=torch.float64, pin_memory=True)
        h.copy_(W64)
        return h
    tick("pinned alloc+copy", pinned)
    h = torch.empty(W64.shape, dtype=torch.float64, pin_memory=True)
    tick("copy into pinned", lambda: h.copy_(W64))
    tick("numpy empty+copy", lambda: torch.from_numpy(np.empty(W64.shape)).copy_(W64))
    st._e.close()
from paper_2505_13723_b200.kernels import to_colmajor
from paper_2505_13723_b200.pipeline import Lookahead
from paper_2505_13723_b200 import dist as _d
for rep in range(2):
    tick("to_colmajor(Y)", lambda: to_colmajor(Y, Y.shape[0], dev, (Y.shape[0] + 3) // 4 * 4))
    tick("Y as_tensor H2D", lambda: torch.as_tensor(Y, device=dev))
    sh = _d.current_shard(o.n) if hasattr(_d, "current_shard") else None
    la = tick("Lookahead init", lambda: Lookahead(o, st._e.shard, 0, C["b"], C["r"], prob.lam, 40, 8, False, tcp=o.tc_points()))
    la.close()
    import threading
    def prefault():
        out = np.empty(W64.shape)
        flat = out.reshape(-1)
        k = 8
        ths = [threading.Thread(target=lambda i=i: flat[i * len(flat) // k:(i + 1) * len(flat) // k].fill(0.0)) for i in range(k)]
        [t.start() for t in ths]; [t.join() for t in ths]
        torch.from_numpy(out).copy_(W64)
        return out
    tick("prefault8+copy", prefault)
