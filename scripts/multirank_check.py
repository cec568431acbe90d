"""N-rank ADASAP on the real kernels, for the multi-rank parity test
(tests/test_gpu_multirank.py): each process runs ``adasap_solve`` on its
shard of the point dimension with the engine's all-reduce of the block
gradient (and, with the distributed lookahead, the owner's broadcast of a
batch's Nystrom/stepsize products). A second, device-resident solve (each rank
passes its rows of Y as a CUDA tensor and keeps its shard of W) feeds the
sharded test-point product (one t x m all-reduce). Launched by torchrun; the process group
backend comes from SAP_DIST_BACKEND (gloo lets two ranks share one GPU for a
correctness check -- no kernel waits on another rank's kernels, the
collectives go through the host). Rank 0 writes W, the block crc32s and the
stepsizes to the .npz path given as argv[1].
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

import paper_2505_13723_b200 as sap  # noqa: E402
from paper_2505_13723_b200.parallel import init_from_env  # noqa: E402

out = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40
if "RANK" in os.environ:
    init_from_env(os.environ.get("SAP_DIST_BACKEND", "gloo"))
torch.cuda.set_device(0)
rng = np.random.default_rng(21)
n, d, m = 6000, 9, 17
X = rng.standard_normal((n, d))
Y = rng.standard_normal((n, m))
o = sap.KernelOracle(sap.KernelSpec("matern32", np.full(d, 2.0), 1.0), X, 1e-2, device=0)
cfg = sap.RunConfig(lam=1e-2, blocksize=512, nystrom_rank=64, residual_every=20, seed=3,
                    max_iters=iters)
res = sap.adasap_solve(o, Y, cfg)
# the device-resident solve: each rank passes only its rows of Y as a CUDA
# tensor and keeps its shard of W; predictions by the sharded cross product
from paper_2505_13723_b200.parallel import current_shard  # noqa: E402
sh = current_shard(n)
Yd = torch.as_tensor(Y, device="cuda")
Yd = Yd[sh.lo:sh.hi].contiguous() if sh.world > 1 else Yd
res_d = sap.adasap_solve(o, Yd, cfg)
assert torch.is_tensor(res_d.W) and res_d.W.shape[0] == sh.size
Xs = np.random.default_rng(5).standard_normal((300, d))
pred_d = o.cross_matmul(Xs, res_d.W).double().cpu().numpy()
pred_h = o.cross_matmul(Xs, res.W)
if not tdist.is_initialized() or tdist.get_rank() == 0:
    np.savez(out, W=res.W, crc=np.array([r.block_hash for r in res.trace.records]),
             eta=np.array([r.stepsize for r in res.trace.records]),
             res=np.array([r.residual for r in res.trace.records]),
             res_d=np.array([r.residual for r in res_d.trace.records]),
             pred_d=pred_d, pred_h=pred_h)
if tdist.is_initialized():
    tdist.barrier()
    tdist.destroy_process_group()
