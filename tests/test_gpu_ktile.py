"""The batched K_BB tile (sap_ktile_f32_batch, the lookahead's power-iteration
input) against the per-block tile kernel sap_ktile_f32: same values bit for
bit, one launch per batch. Both are checked against the CPU oracle's
block_block (KernelOracle.block, kernels.py:129-136) at the headline shape in
tests/test_gpu_config3.py::test_hot_path_kbb_tile_matches_oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
sap = pytest.importorskip("paper_2505_13723_b200")
K = pytest.importorskip("paper_2505_13723_b200.kernels")


@pytest.mark.parametrize("family", ["rbf", "matern32", "matern52"])
@pytest.mark.parametrize("b,d", [(2000, 9), (1000, 11), (37, 3), (64, 16), (130, 1)])
def test_ktile_batch_bitwise(family, b, d):
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(b + d)
    n, count = 3 * b + 5, 3
    X = rng.standard_normal((n, d))
    spec = sap.KernelSpec(family, np.full(d, 0.8 * np.sqrt(d)), 1.7)
    o = sap.KernelOracle(spec, X, 1e-2, device=dev)
    pts = o.points
    ld = (b + 3) // 4 * 4
    Xb = torch.empty((count, b, pts.ldx), dtype=torch.float32, device=dev)
    rsq = torch.empty((count, b), dtype=torch.float32, device=dev)
    ids = []
    for q in range(count):
        blk = torch.as_tensor(np.sort(rng.choice(n, b, replace=False)), device=dev)
        ids.append(blk)
        pts.gather(blk, out=(Xb[q], rsq[q]))
    ref = torch.zeros((count, b, ld), dtype=torch.float32, device=dev)
    got = torch.zeros_like(ref)
    for q in range(count):
        K.ktile_f32(spec, Xb[q], rsq[q], ids[q], Xb[q], rsq[q], ids[q], pts.ldx, pts.d, ref[q])
    K.ktile_f32_batch(spec, Xb, rsq, pts.d, got)
    torch.cuda.synchronize()
    assert torch.equal(ref, got)
    assert torch.equal(got[:, :, :b], got[:, :, :b].transpose(1, 2))  # symmetric
