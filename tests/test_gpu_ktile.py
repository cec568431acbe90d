"""The batched K_BB tile (sap_ktile_f32_batch, the lookahead's power-iteration
input) against the per-block tile kernel sap_ktile_f32: same values bit for
bit, one launch per batch. Both are checked against the CPU oracle's
block_block (KernelOracle.block, kernels.py:129-136) at the headline shape in
tests/test_gpu_config3.py::test_hot_path_kbb_tile_matches_oracle. The power
iteration that consumes those tiles (sap_power_stepsize) is checked for each
cluster size it launches with against a torch fp64 restatement."""
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
    # exactly symmetric (the power iteration reads one triangle of it)
    assert torch.equal(got[:, :, :b], got[:, :, :b].transpose(1, 2))
    assert torch.equal(got[:, :, :b], got[:, :, :b].transpose(1, 2))  # symmetric


@pytest.mark.parametrize("sym", [None, "1"])
@pytest.mark.parametrize("cluster", ["4", "8", "16", None])
@pytest.mark.parametrize("count,b,r", [(32, 2000, 100), (5, 1000, 100), (3, 130, 7), (2, 64, 0),
                                       (2, 333, 5), (2, 332, 5), (3, 124, 6), (2, 20, 3),
                                       (2, 10000, 20)])
def test_power_stepsize_cluster_sizes(sym, cluster, count, b, r, monkeypatch):
    """sap_power_stepsize (csrc/power.cu; randnla.py:165-196) for every cluster
    size the launcher picks (None: its own choice, one wave when it can), with
    the launcher's choice of sweep and with the symmetric sweep forced (empty
    and partial column blocks at small b; rows not 16-byte aligned, or a
    symmetric sweep too large for shared memory (b = 10 000 at C = 4), fall
    back to the full sweep), against the same preconditioned power iteration
    in torch fp64."""
    if cluster is None:
        monkeypatch.delenv("SAP_POWER_CLUSTER", raising=False)
    else:
        monkeypatch.setenv("SAP_POWER_CLUSTER", cluster)
    if sym is None:
        monkeypatch.delenv("SAP_POWER_SYM", raising=False)
    else:
        monkeypatch.setenv("SAP_POWER_SYM", sym)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(count * b + r)
    A = torch.randn(count, b, b, device=dev, generator=g) / b
    Kbb = (A @ A.transpose(1, 2)).float()
    Kbb = (0.5 * (Kbb + Kbb.transpose(1, 2))).contiguous()  # exactly symmetric, as K_BB
    rho = torch.full((count,), 0.5, device=dev, dtype=torch.float64)
    if r:
        U = torch.linalg.qr(torch.randn(count, b, r, device=dev, dtype=torch.float64,
                                        generator=g))[0].contiguous()
        S = torch.rand(count, r, device=dev, dtype=torch.float64, generator=g) * 10
        E = (1 / torch.sqrt(S + rho[:, None]) - 1 / torch.sqrt(rho[:, None])).contiguous()
    else:
        U, E = None, torch.zeros((count, 1), device=dev, dtype=torch.float64)
    v0 = torch.randn(count, b, device=dev, dtype=torch.float64, generator=g)
    v0 /= v0.norm(dim=1, keepdim=True)
    eta = torch.empty(count, device=dev, dtype=torch.float64)
    bad = torch.zeros(count, device=dev, dtype=torch.int32)
    K.power_stepsize(Kbb, U, E, rho, v0, 1e-2, 10, eta, bad)

    def Pd(x):  # P^{-1/2} x
        y = x * rho.rsqrt()[:, None]
        if r:
            y = y + torch.bmm(U, (E * torch.bmm(U.transpose(1, 2), x[:, :, None])[:, :, 0])
                              [:, :, None])[:, :, 0]
        return y

    v, Kd = v0.clone(), Kbb.double()
    for _ in range(10):
        w = Pd(v)
        y = Pd(torch.bmm(Kd, w[:, :, None])[:, :, 0] + 1e-2 * w)
        est = (v * y).sum(1)
        v = y / y.norm(dim=1, keepdim=True)
    torch.cuda.synchronize()
    assert int(bad.abs().sum()) == 0
    assert torch.allclose(eta, 1 / est, rtol=1e-7, atol=0)
