"""The fused Phase IV launch (sap_block_step / sap_woodbury_apply, csrc/phase4.cu)
and the next-operand pass inside the block-row kernel (sap_krows_tc_next),
through the C ABI.

* the Woodbury apply D = (g - U Mc U^T g) / rho against numpy fp64 with the
  reference's Cholesky form (randnla.py:109-134);
* the fused gradient equals the unfused chain (tc_reduce + sap_grad_gather)
  bit for bit, and the lazy update equals sap_pq_update's arithmetic;
* the operand the block-row kernel streams for the next iterate equals the
  stand-alone pass bit for bit;
* a block-row update that leaves the operand's scale triggers the in-launch
  rebuild, which again equals the stand-alone pass bit for bit;
* the solver with the fused step follows the unfused solver's trajectory.
"""

import ctypes
import os

import numpy as np
import pytest
import scipy.linalg as sla
import torch

pytestmark = pytest.mark.gpu

import paper_2505_13723_b200 as sap  # noqa: E402
from paper_2505_13723_b200 import _native as nat  # noqa: E402
from paper_2505_13723_b200.kernels import ZOperand, krows_tc, krows_tc_partials  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def dev():
    return torch.device("cuda", 0)


def ws_for(b, r, m):
    return torch.zeros(nat.load().sap_block_step_workspace(b, r, m) // 8 + 1,
                       dtype=torch.float64, device=dev())


def nystrom_core(rng, b, r, rho):
    U, _ = np.linalg.qr(rng.standard_normal((b, r)))
    S = np.sort(rng.uniform(0.5, 50.0, r))[::-1]
    Mc = np.linalg.inv(rho * np.diag(1.0 / S) + U.T @ U)
    return U, S, Mc


@pytest.mark.parametrize("b,r,m", [(2000, 100, 65), (200, 50, 9), (37, 5, 3), (5000, 100, 65)])
def test_woodbury_apply_matches_reference_form(b, r, m):
    rng = np.random.default_rng(b + r)
    rho = 0.37
    U, S, Mc = nystrom_core(rng, b, r, rho)
    g = rng.standard_normal((b, m))
    # the reference's form: L = chol(rho S^-1 + U^T U); D = (g - U cho_solve(L, U^T g)) / rho
    L = sla.cho_factor(rho * np.diag(1.0 / S) + U.T @ U)
    ref = (g - U @ sla.cho_solve(L, U.T @ g)) / rho
    d = dev()
    Ud = torch.as_tensor(U, device=d).contiguous()
    UMc = torch.as_tensor(U @ Mc, device=d).contiguous()
    gd = torch.as_tensor(g, device=d).contiguous()
    rho_d = torch.tensor([rho], dtype=torch.float64, device=d)
    D = torch.empty((b, m), dtype=torch.float64, device=d)
    ws = ws_for(b, r, m)
    nat.call("sap_woodbury_apply", nat.ptr(Ud), nat.ptr(UMc), r, b, r, nat.ptr(gd), m, m,
             nat.ptr(rho_d), nat.ptr(D), m, nat.ptr(ws), ws.numel() * 8, nat.stream_handle())
    got = D.cpu().numpy()
    assert np.abs(got - ref).max() / np.abs(ref).max() < 1e-12
    # bitwise run-to-run determinism (fixed-order reductions, no atomics)
    D2 = torch.empty_like(D)
    nat.call("sap_woodbury_apply", nat.ptr(Ud), nat.ptr(UMc), r, b, r, nat.ptr(gd), m, m,
             nat.ptr(rho_d), nat.ptr(D2), m, nat.ptr(ws), ws.numel() * 8, nat.stream_handle())
    assert torch.equal(D, D2)


def _problem(n=20000, d=9, fam="matern32", m=65, b=1000, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    o = sap.KernelOracle(sap.KernelSpec(fam, np.full(d, 3.0), 1.0), X, 1e-2, device=0)
    ld = (n + 3) // 4 * 4
    P = torch.zeros((m, ld), dtype=torch.float32, device=dev())
    Q = torch.zeros_like(P)
    Y = torch.zeros_like(P)
    P[:, :n] = torch.as_tensor(rng.standard_normal((m, n)), device=dev())
    Q[:, :n] = torch.as_tensor(rng.standard_normal((m, n)), device=dev())
    Y[:, :n] = torch.as_tensor(rng.standard_normal((m, n)), device=dev())
    B = np.sort(rng.choice(n, b, replace=False))
    return o, P, Q, Y, B, rng


def bounds(A, nz):
    out = torch.zeros(nz, dtype=torch.float32, device=dev())
    nat.call("sap_colabsmax", nat.ptr(A), A.stride(0), A.shape[1], A.shape[0], nat.ptr(out),
             nat.stream_handle())
    return out


@pytest.mark.parametrize("n,m,side", [(20000, 65, "1"), (20000, 65, None), (400000, 9, "1")])
def test_next_operand_and_fused_gradient_match_unfused_passes(n, m, side, monkeypatch):
    """side "1" forces the block-row kernel's side job (short columns per CTA:
    the flat loop at n = 2e4; long ones: the column loop at n = 4e5); None
    lets the launcher choose (here the separate pass)."""
    if side is None:
        monkeypatch.delenv("SAP_ZNEXT_SIDE", raising=False)
    else:
        monkeypatch.setenv("SAP_ZNEXT_SIDE", side)
    o, P, Q, Y, B, rng = _problem(n=n, m=m)
    n, m, b = o.n, P.shape[0], B.size
    d = dev()
    tcp = o.tc_points()
    zop = ZOperand(m, n, d)
    Pb, Qb = bounds(P[:, :n], zop.nz), bounds(Q[:, :n], zop.nz)
    zp, zq, zq1 = 0.7071, -0.31, -0.29
    zop.fill(P, Q, zp, zq, Pb, Qb)
    Bd = torch.as_tensor(B, device=d)
    RAg = tcp.gather_rows(Bd)
    ws = torch.empty(nat.load().sap_krows_tc_workspace(b, m, n) // 4 + 1, dtype=torch.float32,
                     device=d)
    zn = ZOperand(m, n, d)
    splits = krows_tc_partials(o.spec, tcp, RAg, b, Bd, zop, ws,
                               (P, Q, zp, zq1, Pb, Qb, zn))
    # the operand streamed by the block-row kernel == the stand-alone pass
    ref = ZOperand(m, n, d).fill(P, Q, zp, zq1, Pb, Qb)
    assert torch.equal(zn.hi, ref.hi) and torch.equal(zn.lo, ref.lo)
    assert torch.equal(zn.scale, ref.scale)
    # fused GRAD == tc_reduce + sap_grad_gather, bit for bit
    a = nat.StepArgs()
    a.part, a.splits, a.variance, a.zscale = nat.ptr(ws), splits, 1.0, nat.ptr(zop.scale)
    loc = Bd.clone()
    a.P, a.Q, a.Y, a.ldp, a.zp, a.zq, a.lam = nat.ptr(P), nat.ptr(Q), nat.ptr(Y), P.stride(0), \
        zp, zq, 1e-2
    a.loc, a.b, a.m = nat.ptr(loc), b, m
    g = torch.empty((b, m), dtype=torch.float64, device=d)
    a.g, a.ldgo = nat.ptr(g), m
    pws = ws_for(b, 0, m)
    nat.check(nat.load().sap_block_step(ctypes.byref(a), nat.STEP_GRAD, nat.ptr(pws),
                                        pws.numel() * 8, nat.stream_handle()))
    G = torch.empty((b, m), dtype=torch.float32, device=d)
    krows_tc(o.spec, tcp, RAg, b, Bd, zop, G)
    g_ref = torch.empty_like(g)
    nat.call("sap_grad_gather", nat.ptr(G), m, nat.ptr(P), nat.ptr(Q), nat.ptr(Y), P.stride(0),
             zp, zq, nat.ptr(loc), b, m, 1e-2, nat.ptr(g_ref), m, nat.stream_handle())
    assert torch.equal(g, g_ref)


def _apply_args(P, Q, Y, loc, b, m, g, eta, e0, e1, WB, Pb, Qb, zn, zp, zq, zp1, zq1, zflag, fi,
                n, U=None, UMc=None, r=0):
    a = nat.StepArgs()
    a.P, a.Q, a.Y, a.ldp, a.zp, a.zq, a.lam = nat.ptr(P), nat.ptr(Q), nat.ptr(Y), P.stride(0), \
        zp, zq, 1e-2
    a.loc, a.b, a.m, a.g, a.ldgo = nat.ptr(loc), b, m, nat.ptr(g), m
    if r:
        a.U, a.UMc, a.ldu, a.r = nat.ptr(U), nat.ptr(UMc), r, r
    a.Pw, a.Qw, a.eta_dev, a.e0, a.e1 = nat.ptr(P), nat.ptr(Q), nat.ptr(eta), e0, e1
    a.WB, a.ldwb, a.Pb, a.Qb = nat.ptr(WB), m, nat.ptr(Pb), nat.ptr(Qb)
    if zn is not None:
        a.Zhi_next, a.Zlo_next, a.ldz, a.zscale_next = nat.ptr(zn.hi), nat.ptr(zn.lo), zn.ldz, \
            nat.ptr(zn.scale)
        a.zp1, a.zq1, a.zflag, a.flag_idx, a.n_local = zp1, zq1, nat.ptr(zflag), fi, n
    return a


@pytest.mark.parametrize("blowup", [False, True])
def test_apply_update_and_next_operand(blowup):
    """APPLY with the Woodbury core: D, the lazy update (sap_pq_update's
    arithmetic), and the next operand's block rows; with ``blowup`` the
    updated rows leave the operand's scale and the launch rebuilds it."""
    o, P, Q, Y, B, rng = _problem(n=30000, b=600, seed=3)
    n, m, b, r = o.n, P.shape[0], B.size, 40
    d = dev()
    rho = 0.2
    U, S, Mc = nystrom_core(rng, b, r, rho)
    scale = 1e4 if blowup else 1.0
    g_h = scale * rng.standard_normal((b, m))
    g = torch.as_tensor(g_h, device=d).contiguous()
    Ud = torch.as_tensor(U, device=d).contiguous()
    UMc = torch.as_tensor(U @ Mc, device=d).contiguous()
    loc = torch.as_tensor(B, device=d)
    eta = torch.tensor([0.9 / rho], dtype=torch.float64, device=d)
    zp, zq, zp1, zq1, e0, e1 = 0.7071, -0.31, 0.7071, -0.29, -0.4, 1.3
    zop_nz = (m + 15) // 16 * 16
    Pb, Qb = bounds(P[:, :n], zop_nz), bounds(Q[:, :n], zop_nz)
    zn = ZOperand(m, n, d).fill(P, Q, zp1, zq1, Pb, Qb)  # what the block-row kernel left
    P0, Q0 = P.clone(), Q.clone()
    Pb0, Qb0 = Pb.clone(), Qb.clone()
    WB = torch.zeros((b, m), dtype=torch.float32, device=d)
    zflag = torch.zeros(2, dtype=torch.int32, device=d)
    a = _apply_args(P, Q, Y, loc, b, m, g, eta, e0, e1, WB, Pb, Qb, zn, zp, zq, zp1, zq1, zflag,
                    0, n, Ud, UMc, r)
    ws = ws_for(b, r, m)
    nat.check(nat.load().sap_block_step(ctypes.byref(a), nat.STEP_APPLY, nat.ptr(ws),
                                        ws.numel() * 8, nat.stream_handle()))
    torch.cuda.synchronize()
    assert int(zflag[0]) == (1 if blowup else 0)
    # D and the update in fp64 (numpy), cast like the kernel
    D = g_h - (U @ Mc) @ (U.T @ g_h)
    et = float(eta)
    p0 = P0[:, B].T.double().cpu().numpy()
    q0 = Q0[:, B].T.double().cpu().numpy()
    pn = (p0 + e0 * et * D).astype(np.float32)
    qn = (q0 + e1 * et * D).astype(np.float32)
    wb = (zp * p0 + zq * q0 - et * D).astype(np.float32)
    got_p = P[:, B].T.cpu().numpy()
    got_q = Q[:, B].T.cpu().numpy()
    tol = 2e-6
    assert np.abs(got_p - pn).max() <= tol * np.abs(pn).max()
    assert np.abs(got_q - qn).max() <= tol * np.abs(qn).max()
    assert np.abs(WB.cpu().numpy() - wb).max() <= tol * np.abs(wb).max()
    # rows outside the block untouched
    mask = np.ones(n, bool)
    mask[B] = False
    assert torch.equal(P[:, :n][:, torch.as_tensor(mask, device=d)],
                       P0[:, :n][:, torch.as_tensor(mask, device=d)])
    # bounds cover the state
    assert bool((bounds(P[:, :n], zop_nz)[:m] <= Pb[:m]).all())
    assert bool((bounds(Q[:, :n], zop_nz)[:m] <= Qb[:m]).all())
    # the next operand: block rows patched (and rebuilt when the scale was
    # left) == a stand-alone pass over the updated state
    if blowup:  # rebuilt in the launch from the raised bounds
        ref = ZOperand(m, n, d).fill(P, Q, zp1, zq1, Pb, Qb)
    else:  # off-block rows as streamed, block rows patched, at the old scale
        ref = ZOperand(m, n, d).fill(P, Q, zp1, zq1, Pb0, Qb0)
    assert torch.equal(zn.scale, ref.scale)
    assert torch.equal(zn.hi, ref.hi) and torch.equal(zn.lo, ref.lo)


@pytest.mark.parametrize("fam", ["matern32", "rbf"])
def test_fused_solver_follows_unfused(fam, monkeypatch):
    rng = np.random.default_rng(11)
    n, d, m = 40000, 9, 17
    X = rng.standard_normal((n, d))
    Y = rng.standard_normal((n, m))
    spec = sap.KernelSpec(fam, np.full(d, 3.0), 1.0)
    cfg = sap.RunConfig(lam=1e-2, blocksize=512, nystrom_rank=64, max_iters=120,
                        residual_every=0, seed=5)
    out = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("SAP_FUSED_STEP", fused)
        o = sap.KernelOracle(spec, X, 1e-2, device=0)
        out[fused] = sap.adasap_solve(o, Y, cfg)
    a, b = out["1"], out["0"]
    assert [r.block_hash for r in a.trace.records] == [r.block_hash for r in b.trace.records]
    # the paths differ only in rounding: the next operand's fp16 split uses the
    # scale of the pre-update bounds (fused) or the post-update ones (unfused),
    # and the r-term sums run in another order; ~1e-6 per product, grown by the
    # iteration (measured 1.1e-5 for RBF after 120 iterations) -- well inside
    # the block-product bar of 1e-4
    assert np.abs(a.W - b.W).max() / np.abs(b.W).max() < 1e-4


def test_shapes_outside_the_fused_step_fall_back():
    """m > 128 right-hand sides: the fused Phase IV (and the tensor-core
    product) do not apply; the solver takes the unfused kernels and still
    follows the oracle."""
    from oracle import sapgp_oracle as orc
    rng = np.random.default_rng(9)
    n, d, m = 2500, 5, 130
    X = rng.standard_normal((n, d))
    Y = rng.standard_normal((n, m))
    assert not nat.load().sap_block_step_supported(256, 32, m)
    o = sap.KernelOracle(sap.KernelSpec("rbf", np.full(d, 1.5), 1.0), X, 1e-1, device=0)
    cfg = sap.RunConfig(lam=1e-1, blocksize=256, nystrom_rank=32, max_iters=10, residual_every=0,
                        seed=2)
    res = sap.adasap_solve(o, Y, cfg)
    Wref, etas, crcs, _ = orc.adasap_solve(orc.Points("rbf", np.full(d, 1.5), 1.0, X), 1e-1, Y,
                                           10, 2, 256, 32)
    assert [r.block_hash for r in res.trace.records] == list(crcs)
    assert np.abs(res.W - Wref).max() / np.abs(Wref).max() < 1e-3
