"""Kernel families and matrix-free block access to K = k(X, X) on a B200.

Drop-in mirror of the reference ``sapgp.kernels`` (kernels.py:1-221): the
same ``KernelSpec`` / ``KernelOracle`` names, argument meaning and errors,
but the oracle keeps its points resident in HBM and every product runs in
``libsapgp_b200.so``:

* points are pre-scaled by 1/lengthscale and their squared norms formed
  once, in fp64, then stored as fp32 rows padded to 4/8/12/16/32/64 floats
  (kernels.py:45-53, :100-112);
* ``tile``/``block``/``dense`` -> ``sap_ktile`` (kernels.py:118-143);
* ``matmul`` / ``cross_matmul`` / block-row products -> ``sap_krows_times``
  (kernels.py:145-176, dist.py:108-147).

Arithmetic is fp32 with fixed-order reductions (the reference is fp64):
block products agree with the reference to ~1e-6 relative, well inside the
1e-4 parity bound of BASELINE.json. Numpy inputs return numpy float64
outputs (fresh arrays, like the reference); CUDA tensor inputs return CUDA
tensors.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from . import xfer
from .errors import ContractError, ValidationError

FAMILIES = ("rbf", "matern32", "matern52")
DENSE_LIMIT = 4096
PADDED_DIMS = (4, 8, 12, 16, 32, 64)


@dataclass(frozen=True)
class KernelSpec:
    """Family, ARD lengthscales and variance (kernels.py:25-42)."""

    family: str
    lengthscales: np.ndarray
    variance: float = 1.0

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ContractError(f"unknown kernel family {self.family!r}")
        ls = np.atleast_1d(np.asarray(self.lengthscales, dtype=np.float64))
        if ls.ndim != 1 or not np.all(np.isfinite(ls)) or np.any(ls <= 0.0):
            raise ContractError("lengthscales must be positive finite reals")
        if not np.isfinite(self.variance) or self.variance <= 0.0:
            raise ContractError("variance must be positive")
        object.__setattr__(self, "lengthscales", ls)
        object.__setattr__(self, "variance", float(self.variance))

    @property
    def code(self):
        return nat.FAMILY_CODES[self.family]


def padded_dim(d):
    for dp in PADDED_DIMS:
        if d <= dp:
            return dp
    raise ContractError(f"d={d} exceeds the supported maximum of 64 features")


def _device(device):
    nat.require_cuda()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    if dev.type != "cuda":
        raise ContractError("the B200 oracle lives on a CUDA device")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


class DevicePoints:
    """Pre-scaled fp32 points + fp32 squared norms resident on one device."""

    def __init__(self, spec, X, device):
        X = np.asarray(X, dtype=np.float64) if not torch.is_tensor(X) else X
        if X.ndim != 2:
            raise ContractError("points must form a 2-d array")
        n, d = X.shape
        ls = spec.lengthscales
        if ls.size not in (1, d):
            raise ContractError(f"lengthscales of size {ls.size} do not match d={d}")
        self.n, self.d, self.ldx = n, d, padded_dim(d)
        self.device = device
        inv = np.broadcast_to(1.0 / ls, (d,)).astype(np.float64)
        Xd = torch.as_tensor(X, dtype=torch.float64).to(device).contiguous()
        inv_d = torch.as_tensor(inv.copy(), device=device)
        self.Xs = torch.empty((max(n, 1), self.ldx), dtype=torch.float32, device=device)
        self.sqn = torch.empty(max(n, 1), dtype=torch.float32, device=device)
        with torch.cuda.device(device):
            nat.call("sap_prepare_points", nat.ptr(Xd), n, d, nat.ptr(inv_d), nat.ptr(self.Xs),
                     self.ldx, nat.ptr(self.sqn), nat.stream_handle())

    def gather(self, idx_dev, base=0, out=None):
        """Rows idx (global ids, minus ``base``) as a new DevicePoints-like pair."""
        b = idx_dev.numel()
        Rs = torch.empty((b, self.ldx), dtype=torch.float32, device=self.device) if out is None \
            else out[0]
        rsq = torch.empty(b, dtype=torch.float32, device=self.device) if out is None else out[1]
        nat.call("sap_gather_points", nat.ptr(self.Xs), nat.ptr(self.sqn), self.ldx,
                 nat.ptr(idx_dev), b, base, nat.ptr(Rs), nat.ptr(rsq), nat.stream_handle())
        return Rs, rsq


def krows_times(spec, cols, Rs, rsq, row_ids, R, out, col_ids=None, col_base=0, R2=None,
                ca=1.0, cb=0.0, accumulate=False, ws=None, ncols=None, col_offset=0):
    """out (b x m fp32) = variance * K(rows, cols) @ (ca*R + cb*R2).

    ``R``/``R2`` are column-major (m x ld) fp32 device tensors whose columns
    index the column points; ``col_offset`` selects a contiguous sub-range of
    the column point set (a shard)."""
    b = Rs.shape[0]
    m = R.shape[0]
    nc = cols.n - col_offset if ncols is None else ncols
    need = nat.load().sap_krows_workspace(b, m, nc)
    if need and (ws is None or ws.numel() * ws.element_size() < need):
        ws = torch.empty(need // 4 + 1, dtype=torch.float32, device=cols.device)
    Xs = cols.Xs[col_offset:] if col_offset else cols.Xs
    sq = cols.sqn[col_offset:] if col_offset else cols.sqn
    nat.call("sap_krows_times", nat.ptr(Xs), nat.ptr(sq), cols.ldx, nc, nat.ptr(col_ids), col_base,
             nat.ptr(Rs), nat.ptr(rsq), nat.ptr(row_ids), b, cols.d, nat.ptr(R), nat.ptr(R2),
             R.stride(0), m, ca, cb, spec.code, spec.variance, nat.ptr(out), out.stride(0),
             int(accumulate), nat.ptr(ws), 0 if ws is None else ws.numel() * 4,
             nat.stream_handle())
    return out


_LOG2E = 1.4426950408889634
# c_fam of the augmented features (krows_tc.cu, sap_tc_points): z = x sqrt(c) / l
_CFAM = {"rbf": 0.5 * _LOG2E, "matern32": 3.0 * _LOG2E ** 2, "matern52": 5.0 * _LOG2E ** 2}


class TcPoints:
    """Augmented features of the tensor-core path (krows_tc.cu): row form RA
    for every point (rows are gathered per block) and column form CA for the
    points of one shard [lo, hi)."""

    def __init__(self, spec, X, device, lo=0, hi=None, with_rows=True):
        Xd = torch.as_tensor(np.asarray(X, dtype=np.float64) if not torch.is_tensor(X) else X,
                             dtype=torch.float64).to(device).contiguous()
        n, d = Xd.shape
        hi = n if hi is None else hi
        feats = 3 * d + 4 + (1 if spec.family == "rbf" else 0)  # krows_tc.cu tc_features
        self.ka = 32 if feats <= 32 else 64
        if feats > 64:
            raise ContractError(f"tensor-core path supports d <= 19 (got d={d})")
        inv = torch.as_tensor(np.broadcast_to(1.0 / spec.lengthscales, (d,)).copy(), device=device)
        self._ls, self._family = spec.lengthscales, spec.family
        # with_rows=False: column features of [lo, hi) only (a shard's columns
        # for a one-off product); gather_rows is then unavailable
        self.RA = torch.empty((max(n, 1) if with_rows else 1, self.ka), dtype=torch.float32,
                              device=device)
        self.CA = torch.empty((max(hi - lo, 1), self.ka), dtype=torch.float32, device=device)
        with torch.cuda.device(device):
            if with_rows:
                nat.call("sap_tc_points", nat.ptr(Xd), n, d, nat.ptr(inv), spec.code, self.ka,
                         nat.ptr(self.RA), None, nat.stream_handle())
            if hi > lo:
                nat.call("sap_tc_points", nat.ptr(Xd[lo:hi]), hi - lo, d, nat.ptr(inv), spec.code,
                         self.ka, None, nat.ptr(self.CA), nat.stream_handle())
        self.lo, self.hi, self.n, self.d, self.device = lo, hi, n, d, device
        self.code = spec.code
        # fp16 features (GEMM1 kind::f16 at twice the tf32 rate, half the bytes):
        # the features are tf32-rounded splits, so the fp16 copy is exact while
        # every magnitude stays inside fp16's range (|z|^2 < 2^14 leaves room
        # for the -2 z column form); SAP_TC_F16=0 keeps fp32
        # (d >= 10 needs 64 features: fp16 too, 128-byte rows, since round 2)
        xfer.mark("tc points: features")
        self.half = False
        if os.environ.get("SAP_TC_F16", "1") == "1":
            zmax2 = _CFAM[spec.family] * float(((Xd * inv) ** 2).sum(1).max())
            self.half = zmax2 < 2.0 ** 14
        self.ka_code = ((nat.SAP_TC_KA_F16 if self.ka == 32 else nat.SAP_TC_KA_F16X64)
                        if self.half else self.ka)
        self.dtype = torch.float16 if self.half else torch.float32
        xfer.mark("tc points: range check")
        if self.half:
            self.CA = self.CA.half()

    def fits_half(self, Xs):
        """True when external points (test points) keep their features in fp16 range."""
        if not self.half:
            return True
        Xs = torch.as_tensor(Xs, dtype=torch.float64, device=self.device)
        inv = torch.as_tensor(np.broadcast_to(1.0 / self._ls, (self.d,)).copy(),
                              device=self.device)
        return _CFAM[self._family] * float(((Xs * inv) ** 2).sum(1).max()) < 2.0 ** 14

    def _scratch(self, rows):
        # fp32 staging for the gathers when the kernel reads fp16 features: a
        # fresh (stream-ordered, caching-allocator) buffer per call, since the
        # lookahead's producer threads gather concurrently
        return torch.empty((rows, self.ka), dtype=torch.float32, device=self.device)

    def gather_cols(self, idx_dev, out=None):
        """Column-form features of the points idx (any ids, not only this shard),
        in the kernel's feature dtype."""
        b = idx_dev.numel()
        if out is None:
            out = torch.empty((b, self.ka), dtype=self.dtype, device=self.device)
        dst = self._scratch(out.shape[0]) if self.half else out
        nat.call("sap_tc_gather_cols", nat.ptr(self.RA), self.ka, self.d, self.code,
                 nat.ptr(idx_dev), b, dst.shape[0], nat.ptr(dst), nat.stream_handle())
        if self.half:
            out.copy_(dst)
        return out

    def gather_rows_batch(self, idx2d, out):
        """Row-form features of a batch of blocks (idx2d: (count, b)) into
        out[:, :b] ((count, bpad, ka) in the kernel's dtype; the pad rows
        b..bpad are the caller's, zero): one gather and one copy per batch."""
        count, b = idx2d.shape
        dst = self._scratch(count * b)
        nat.call("sap_tc_gather_rows", nat.ptr(self.RA), self.ka, nat.ptr(idx2d), count * b,
                 count * b, nat.ptr(dst), nat.stream_handle())
        out[:, :b].copy_(dst.view(count, b, self.ka))
        return out

    def gather_rows(self, idx_dev, out=None):
        b = idx_dev.numel()
        bpad = (b + 255) // 256 * 256  # whole 256-row tiles of the CTA-pair kernel
        if out is None:
            out = torch.empty((bpad, self.ka), dtype=self.dtype, device=self.device)
        dst = self._scratch(out.shape[0]) if self.half else out
        nat.call("sap_tc_gather_rows", nat.ptr(self.RA), self.ka, nat.ptr(idx_dev), b, bpad,
                 nat.ptr(dst), nat.stream_handle())
        if self.half:
            out.copy_(dst)
        return out


class ZOperand:
    """fp16 hi/lo split of a (scaled) RHS in the tensor-core B layout [nz][ldz]."""

    def __init__(self, m, n, device):
        self.m, self.n = m, n
        self.nz = (m + 15) // 16 * 16  # MMA N granularity of the CTA pair
        if self.nz > 128:
            raise ContractError("tensor-core path supports at most 128 right-hand sides")
        self.ldz = max(8, (n + 7) // 8 * 8)
        # rows m..nz-1 are MMA padding: zeroed here once, never rewritten
        self.hi = torch.zeros((self.nz, self.ldz), dtype=torch.float16, device=device)
        self.lo = torch.zeros((self.nz, self.ldz), dtype=torch.float16, device=device)
        self.scale = torch.ones(self.nz, dtype=torch.float32, device=device)
        self.bound = torch.zeros(self.nz, dtype=torch.float32, device=device)

    def fill(self, P, Q=None, zp=1.0, zq=0.0, Pb=None, Qb=None):
        """Z = zp P + zq Q (column-major fp32, m x ld); bounds computed if not given."""
        if Pb is None:
            nat.call("sap_colabsmax", nat.ptr(P), P.stride(0), self.n, self.m, nat.ptr(self.bound),
                     nat.stream_handle())
            Pb, Q, Qb, zq = self.bound, None, None, 0.0
        nat.call("sap_z_operand", nat.ptr(P), nat.ptr(Q), P.stride(0), self.n, self.m, zp, zq,
                 nat.ptr(Pb), nat.ptr(Qb), self.nz, self.ldz, nat.ptr(self.hi), nat.ptr(self.lo),
                 nat.ptr(self.scale), nat.stream_handle())
        return self


def krows_tc(spec, tcp, RAg, b, row_ids, zop, out, ws=None, accumulate=False, cols=None):
    """out (b x m fp32) = variance * K(rows, shard columns) @ Z on the tensor cores.
    ``cols`` = (CA, col_base) replaces the shard's column features (e.g. a
    gathered block, with row_ids given as positions in it)."""
    CA, col_base = (tcp.CA, tcp.lo) if cols is None else cols
    ncols = (tcp.hi - tcp.lo) if cols is None else CA.shape[0]
    need = nat.load().sap_krows_tc_workspace(b, zop.m, ncols)
    if ws is None or ws.numel() * 4 < need:
        ws = torch.empty(need // 4 + 1, dtype=torch.float32, device=tcp.device)
    if RAg.dtype != tcp.dtype or CA.dtype != tcp.dtype:
        raise ContractError("tensor-core features must be in the point set's dtype")
    nat.call("sap_krows_tc", nat.ptr(CA), ncols, tcp.ka_code, nat.ptr(RAg), RAg.shape[0],
             nat.ptr(row_ids), b, col_base, nat.ptr(zop.hi), nat.ptr(zop.lo), zop.nz, zop.ldz,
             nat.ptr(zop.scale), zop.m, spec.code, spec.variance, nat.ptr(out), out.stride(0),
             int(accumulate), nat.ptr(ws), ws.numel() * 4, nat.stream_handle())
    return out


def krows_tc_partials(spec, tcp, RAg, b, row_ids, zop, ws, nxt=None):
    """The block-row product's unreduced partials ([splits][m][b] in ``ws``,
    reduced by the fused Phase IV kernel, sap_block_step) and, with
    ``nxt = (P, Q, zp, zq, Pb, Qb, zop_next)``, the next iterate's operand
    Z_{t+1} = zp P + zq Q filled into ``zop_next`` inside the same kernel.
    Returns the split count."""
    CA, col_base, ncols = tcp.CA, tcp.lo, tcp.hi - tcp.lo
    need = nat.load().sap_krows_tc_workspace(b, zop.m, ncols)
    if ws.numel() * ws.element_size() < need:
        raise ContractError("block-row workspace too small")
    if nxt is not None:
        P, Q, zp, zq, Pb, Qb, zn = nxt
        extra = (nat.ptr(P), nat.ptr(Q), P.stride(0), zp, zq, nat.ptr(Pb), nat.ptr(Qb),
                 nat.ptr(zn.hi), nat.ptr(zn.lo), nat.ptr(zn.scale))
    else:
        extra = (None, None, 0, 0.0, 0.0, None, None, None, None, None)
    splits = ctypes.c_int(0)
    nat.call("sap_krows_tc_next", nat.ptr(CA), ncols, tcp.ka_code, nat.ptr(RAg), RAg.shape[0],
             nat.ptr(row_ids), b, col_base, nat.ptr(zop.hi), nat.ptr(zop.lo), zop.nz, zop.ldz,
             nat.ptr(zop.scale), zop.m, spec.code, spec.variance, None, zop.m, 0, nat.ptr(ws),
             ws.numel() * ws.element_size(), 0, ctypes.byref(splits), *extra,
             nat.stream_handle())
    return splits.value


def ktile_f32(spec, A, asq, aid, C, csq, cid, ldx, d, out):
    """fp32 K(A, C) into ``out`` (same values as ktile, half the bytes)."""
    nat.call("sap_ktile_f32", nat.ptr(A), nat.ptr(asq), nat.ptr(aid), A.shape[0], nat.ptr(C),
             nat.ptr(csq), nat.ptr(cid), C.shape[0], ldx, d, spec.code, spec.variance,
             nat.ptr(out), out.stride(0), nat.stream_handle())
    return out


def ktile_f32_batch(spec, X, xsq, d, out):
    """K_BB of each block in a batch (X: (count, b, ldx), xsq: (count, b)) into
    out (count, b, ldo) fp32 in one launch: ktile_f32's values, bit for bit."""
    count, b, ldx = X.shape
    nat.call("sap_ktile_f32_batch", nat.ptr(X), X.stride(0), nat.ptr(xsq), xsq.stride(0), b,
             count, ldx, d, spec.code, spec.variance, nat.ptr(out), out.stride(1), out.stride(0),
             nat.stream_handle())
    return out


def ktile_f32_batch_split(spec, X, xsq, d, out, outh, outl):
    """ktile_f32_batch, plus K / variance as fp16 hi + lo into outh / outl
    ((count, b, ldh) each): the three-pass tensor-core sketch's operands."""
    count, b, ldx = X.shape
    nat.call("sap_ktile_f32_batch_split", nat.ptr(X), X.stride(0), nat.ptr(xsq), xsq.stride(0), b,
             count, ldx, d, spec.code, spec.variance, nat.ptr(out), out.stride(1), out.stride(0),
             nat.ptr(outh), nat.ptr(outl), outh.stride(1), outh.stride(0), nat.stream_handle())
    return out


def power_stepsize(Kbb, U, E, rho, v0, lam, iters, eta, bad):
    """Batched preconditioned power iteration (randnla.py:165-196) over the
    leading ``Kbb.shape[0]`` problems: eta[q] = 1/(v.Hv), bad[q] |= failure."""
    count, b = Kbb.shape[0], Kbb.shape[1]
    r = 0 if U is None else U.shape[2]
    nat.call("sap_power_stepsize", nat.ptr(Kbb), Kbb.stride(1), Kbb.stride(0),
             nat.ptr(U) if r else None, U.stride(0) if r else 0, r, nat.ptr(E) if r else None,
             nat.ptr(rho), nat.ptr(v0), b, count, lam, iters, nat.ptr(eta), nat.ptr(bad),
             nat.stream_handle())


def ktile(spec, A, asq, aid, C, csq, cid, ldx, d):
    out = torch.empty((A.shape[0], C.shape[0]), dtype=torch.float64, device=A.device)
    nat.call("sap_ktile", nat.ptr(A), nat.ptr(asq), nat.ptr(aid), A.shape[0], nat.ptr(C),
             nat.ptr(csq), nat.ptr(cid), C.shape[0], ldx, d, spec.code, spec.variance,
             nat.ptr(out), out.stride(0), nat.stream_handle())
    return out


def to_colmajor(M, n, device, ld=None):
    """(n x m) host/device matrix -> (m x ld) fp32 device tensor (column-major).
    A CUDA fp32 (n x m) view of a column-major (m x n) buffer with ld == n is
    adopted without a copy (large right-hand sides built in place)."""
    if torch.is_tensor(M) and M.is_cuda and M.dtype == torch.float32 and M.ndim == 2 and \
            M.shape[0] == n and M.stride(0) == 1 and M.stride(1) == n and \
            (ld is None or ld == n) and torch.device(device) == M.device:
        return M.T
    if torch.is_tensor(M):
        Mt = M.to(device=device, dtype=torch.float32)
    else:
        Mt = xfer.upload(np.asarray(M, dtype=np.float64), torch.float32, device)
    if Mt.ndim == 1:
        Mt = Mt[:, None]
    if Mt.shape[0] != n:
        raise ContractError("matrix must have one row per point")
    ld = n if ld is None else ld
    out = torch.zeros((Mt.shape[1], max(ld, 1)), dtype=torch.float32, device=device)
    out[:, :n] = Mt.T
    return out


def _finish(t, like_numpy, vector):
    t = t[:, 0] if vector else t
    if like_numpy:
        return t.to(torch.float64).cpu().numpy()
    return t


class KernelOracle:
    """Lazy evaluator of K = k(X, X) with points resident in HBM
    (kernels.py:94-176). ``lam`` is housed here for products with K + lam I."""

    def __init__(self, spec, X, lam, device=None):
        is_t = torch.is_tensor(X)
        Xn = X if is_t else np.ascontiguousarray(np.asarray(X, dtype=np.float64))
        if Xn.ndim != 2 or Xn.shape[0] < 1:
            raise ContractError("X must be a non-empty 2-d array")
        if not lam > 0.0:
            raise ContractError("likelihood variance lam must be positive")
        self.spec = spec
        self.X = Xn
        self.lam = float(lam)
        self.device = _device(device)
        # one host->device copy of X (fp64); the FFMA and tensor-core point
        # formats are both derived from it on the device
        if is_t:
            self._Xd = Xn.to(device=self.device, dtype=torch.float64).contiguous()
        else:
            self._Xd = xfer.upload(Xn, torch.float64, self.device)
        xfer.mark("oracle: X upload")
        # the reference's finiteness check (kernels.py:100-112), on the device
        # copy: np.isfinite over a 10^6 x 9 host array alone took ~10 ms
        if not bool(torch.isfinite(self._Xd).all()):
            raise ValidationError("non-finite training inputs")
        xfer.mark("oracle: finite check")
        self.points = DevicePoints(spec, self._Xd, self.device)
        xfer.mark("oracle: points")
        self._ws = None
        self._tc = None
        self.backend = "auto"  # "tc" (tcgen05), "ffma", or "auto" (tc when the shape fits)

    def tc_points(self, lo=0, hi=None):
        hi = self.n if hi is None else hi
        if self._tc is None or (self._tc.lo, self._tc.hi) != (lo, hi):
            self._tc = TcPoints(self.spec, self._Xd, self.device, lo, hi)
        return self._tc

    def use_tc(self, m):
        if self.backend == "ffma":
            return False
        fits = bool(nat.load().sap_tc_supported(self.d, m))
        if self.backend == "tc" and not fits:
            raise ContractError("shape outside the tensor-core path (d <= 20, m <= 128)")
        return fits

    @property
    def n(self):
        return self.points.n

    @property
    def d(self):
        return self.points.d

    # -- dense access -----------------------------------------------------
    def _ids(self, idx):
        return torch.as_tensor(np.asarray(idx, dtype=np.int64), device=self.device)

    def tile(self, rows, cols):
        """Dense K[rows, cols]; equal row/col ids give exactly the variance."""
        r, c = self._ids(rows), self._ids(cols)
        if r.numel() == 0 or c.numel() == 0:
            return np.zeros((r.numel(), c.numel()))
        if int(r.min()) < 0 or int(r.max()) >= self.n or int(c.min()) < 0 or int(c.max()) >= self.n:
            raise ContractError("tile index out of range")
        return self._tile64(r, c).cpu().numpy()

    def _tile64(self, r, c):
        """fp64 K[r, c] in the reference's arithmetic (sap_ktile64)."""
        out = torch.empty((r.numel(), c.numel()), dtype=torch.float64, device=self.device)
        inv = torch.as_tensor(np.broadcast_to(1.0 / self.spec.lengthscales, (self.d,)).copy(),
                              device=self.device)
        nat.call("sap_ktile64", nat.ptr(self._Xd), nat.ptr(inv), self.d, nat.ptr(r), r.numel(),
                 nat.ptr(c), c.numel(), self.spec.code, self.spec.variance, nat.ptr(out),
                 out.stride(0), nat.stream_handle())
        return out

    def block_device(self, block_dev):
        return self._tile64(block_dev, block_dev)

    def block(self, block):
        """Exact symmetric K[block, block] with the variance on the diagonal."""
        from .dist import check_indices
        block = check_indices(block, self.n)
        return self.block_device(self._ids(block)).cpu().numpy()

    def dense(self):
        if self.n > DENSE_LIMIT:
            raise ContractError(f"dense kernel matrix refused for n={self.n}")
        return self.block(np.arange(self.n))

    # -- products -----------------------------------------------------------
    def _workspace(self, b, m, nc):
        need = nat.load().sap_krows_workspace(b, m, nc)
        if need and (self._ws is None or self._ws.numel() * 4 < need):
            self._ws = torch.empty(need // 4 + 1, dtype=torch.float32, device=self.device)
        return self._ws

    def rows_times_device(self, block_dev, Rcm, out=None, R2=None, ca=1.0, cb=0.0):
        """K[block, :] @ R for a column-major device RHS; fp32 (b x m) out."""
        b, m = block_dev.numel(), Rcm.shape[0]
        if out is None:
            out = torch.empty((b, m), dtype=torch.float32, device=self.device)
        if self.use_tc(m) and b >= 16:
            tcp = self.tc_points()
            zop = ZOperand(m, self.n, self.device)
            if R2 is None:
                zop.fill(Rcm, zp=ca)
            else:
                b1 = torch.zeros(zop.nz, dtype=torch.float32, device=self.device)
                b2 = torch.zeros(zop.nz, dtype=torch.float32, device=self.device)
                nat.call("sap_colabsmax", nat.ptr(Rcm), Rcm.stride(0), self.n, m, nat.ptr(b1),
                         nat.stream_handle())
                nat.call("sap_colabsmax", nat.ptr(R2), R2.stride(0), self.n, m, nat.ptr(b2),
                         nat.stream_handle())
                zop.fill(Rcm, R2, ca, cb, b1, b2)
            return krows_tc(self.spec, tcp, tcp.gather_rows(block_dev), b, block_dev, zop, out)
        Rs, rsq = self.points.gather(block_dev)
        return krows_times(self.spec, self.points, Rs, rsq, block_dev, Rcm, out, R2=R2, ca=ca,
                           cb=cb, ws=self._workspace(b, m, self.n))

    def matmul(self, M):
        """K @ M without materialising K (kernels.py:145-159)."""
        vector = (M.ndim == 1)
        like_np = not torch.is_tensor(M)
        if M.shape[0] != self.n:
            raise ContractError("M must have n rows")
        Rcm = to_colmajor(M, self.n, self.device)
        ids = torch.arange(self.n, device=self.device, dtype=torch.int64)
        out = self.rows_times_device(ids, Rcm)
        return _finish(out, like_np, vector)

    def cross_matmul(self, Xstar, W):
        """k(Xstar, X) @ W -- external rows, no diagonal rule (kernels.py:161-176)."""
        vector = (W.ndim == 1)
        like_np = not torch.is_tensor(W)
        from .parallel import allreduce_sum_, current_shard
        sh = current_shard(self.n)
        if torch.is_tensor(W) and W.is_cuda and sh.world > 1 and W.shape[0] == sh.size \
                and sh.size != self.n:
            # W is this rank's shard (a device-resident solve, solvers.py): the
            # partial k(X*, X_shard) W_shard, summed over ranks (one t x m
            # all-reduce) -- no n x m gather
            return self._cross_matmul_shard(Xstar, W, sh, vector, allreduce_sum_)
        if W.shape[0] != self.n:
            raise ContractError("W must have n rows")
        star = DevicePoints(self.spec, Xstar, self.device)
        if star.d != self.d:
            raise ContractError("point dimension does not match the training inputs")
        Rcm = to_colmajor(W, self.n, self.device)
        t, m = star.n, Rcm.shape[0]
        out = torch.empty((t, m), dtype=torch.float32, device=self.device)
        if self.use_tc(m) and t >= 16 and self.tc_points().fits_half(Xstar):
            # test points as the rows of the tensor-core kernel: their row-form
            # features, zero padded to whole 256-row tiles; no row ids, so no
            # diagonal rule (kernels.py:161-176)
            tcp = self.tc_points()
            Xs64 = torch.as_tensor(np.asarray(Xstar, dtype=np.float64) if not torch.is_tensor(
                Xstar) else Xstar, dtype=torch.float64).to(self.device).contiguous()
            RAs = torch.zeros(((t + 255) // 256 * 256, tcp.ka), dtype=torch.float32,
                              device=self.device)
            inv = torch.as_tensor(np.broadcast_to(1.0 / self.spec.lengthscales,
                                                  (self.d,)).copy(), device=self.device)
            nat.call("sap_tc_points", nat.ptr(Xs64), t, self.d, nat.ptr(inv), self.spec.code,
                     tcp.ka, nat.ptr(RAs), None, nat.stream_handle())
            RAs = RAs.to(tcp.dtype)
            zop = ZOperand(m, self.n, self.device).fill(Rcm)
            krows_tc(self.spec, tcp, RAs, t, None, zop, out)
            return _finish(out, like_np, vector)
        krows_times(self.spec, self.points, star.Xs, star.sqn, None, Rcm, out,
                    ws=self._workspace(t, m, self.n))
        return _finish(out, like_np, vector)

    def star_rows(self, Xstar, m):
        """Row operands of external points: ("tc", features) or ("pts", Xs, sqn)."""
        star = DevicePoints(self.spec, Xstar, self.device)
        if star.d != self.d:
            raise ContractError("point dimension does not match the training inputs")
        t = star.n
        if self.use_tc(m) and t >= 16 and self.tc_points(*self._tc_range()).fits_half(Xstar):
            tcp = self._tc
            Xs64 = torch.as_tensor(np.asarray(Xstar, dtype=np.float64) if not torch.is_tensor(
                Xstar) else Xstar, dtype=torch.float64).to(self.device).contiguous()
            RAs = torch.zeros(((t + 255) // 256 * 256, tcp.ka), dtype=torch.float32,
                              device=self.device)
            inv = torch.as_tensor(np.broadcast_to(1.0 / self.spec.lengthscales,
                                                  (self.d,)).copy(), device=self.device)
            nat.call("sap_tc_points", nat.ptr(Xs64), t, self.d, nat.ptr(inv), self.spec.code,
                     tcp.ka, nat.ptr(RAs), None, nat.stream_handle())
            return ("tc", RAs.to(tcp.dtype)), t
        return ("pts", star.Xs, star.sqn), t

    def _tc_range(self):
        return (self._tc.lo, self._tc.hi) if self._tc is not None else (0, self.n)

    def _cross_matmul_shard(self, Xstar, W_local, sh, vector, allreduce):
        Wl = W_local[:, None] if W_local.ndim == 1 else W_local
        m = Wl.shape[1]
        Wcm = to_colmajor(Wl, sh.size, self.device)
        rows, t = self.star_rows(Xstar, m)
        out = torch.empty((t, m), dtype=torch.float32, device=self.device)
        tcp = self._tc if self._tc is not None and (self._tc.lo, self._tc.hi) == (sh.lo, sh.hi) \
            else None
        range_product(self, rows, None, Wcm, sh.lo, sh.hi, out, tcp=tcp)
        allreduce(out)
        return out[:, 0] if vector else out


def range_product(oracle, rows, row_ids, Wcm, lo, hi, out, accumulate=False, tcp=None):
    """out (nrows x m fp32) (+)= variance * K(rows, X[lo:hi]) @ W[lo:hi]: the
    block-row kernel over one contiguous range of column points (a shard).

    ``rows``: ("tc", RAg) tensor-core row features (nrows padded to 256) or
    ("pts", Rs, rsq) prepared FFMA rows; ``Wcm`` column-major (m x >= hi-lo)
    fp32; ``row_ids`` global ids of the rows (diagonal rule) or None.
    ``tcp``: the TcPoints of [lo, hi) if the caller holds them; otherwise the
    column features are built for the call and not cached in the oracle."""
    nrows = out.shape[0]
    m = Wcm.shape[0]
    if hi <= lo:
        if not accumulate:
            out.zero_()
        return out
    if rows[0] == "tc":
        if tcp is None or (tcp.lo, tcp.hi) != (lo, hi):
            tcp = TcPoints(oracle.spec, oracle._Xd, oracle.device, lo, hi, with_rows=False)
        zop = ZOperand(m, hi - lo, oracle.device).fill(Wcm)
        return krows_tc(oracle.spec, tcp, rows[1], nrows, row_ids, zop, out,
                        accumulate=accumulate)
    return krows_times(oracle.spec, oracle.points, rows[1], rows[2], row_ids, Wcm, out,
                       col_base=lo, accumulate=accumulate, ncols=hi - lo, col_offset=lo)


def kernel_eval(spec, x, y):
    """Single kernel value k(x, y), evaluated on the device (kernels.py:69-79)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    y = np.atleast_1d(np.asarray(y, dtype=np.float64))
    if x.shape != y.shape:
        raise ContractError("point dimensions do not match")
    return float(cross_kernel(spec, x[None, :], y[None, :])[0, 0])


def cross_kernel(spec, Xa, Xb, device=None):
    """Dense k(Xa, Xb) (kernels.py:82-91)."""
    dev = _device(device)
    A = DevicePoints(spec, Xa, dev)
    C = DevicePoints(spec, Xb, dev)
    if A.d != C.d:
        raise ContractError("point dimensions do not match")
    return ktile(spec, A.Xs[:A.n], A.sqn[:A.n], None, C.Xs[:C.n], C.sqn[:C.n], None, A.ldx,
                 A.d).cpu().numpy()


def block_rows_times(oracle, block, M, pool=None):
    """K[block, :] @ M (kernels.py:214-216)."""
    from .dist import col_dist_matmul
    return col_dist_matmul(oracle, M, block, pool)


def block_block(oracle, block):
    """Exact dense K[block, block] (kernels.py:219-221)."""
    return oracle.block(block)


def default_lengthscales(d):
    return np.full(d, math.sqrt(d))


SAP_COSINE = 3  # include/sapgp_b200.h: the random-feature "family" of sap_krows_tc


def cos_features_times(freq, phases, variance, X, theta, device):
    """phi(X) @ theta with phi = sqrt(2 var / q) cos(X F^T + p) (gp.py:49-114) on
    the tensor-core kernel: rows = points, columns = the q features, Z = theta,
    the epilogue evaluating cos instead of a covariance (never materialising
    phi). Returns an (n x s) float32 device tensor, or None when the shape is
    outside the tensor path (d > 9, s > 128)."""
    dev = _device(device)
    Xd = torch.as_tensor(X if torch.is_tensor(X) else np.asarray(X, dtype=np.float64),
                         dtype=torch.float64).to(dev).contiguous()
    F = torch.as_tensor(np.asarray(freq, dtype=np.float64), device=dev).contiguous()
    P = torch.as_tensor(np.asarray(phases, dtype=np.float64), device=dev).contiguous()
    T = theta if torch.is_tensor(theta) else np.asarray(theta, dtype=np.float64)
    n, d = Xd.shape
    q, s = F.shape[0], T.shape[1]
    if d > 9 or s > 128 or n < 1 or q < 1:
        return None
    bpad = (n + 255) // 256 * 256
    RA = torch.zeros((bpad, 32), dtype=torch.float32, device=dev)
    CA = torch.empty((q, 32), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        nat.call("sap_cos_features", nat.ptr(Xd), n, d, nat.ptr(F), nat.ptr(P), q, nat.ptr(RA),
                 nat.ptr(CA), nat.stream_handle())
        zop = ZOperand(s, q, dev).fill(to_colmajor(T, q, dev))
        out = torch.empty((n, s), dtype=torch.float32, device=dev)
        need = nat.load().sap_krows_tc_workspace(n, s, q)
        ws = torch.empty(need // 4 + 1, dtype=torch.float32, device=dev)
        nat.call("sap_krows_tc", nat.ptr(CA), q, 32, nat.ptr(RA), bpad, None, n, 0,
                 nat.ptr(zop.hi), nat.ptr(zop.lo), zop.nz, zop.ldz, nat.ptr(zop.scale), s,
                 SAP_COSINE, math.sqrt(2.0 * variance / q), nat.ptr(out), out.stride(0), 0,
                 nat.ptr(ws), ws.numel() * 4, nat.stream_handle())
    return out
