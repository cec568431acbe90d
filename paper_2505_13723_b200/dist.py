"""Partitioned kernel products -- the drop-in operator boundary.

Mirrors ``sapgp.dist`` (dist.py:1-147). ``col_dist_matmul`` (ColDistMatMat,
paper Alg. 6) and ``row_dist_matmul`` (RowDistMatMat, Alg. 7) keep their
signatures; the work they hand to a thread pool in the reference runs here
as one fused CUDA launch (``sap_krows_times``) per call. Determinism is
preserved in the sense the reference tests use it: the reduction over the
point dimension has a fixed order for a given shape, so repeated calls are
bitwise identical and independent of the ``pool`` argument.

``WorkerPool`` is kept for API compatibility (solvers and CLIs pass it
around); on the B200 path its worker count does not change the arithmetic.
Multi-GPU sharding of the point dimension lives in ``parallel.py``.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .errors import ContractError

TILE = 256  # dist.py:19 -- kept for tile_ranges() users


def partition(size, parts):
    """Contiguous ranges covering [0, size), sizes differing by <= 1 (dist.py:22-35)."""
    if size < 0 or parts < 1:
        raise ContractError("partition needs size >= 0 and parts >= 1")
    parts = min(parts, max(size, 1))
    base, extra = divmod(size, parts)
    out, lo = [], 0
    for i in range(parts):
        hi = lo + base + (1 if i < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def tile_ranges(size):
    """Worker-count-free tile decomposition (dist.py:38-40)."""
    return partition(size, max(1, math.ceil(size / TILE)))


class WorkerPool:
    """API-compatible stand-in for the reference thread pool (dist.py:43-66).

    The device executes every tile of a product in one launch, so the pool
    only carries ``num_workers`` for callers that inspect it."""

    def __init__(self, num_workers=1):
        if int(num_workers) < 1:
            raise ContractError("num_workers must be >= 1")
        self.num_workers = int(num_workers)

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def check_indices(block, n):
    """Non-empty, in range, no duplicates (dist.py:96-105)."""
    block = np.asarray(block, dtype=np.intp).ravel()
    if block.size == 0:
        raise ContractError("empty index block")
    if block.min() < 0 or block.max() >= n:
        raise ContractError("block index out of range")
    if np.unique(block).size != block.size:
        raise ContractError("duplicate index in block")
    return block


def _device_oracle(oracle):
    if not hasattr(oracle, "rows_times_device"):
        raise ContractError(
            "oracle has no device representation; the B200 path needs a KernelOracle")
    return oracle


def col_dist_matmul(oracle, W, block, pool=None):
    """K[block, :] @ W (dist.py:108-127), one fused launch."""
    from .kernels import to_colmajor, _finish

    oracle = _device_oracle(oracle)
    n = oracle.n
    block = check_indices(block, n)
    like_np = not torch.is_tensor(W)
    Wa = W if torch.is_tensor(W) else np.asarray(W, dtype=np.float64)
    vector = Wa.ndim == 1
    if Wa.shape[0] != n:
        raise ContractError("W must have n rows")
    Rcm = to_colmajor(Wa, n, oracle.device)
    ids = torch.as_tensor(block.astype(np.int64), device=oracle.device)
    out = oracle.rows_times_device(ids, Rcm)
    return _finish(out, like_np, vector)


def row_dist_matmul(oracle, omega, block, pool=None):
    """K[block, block] @ omega (dist.py:130-147), one fused launch."""
    from .kernels import krows_times, to_colmajor, _finish

    oracle = _device_oracle(oracle)
    block = check_indices(block, oracle.n)
    like_np = not torch.is_tensor(omega)
    om = omega if torch.is_tensor(omega) else np.asarray(omega, dtype=np.float64)
    vector = om.ndim == 1
    if om.shape[0] != block.size:
        raise ContractError("omega must have one row per block index")
    ids = torch.as_tensor(block.astype(np.int64), device=oracle.device)
    Rs, rsq = oracle.points.gather(ids)
    Rcm = to_colmajor(om, block.size, oracle.device)
    out = torch.empty((block.size, Rcm.shape[0]), dtype=torch.float32, device=oracle.device)
    krows_times(oracle.spec, _Gathered(oracle.points, Rs, rsq), Rs, rsq, ids, Rcm, out,
                col_ids=ids)
    return _finish(out, like_np, vector)


class _Gathered:
    """A gathered point subset viewed as a column point set."""

    def __init__(self, pts, Xs, sqn):
        self.Xs, self.sqn = Xs, sqn
        self.n, self.d, self.ldx, self.device = Xs.shape[0], pts.d, pts.ldx, pts.device
