"""Sharding of the point dimension over GPUs (paper Alg. 6, ColDistMatMat).

One process per GPU (``torchrun``), ``torch.distributed`` for the plumbing.
Rows of the iterate state (the lazy Nesterov pair P, Q) and of the
right-hand sides Y are split into contiguous shards; the prepared points X
are replicated (n x 12 fp32 = 4.8 GB at n = 10^8, small next to 180 GB).
Per ADASAP iteration the only exchange is one all-reduce (sum) of the
b x m float64 block gradient: every other quantity is
either a pure function of (seed, t) -- computed redundantly on every rank
-- or owned by exactly one rank.

``ShardInfo`` is also what the world_size-2 gloo tests exercise on CPU.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch
import torch.distributed as tdist

from .dist import partition


@dataclass(frozen=True)
class ShardInfo:
    rank: int
    world: int
    lo: int
    hi: int
    n: int

    @property
    def size(self):
        return self.hi - self.lo

    @classmethod
    def single(cls, n):
        return cls(0, 1, 0, n, n)

    @classmethod
    def of(cls, n, rank, world):
        lo, hi = partition(n, world)[rank] if n >= world else (
            (0, n) if rank == 0 else (n, n))
        return cls(rank, world, lo, hi, n)

    def owned(self, block):
        """Boolean mask of the global ids this shard owns."""
        return (block >= self.lo) & (block < self.hi)

    def local_positions(self, block):
        """Local row of each global id, or -1 when another shard owns it."""
        loc = block - self.lo
        return torch.where(self.owned(block), loc, torch.full_like(loc, -1)) \
            if torch.is_tensor(block) else _np_loc(block, self.lo, self.hi)


def _np_loc(block, lo, hi):
    import numpy as np
    b = np.asarray(block, dtype=np.int64)
    return np.where((b >= lo) & (b < hi), b - lo, -1)


def current_shard(n):
    """Shard of this process when torch.distributed is initialised, else all rows."""
    if tdist.is_available() and tdist.is_initialized():
        return ShardInfo.of(n, tdist.get_rank(), tdist.get_world_size())
    return ShardInfo.single(n)


def allreduce_sum_(t):
    """In-place sum over ranks (no-op for a single process)."""
    if tdist.is_available() and tdist.is_initialized() and tdist.get_world_size() > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.SUM)
    return t


def gather_rows(local, n, shard):
    """Concatenate the row shards of an (n_local x m) tensor on every rank
    (the inverse of ShardInfo.of); works for CUDA (NCCL) and CPU (gloo)."""
    if shard.world == 1:
        return local
    sizes = [hi - lo for lo, hi in partition(n, shard.world)] if n >= shard.world else \
        [n if r == 0 else 0 for r in range(shard.world)]
    mx = max(sizes)
    buf = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[:local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in sizes]
    tdist.all_gather(parts, buf)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)


def init_from_env(backend=None):
    """Initialise torch.distributed from torchrun's environment, if present."""
    if "RANK" not in os.environ or "WORLD_SIZE" not in os.environ:
        return False
    if tdist.is_initialized():
        return True
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        # bind the communicator to this rank's GPU up front (no device guessing)
        tdist.init_process_group(backend=backend, device_id=torch.device("cuda", local))
    else:
        tdist.init_process_group(backend=backend)
    return True
