"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 path's host logic.

The B200 engine shards the point dimension (ShardInfo), adds the owned block
rows' lam*Z - Y terms before ONE all-reduce of the b x m gradient, computes
the block direction redundantly and updates only owned rows (paper Alg. 6,
SURVEY.md §8e). Here every rank runs exactly that decomposition with the CPU
oracle standing in for the device block product, and the gathered result
must equal the single-process reference trajectory.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import sapgp_oracle as orc
from paper_2505_13723_b200.parallel import ShardInfo, allreduce_sum_, gather_rows


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded_adasap(rank, world, port, n, d, b, r, iters, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        X = rng.standard_normal((n, d))
        Y = rng.standard_normal((n, 3))
        lam, seed = 0.1, 5
        pts = orc.Points("matern32", np.full(d, 1.5), 1.0, X)
        sh = ShardInfo.of(n, rank, world)
        beta, gamma, alpha = orc.accel_coeffs(lam, n, b)
        V = np.zeros((sh.size, 3))
        Z = np.zeros((sh.size, 3))
        W = np.zeros((sh.size, 3))
        for t in range(iters):
            blk = orc.uniform_block(seed, t, n, b)
            loc = sh.local_positions(blk)
            own = loc >= 0
            # partial K[B, shard] Z[shard] + owned rows' lam Z - Y, then one all-reduce
            g = pts.tile(blk, np.arange(sh.lo, sh.hi)) @ Z if sh.size else np.zeros((b, 3))
            g[own] += lam * Z[loc[own]] - Y[sh.lo:sh.hi][loc[own]]
            gt = torch.from_numpy(g)
            allreduce_sum_(gt)
            g = gt.numpy()
            # redundant direction (every rank draws the same Omega / power start)
            omega = orc.substream(seed, "omega", t).standard_normal((b, r))
            U, S = orc.rand_nystrom_retry(orc.row_dist_matmul(pts, omega, blk), omega, r)
            rho = float(S[-1]) + lam
            Kbb = orc.block_block(pts, blk)
            eta = orc.rand_power_stepsize(lambda v: Kbb @ v + lam * v, U, S, rho, 10,
                                          orc.substream(seed, "power", t))
            DB = orc.apply_inv(U, S, rho, g)
            D = np.zeros((sh.size, 3))
            D[loc[own]] = DB[own]
            W, V, Z = orc.nesterov_update(W, V, Z, D, eta, beta, gamma, alpha)
        full = gather_rows(torch.from_numpy(W), n, sh).numpy()
        if rank == 0:
            np.save(out, full)
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_adasap_matches_single_process(tmp_path, world):
    n, d, b, r, iters = 157, 3, 20, 8, 6
    out = str(tmp_path / "w.npy")
    mp.spawn(_sharded_adasap, args=(world, _free_port(), n, d, b, r, iters, out), nprocs=world,
             join=True)
    got = np.load(out)
    rng = np.random.default_rng(3)
    X = rng.standard_normal((n, d))
    Y = rng.standard_normal((n, 3))
    pts = orc.Points("matern32", np.full(d, 1.5), 1.0, X)
    ref, _, _, _ = orc.adasap_solve(pts, 0.1, Y, iters, 5, b, r)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-10 * max(1.0, np.abs(ref).max()))


def _allreduce_and_gather(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 11
        sh = ShardInfo.of(n, rank, world)
        local = torch.arange(sh.lo, sh.hi, dtype=torch.float64)[:, None].repeat(1, 2)
        full = gather_rows(local, n, sh)
        s = torch.tensor([float(rank + 1)])
        allreduce_sum_(s)
        if rank == 0:
            np.save(out, np.concatenate([full[:, 0].numpy(), s.numpy()]))
    finally:
        tdist.destroy_process_group()


def test_gather_rows_and_allreduce(tmp_path):
    out = str(tmp_path / "g.npy")
    mp.spawn(_allreduce_and_gather, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    assert np.array_equal(got[:11], np.arange(11.0)) and got[11] == 3.0
