"""The N > 1 path on the real kernels: two or three ranks (torchrun, gloo)
share the one GPU of the test box and each solves on its half of the point dimension
(sharded block product, one all-reduce of the b x m gradient per iteration,
owner-rank production of the lookahead batches); the trajectory must equal
the single-process one: identical blocks, stepsizes and residual trace to
fp32 accuracy, W to 1e-4 (fp32 sums in a different shard order). The
residual is the shard-local ring (no n x m all-gather), and a device-resident
solve (per-rank rows of Y as a CUDA tensor, W kept as shards) predicts by the
sharded cross product with one t x m all-reduce."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, nproc):
    out = str(tmp_path / f"mr{nproc}.npz")
    script = os.path.join(ROOT, "scripts", "multirank_check.py")
    if nproc == 1:
        cmd = [sys.executable, script, out]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1", "--master-port",
               str(29600 + nproc), script, out]
    env = dict(os.environ, SAP_DIST_BACKEND="gloo")
    subprocess.run(cmd, check=True, timeout=600, env=env, cwd=ROOT)
    return np.load(out)


@pytest.mark.parametrize("ranks", [2, 3])
def test_ranks_match_one(tmp_path, ranks):
    one = _run(tmp_path, 1)
    two = _run(tmp_path, ranks)
    assert np.array_equal(one["crc"], two["crc"])
    np.testing.assert_allclose(two["eta"], one["eta"], rtol=1e-6)
    due = ~np.isnan(one["res"])
    np.testing.assert_allclose(two["res"][due], one["res"][due], rtol=1e-4)
    assert np.abs(two["W"] - one["W"]).max() / np.abs(one["W"]).max() < 1e-4
    # the shard-local residual ring and the device-resident solve + sharded
    # prediction agree with the single-process run
    np.testing.assert_allclose(two["res_d"][due], one["res"][due], rtol=1e-4)
    for k in ("pred_d", "pred_h"):
        assert np.abs(two[k] - one["pred_h"]).max() / np.abs(one["pred_h"]).max() < 1e-4
