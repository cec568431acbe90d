"""sap_host_draws (csrc/host_rng.cu) against numpy, the reference's own RNG
(rng.py:14-24 substreams; solvers.py:260-262 block, :250-251 crc, :384 omega
stream, :395 power start vector). Host code only: runs without a GPU."""
import ctypes
import zlib

import numpy as np
import pytest

nat = pytest.importorskip("paper_2505_13723_b200._native")

from paper_2505_13723_b200.rng import pcg64_words, substream, uniform_block  # noqa: E402


def _lib():
    try:
        return nat.load()
    except Exception as exc:  # pragma: no cover - library not built
        pytest.skip(f"native library unavailable: {exc}")


def draws(seed, t0, count, n, b, omega=True, v0=True, threads=3):
    lib = _lib()
    blocks = np.empty((count, b), dtype=np.int64)
    crcs = np.empty(count, dtype=np.uint32)
    om = np.empty((count, 4), dtype=np.int64) if omega else None
    v = np.empty((count, b), dtype=np.float64) if v0 else None
    p = (lambda a: None if a is None else a.ctypes.data_as(ctypes.c_void_p))
    nat.check(lib.sap_host_draws(seed, t0, count, n, b, p(blocks), p(crcs), p(om), p(v), threads))
    return blocks, crcs, om, v


def _power_v0(seed, t, b):
    rng = substream(seed, "power", t)
    v = rng.standard_normal(b)
    return v / np.linalg.norm(v)


@pytest.mark.parametrize("seed,n,b", [
    (0, 500, 100),            # Floyd (n <= 10000)
    (3, 100_000, 1000),       # Floyd
    (4, 100_000, 5000),       # tail shuffle (b > n/50)
    (5, 10_000, 9_000),       # Floyd, dense
    (6, 20_000, 20_000),      # tail shuffle, b == n
    (7, 1, 1),
    (2**40 + 17, 1_000_000, 2000),  # two-word seed
])
def test_draws_match_numpy(seed, n, b):
    t0, count = 11, 5
    blocks, crcs, om, v = draws(seed, t0, count, n, b)
    for i in range(count):
        t = t0 + i
        ref = uniform_block(seed, t, n, b).astype(np.int64)
        assert np.array_equal(blocks[i], ref)
        assert int(crcs[i]) == zlib.crc32(ref.tobytes())
        assert om[i].tolist() == pcg64_words(substream(seed, "omega", t))
        # normals bit-exact; the normalisation differs from BLAS ddot by rounding
        np.testing.assert_allclose(v[i], _power_v0(seed, t, b), rtol=1e-14, atol=1e-300)


def test_draws_64bit_range_and_large_t():
    n, b, seed, t = 2**33 + 5, 7, 9, 2**35 + 3
    blocks, crcs, _, _ = draws(seed, t, 1, n, b, omega=False, v0=False)
    ref = uniform_block(seed, t, n, b).astype(np.int64)
    assert np.array_equal(blocks[0], ref)


def test_draw_normals_exact_over_tail():
    """Many normals (tail branch included): v0 * |v| reproduces numpy's draws."""
    seed, t, b = 2, 0, 200_000
    _, _, _, v = draws(seed, t, 1, 10**6, b, omega=False)
    ref = substream(seed, "power", t).standard_normal(b)
    scale = np.linalg.norm(ref)
    np.testing.assert_allclose(v[0] * scale, ref, rtol=1e-14, atol=0)
    assert np.array_equal(np.sign(v[0]), np.sign(ref))
    assert (np.abs(ref) > 3.6541528853610088).any()  # the ziggurat tail was drawn


def test_draws_thread_count_invariant():
    a = draws(1, 0, 9, 50_000, 300, threads=1)
    c = draws(1, 0, 9, 50_000, 300, threads=8)
    for x, y in zip(a, c):
        assert np.array_equal(x, y)


def test_draws_contract_errors():
    lib = _lib()
    buf = np.empty(8, dtype=np.int64)
    crc = np.empty(1, dtype=np.uint32)
    p = (lambda a: a.ctypes.data_as(ctypes.c_void_p))
    with pytest.raises(nat.ContractError):
        nat.check(lib.sap_host_draws(0, 0, 1, 4, 8, p(buf), p(crc), None, None, 1))


def test_native_blocks_helper():
    from paper_2505_13723_b200.rng import native_blocks
    _lib()
    blocks, crcs = native_blocks(5, 3, 4, 7000, 300, threads=2)
    for i in range(4):
        ref = uniform_block(5, 3 + i, 7000, 300).astype(np.int64)
        assert np.array_equal(blocks[i], ref) and crcs[i] == zlib.crc32(ref.tobytes())
