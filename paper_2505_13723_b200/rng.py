"""Named random substreams (reference rng.py:14-33).

Index sampling must be bit-exact with the reference, so the same numpy
``Generator`` (PCG64 seeded through ``SeedSequence``) is used with the same
key layout: (seed, crc32(name), *indices).
"""

import zlib

import numpy as np


def substream(seed, name, *indices):
    """Generator for stream ``name`` at optional per-call indices (rng.py:14-24)."""
    key = (int(seed), zlib.crc32(name.encode("utf-8"))) + tuple(int(i) for i in indices)
    return np.random.default_rng(np.random.SeedSequence(key))


def as_generator(seed):
    """Integer seed, SeedSequence or ready Generator -> Generator (rng.py:27-33)."""
    if isinstance(seed, np.random.Generator):
        return seed
    if isinstance(seed, np.random.SeedSequence):
        return np.random.default_rng(seed)
    return np.random.default_rng(int(seed))


def uniform_block(seed, iteration, n, blocksize):
    """Sorted uniform block without replacement (solvers.py:260-262)."""
    rng = substream(seed, "block", iteration)
    return np.sort(rng.choice(n, size=blocksize, replace=False))


def block_hash(block):
    """crc32 of the index bytes, the trace's cross-implementation check
    (solvers.py:250-251)."""
    return zlib.crc32(np.ascontiguousarray(block).tobytes())
