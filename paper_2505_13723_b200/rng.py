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


def native_blocks(seed, t0, count, n, blocksize, threads=1):
    """``uniform_block`` and ``block_hash`` for iterations t0..t0+count-1 in one
    native call (csrc/host_rng.cu, numpy-exact, GIL released): ((count, b)
    int64 blocks, list of crcs)."""
    import ctypes
    from . import _native as nat
    blocks = np.empty((count, blocksize), dtype=np.int64)
    crcs = np.empty(count, dtype=np.uint32)
    nat.call("sap_host_draws", int(seed), int(t0), int(count), int(n), int(blocksize),
             blocks.ctypes.data_as(ctypes.c_void_p), crcs.ctypes.data_as(ctypes.c_void_p),
             None, None, int(threads))
    return blocks, [int(c) for c in crcs]


def block_hash(block):
    """crc32 of the index bytes, the trace's cross-implementation check
    (solvers.py:250-251)."""
    return zlib.crc32(np.ascontiguousarray(block).tobytes())


def pcg64_words(gen):
    """PCG64 state of a fresh Generator as the 4 u64 words sap_normal_fill takes
    (state_hi, state_lo, inc_hi, inc_lo), as signed int64 for a torch tensor."""
    st = gen.bit_generator.state
    if st["bit_generator"] != "PCG64" or st.get("has_uint32", 0):
        raise ValueError("device normals need a fresh PCG64 generator")
    words = []
    for v in (st["state"]["state"], st["state"]["inc"]):
        for w in (v >> 64, v & 0xFFFFFFFFFFFFFFFF):
            words.append(w - (1 << 64) if w >= 1 << 63 else w)
    return words


class DeviceNormals:
    """Generator.standard_normal on the GPU, bit-exact with numpy (csrc/rng.cu).

    ``fill(states, out)`` writes the first ``count`` normals of each of the
    ``nstreams`` PCG64 streams (rows of the int64 (nstreams, 4) device tensor
    ``states``, see :func:`pcg64_words`) to the rows of ``out``
    ((nstreams, >= count) float64, row stride ``out.stride(0)``): the draw
    ``substream(seed, "omega", t).standard_normal((b, r))`` is row-major, so a
    (b, r) array is filled by count = b * r (solvers.py:384)."""

    def __init__(self, count, nstreams, device):
        import torch
        from . import _native as nat
        self.nat = nat
        self.count, self.nstreams = int(count), int(nstreams)
        lib = nat.load()
        nbytes = lib.sap_normal_workspace(self.count, self.nstreams)
        self.ws = torch.empty(nbytes // 8 + 1, dtype=torch.float64, device=device)
        assert lib.sap_normal_status(nat.ptr(self.ws)) == self.ws.data_ptr()
        self.ws[0] = 0  # status word: 0 until a fill reports otherwise

    def fill(self, states, out, nstreams=None):
        ns = self.nstreams if nstreams is None else int(nstreams)
        if not 0 < ns <= self.nstreams:
            raise ValueError("more streams than the workspace was sized for")
        nat = self.nat
        nat.check(nat.load().sap_normal_fill(nat.ptr(states), ns, self.count, nat.ptr(out),
                                             out.stride(0), nat.ptr(self.ws),
                                             self.ws.numel() * 8, nat.stream_handle()))

    def status(self):
        """Device int32 status of the fills on this workspace (0 = ok; sticky:
        a failed fill stays reported after reuse); reading it syncs."""
        return self.ws.view(dtype=__import__("torch").int32)[0]


def standard_normal(gen, shape, device=None):
    """``gen.standard_normal(shape)`` -- the same numbers, drawn on the GPU
    (csrc/rng.cu) when ``device`` is a CUDA device and the draw is large
    (>= 2^16 values, at most 2^30); returns a float64 torch tensor on the
    device then, a numpy array otherwise. ``gen`` must be fresh (nothing drawn
    from it yet); it is left untouched by the device path."""
    import math
    import torch
    shape = (shape,) if isinstance(shape, int) else tuple(shape)
    count = math.prod(shape)
    dev = torch.device(device) if device is not None else None
    if dev is None or dev.type != "cuda" or not (1 << 16) <= count <= (1 << 30):
        return gen.standard_normal(shape)
    states = torch.tensor([pcg64_words(gen)], dtype=torch.int64, device=dev)
    out = torch.empty((1, count), dtype=torch.float64, device=dev)
    dn = DeviceNormals(count, 1, dev)
    dn.fill(states, out)
    if int(dn.status()) != 0:  # one large draw: checking it costs one sync
        from .errors import NumericalError
        raise NumericalError("device normal draw failed (raw stream words ran out)")
    return out.view(shape)


def standard_normal_chunks(gen, rows, cols, device, rows_per_chunk):
    """``gen.standard_normal((rows, cols))`` drawn on the GPU in row chunks:
    yields (lo, hi, (hi - lo, cols) float64 device tensor). Each chunk is one
    device fill of more than 2^20 normals; the fill reports the raw words it
    consumed (``sap_normal_words``), and the stream's PCG64 state is advanced
    by exactly that many words on the host (``PCG64.advance``), so chunk k+1
    starts where numpy would draw the next value. No size limit (the one-shot
    device draw stops at 2^30 values). ``gen`` must be fresh; it is not
    modified."""
    import torch
    from . import _native as nat
    from .errors import NumericalError
    dev = torch.device(device)
    bg = np.random.PCG64()
    bg.state = gen.bit_generator.state
    min_count = (1 << 20) + 1  # the path that reports its consumption
    # every chunk but the last must be a full fill of its own values (the
    # reported consumption is that of the fill); only the last may be padded
    step = max(int(rows_per_chunk), -(-min_count // cols))
    cap = max(step * cols, min_count)
    dn = DeviceNormals(cap, 1, dev)
    buf = torch.empty((1, cap), dtype=torch.float64, device=dev)
    for lo in range(0, rows, step):
        hi = min(rows, lo + step)
        count = max((hi - lo) * cols, min_count)
        states = torch.tensor([pcg64_words(np.random.Generator(bg))], dtype=torch.int64,
                              device=dev)
        dn.count = count
        dn.fill(states, buf[:, :count])
        used = int(dn.ws.view(torch.int64)[1].item())  # sap_normal_words
        if int(dn.status()) != 0:
            raise NumericalError("device normal draw failed (raw stream words ran out)")
        bg.advance(used)
        yield lo, hi, buf[0, :(hi - lo) * cols].view(hi - lo, cols)
