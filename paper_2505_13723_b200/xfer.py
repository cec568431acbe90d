"""Host<->device transfer accounting (bytes actually copied, counted at each
copy site of the solver path): the benchmark's e2e line reports these instead
of formulas."""

import threading

_lock = threading.Lock()
_bytes = {"h2d": 0, "d2h": 0}


def add(kind, nbytes):
    with _lock:
        _bytes[kind] += int(nbytes)


def snapshot():
    with _lock:
        return dict(_bytes)


# ---------------------------------------------------------------------------
# host -> device uploads of large numpy arrays through a pinned double buffer

_UP = {"buf": None}
_UP_CHUNK = 1 << 23  # elements per chunk


def _up_staging(nbytes):
    import torch
    buf = _UP["buf"]
    if buf is None or buf.numel() < 2 * nbytes:
        buf = torch.empty(2 * nbytes, dtype=torch.uint8, pin_memory=True)
        _UP["buf"] = buf
    return buf


def upload(A, dtype, device):
    """numpy array -> new contiguous device tensor of ``dtype`` (same shape).

    Host threads convert/copy chunk k into one half of a pinned buffer while
    the DMA of chunk k-1 from the other half runs: pageable uploads (~11 GB/s
    here) would otherwise dominate a solve's setup. Values are rounded exactly
    as a device-side cast would (round to nearest)."""
    import numpy as np
    import torch
    from concurrent.futures import ThreadPoolExecutor
    A = np.ascontiguousarray(A)
    np_dt = {torch.float32: np.float32, torch.float64: np.float64}[dtype]
    out = torch.empty(A.shape, dtype=dtype, device=device)
    total = A.size
    add("h2d", total * np.dtype(np_dt).itemsize)
    if total < (1 << 20):
        out.copy_(torch.from_numpy(A.astype(np_dt, copy=False)))
        return out
    flat_in, flat_out = A.reshape(-1), out.reshape(-1)
    chunk = min(_UP_CHUNK, total)
    esz = np.dtype(np_dt).itemsize
    stage = _up_staging(chunk * esz)
    halves = [stage[h * chunk * esz:(h + 1) * chunk * esz].view(dtype) for h in range(2)]
    stream = torch.cuda.current_stream(device)
    done = [None, None]  # event: the half's last DMA finished reading it
    with ThreadPoolExecutor(max_workers=4) as ex:
        for k, lo in enumerate(range(0, total, chunk)):
            hi = min(total, lo + chunk)
            h = k & 1
            if done[h] is not None:
                done[h].synchronize()
            dst = halves[h][:hi - lo].numpy()
            step = (hi - lo + 3) // 4
            list(ex.map(lambda s0: np.copyto(dst[s0 - lo:min(hi, s0 + step) - lo],
                                             flat_in[s0:min(hi, s0 + step)], casting="same_kind"),
                        range(lo, hi, step)))
            flat_out[lo:hi].copy_(halves[h][:hi - lo], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            done[h] = ev
    for ev in done:
        if ev is not None:
            ev.synchronize()
    return out
