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


# SAP_TRACE=1: (time, thread, tag) marks of the bind and the lookahead
# producers (diagnosis: scripts/e2e_phases.py prints them)
import os as _os
import time as _time

TRACE = [] if _os.environ.get("SAP_TRACE") == "1" else None


def mark(tag):
    if TRACE is not None:
        TRACE.append((_time.perf_counter(), threading.current_thread().name, tag))


# ---------------------------------------------------------------------------
# host -> device uploads of large numpy arrays through a pinned double buffer

_UP = {"buf": None}
_UP_CHUNK = 1 << 23  # elements per chunk
def _host_threads():
    try:
        cores = len(_os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        cores = _os.cpu_count() or 8
    return max(2, min(8, cores))


# host conversion tasks per chunk (and the pool's threads): the casting copies
# are memory-bound, and a fresh float64 output's first touch (the kernel
# zeroing its pages) scales with threads: 55 ms on one thread for 520 MB, 11
# ms on eight (scripts/readback_probe.py). Twelve threads read W back ~2 ms
# faster on a 16-core box but slowed the concurrent steps as much (e2e
# 88.0-88.8 ms either way), so eight; SAP_HOST_THREADS overrides
_TASKS = int(_os.environ.get("SAP_HOST_THREADS", "0")) or _host_threads()
_POOL = {"ex": None}
_POOL_LOCK = threading.Lock()


def host_pool():
    """Process-wide host threads for the large casting copies of uploads and
    readbacks (numpy's casting copy releases the GIL)."""
    with _POOL_LOCK:
        if _POOL["ex"] is None:
            from concurrent.futures import ThreadPoolExecutor
            _POOL["ex"] = ThreadPoolExecutor(max_workers=_TASKS, thread_name_prefix="sap-host")
        return _POOL["ex"]


# Pre-faulted readback arrays: a fresh float64 host array's first touch costs
# ~55 ms per 520 MB on one thread (the kernel zeroing its pages), the largest
# single item of a W readback. An engine bound from host arrays asks for its
# readback array up front; these threads fault its pages in while the device
# runs the steps, and the readback then only copies and widens.
# SAP_PREFAULT_THREADS=0 turns it off.
_PF_THREADS = int(_os.environ.get("SAP_PREFAULT_THREADS", "4"))
_PF = {"ex": None}


def _touch(a):
    a[::512] = 0.0  # one store per 4 KB page


def prefaulted(shape):
    """(array, futures): a fresh C-contiguous float64 array of ``shape`` whose
    pages background threads fault in; wait on the futures before relying on
    it being resident (its contents are zeros wherever touched, otherwise
    undefined -- callers overwrite it entirely). None when turned off."""
    import numpy as np
    if _PF_THREADS <= 0:
        return None
    with _POOL_LOCK:
        if _PF["ex"] is None:
            from concurrent.futures import ThreadPoolExecutor
            _PF["ex"] = ThreadPoolExecutor(max_workers=_PF_THREADS,
                                           thread_name_prefix="sap-prefault")
        ex = _PF["ex"]
    out = np.empty(shape, dtype=np.float64)
    flat = out.reshape(-1)
    step = -(-flat.size // _PF_THREADS) if flat.size else 1
    step = -(-step // 512) * 512  # page-aligned slices
    futs = [ex.submit(_touch, flat[lo:lo + step]) for lo in range(0, flat.size, step)]
    return out, futs


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
    the DMA of chunk k-1 from the other half runs and the conversion of chunk
    k-1 finishes: pageable uploads (~11 GB/s here) would otherwise dominate a
    solve's setup. Values are rounded exactly as a device-side cast would
    (round to nearest)."""
    import numpy as np
    import torch
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
    ex = host_pool()
    done = [None, None]  # event: the half's last DMA finished reading it

    def convert(dst, lo, s0, s1):
        np.copyto(dst[s0 - lo:s1 - lo], flat_in[s0:s1], casting="same_kind")

    def dma(k, lo, hi, futs):
        for f in futs:
            f.result()
        h = k & 1
        flat_out[lo:hi].copy_(halves[h][:hi - lo], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        done[h] = ev

    prev = None
    for k, lo in enumerate(range(0, total, chunk)):
        hi = min(total, lo + chunk)
        h = k & 1
        if done[h] is not None:
            done[h].synchronize()
        dst = halves[h][:hi - lo].numpy()
        step = (hi - lo + _TASKS - 1) // _TASKS
        futs = [ex.submit(convert, dst, lo, s0, min(hi, s0 + step)) for s0 in range(lo, hi, step)]
        if prev is not None:
            dma(*prev)
        prev = (k, lo, hi, futs)
    dma(*prev)
    for ev in done:
        if ev is not None:
            ev.synchronize()
    return out
