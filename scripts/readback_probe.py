import time, numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
n = 65_000_000
for rep in range(3):
    t0 = time.perf_counter(); a = np.empty(n, dtype=np.float64); a[::512] = 0; t1 = time.perf_counter()
    print(f"fresh 520 MB first touch (1 thread): {1e3*(t1-t0):.1f} ms")
    del a
ex = ThreadPoolExecutor(8)
for rep in range(3):
    a = np.empty(n, dtype=np.float64)
    t0 = time.perf_counter()
    step = n // 8
    list(ex.map(lambda i: a[i*step:(i+1)*step].__setitem__(slice(None, None, 512), 0), range(8)))
    t1 = time.perf_counter()
    print(f"fresh 520 MB first touch (8 threads): {1e3*(t1-t0):.1f} ms")
    del a
src = torch.randn(n // 2 * 2, device="cuda", dtype=torch.float32)[: n]
pin = torch.empty(1 << 23, dtype=torch.float32, pin_memory=True)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for k in range(0, n, 1 << 23):
        m = min(1 << 23, n - k); pin[:m].copy_(src[k:k+m], non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"D2H 260 MB pinned chunks: {1e3*(t1-t0):.1f} ms = {n*4/(t1-t0)/1e9:.1f} GB/s")
