"""Where the e2e (public step API from host arrays) time goes: oracle setup,
first step (engine bind + first plan), remaining steps, W readback."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import SolverState, adasap_step
n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, "matern32", m, seed=0, lam=1e-2, device="cuda")
X, Y = np.ascontiguousarray(prob.X), np.ascontiguousarray(prob.Y)
cfg = sap.RunConfig(lam=1e-2, blocksize=b, nystrom_rank=r, residual_every=0, seed=0)
if os.environ.get("GC") == "freeze":  # diagnosis: full collections over the imported modules
    import gc
    gc.freeze()
elif os.environ.get("GC") in ("off", "check"):
    import gc
    gc.disable()
for rep in range(int(os.environ.get("REPS", "8"))):
    torch.cuda.synchronize()
    T = [time.perf_counter()]
    o = sap.KernelOracle(prob.spec(), X, 1e-2, device="cuda"); torch.cuda.synchronize(); T.append(time.perf_counter())
    accel = sap.resolve_accel(cfg, n, b)
    st = SolverState.zeros(n, m, accelerated=True)
    st, eta, _ = adasap_step(o, st, Y, cfg, accel); torch.cuda.synchronize(); T.append(time.perf_counter())
    slow = []
    for k in range(19):
        h0 = time.perf_counter()
        st, eta, _ = adasap_step(o, st, Y, cfg, accel)
        dt = time.perf_counter() - h0
        if dt > 5e-3:
            slow.append((k + 1, round(dt * 1e3, 1)))
    torch.cuda.synchronize(); T.append(time.perf_counter())
    if st._e is not None and st._e.la.timings is not None:  # SAP_PROFILE=1
        for tm in sorted(st._e.la.timings, key=lambda x: x["start"]):
            print(f"   batch count={tm['count']:3d} start {1e3 * (tm['start'] - T[1]):7.1f} "
                  f"end {1e3 * (tm['end'] - T[1]):7.1f} ms (rng {1e3 * tm['rng']:.1f}, "
                  f"enqueue {1e3 * tm['gpu_wait']:.1f}, factor {1e3 * tm['factor']:.1f})")
    from paper_2505_13723_b200 import xfer
    if xfer.TRACE is not None:  # SAP_TRACE=1
        for tt, th, tag in xfer.TRACE:  # from the start of the rep (oracle included)
            if tt >= T[0]:
                print(f"   {1e3 * (tt - T[0]):8.2f} ms  {th:22s} {tag}")
        xfer.TRACE.clear()
    W = st.W; torch.cuda.synchronize(); T.append(time.perf_counter())
    st.iteration = st.iteration; T.append(time.perf_counter())
    names = ["oracle", "bind+step0", "19 steps", "W readback", "close"]
    if os.environ.get("GC") == "check":  # what one rep leaves to the cyclic collector
        import gc
        del st, W
        gc.set_debug(gc.DEBUG_SAVEALL)
        g0 = time.perf_counter()
        found = gc.collect()
        dt_gc = 1e3 * (time.perf_counter() - g0)
        import collections
        kinds = collections.Counter(type(x).__qualname__ for x in gc.garbage).most_common(8)
        gc.garbage.clear()
        gc.set_debug(0)
        print(f"   gc.collect: {found} unreachable objects in {dt_gc:.1f} ms; tracked objects "
              f"{len(gc.get_objects())}; kinds {kinds}", flush=True)
    print(rep, "  ".join(f"{k} {1e3*(T[i+1]-T[i]):.1f} ms" for i, k in enumerate(names)),
          "slow steps (host ms):", slow, flush=True)
