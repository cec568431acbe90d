"""Poor man's sampling profiler for the e2e path (the step API from host
arrays): every 0.5 ms a sampler thread records the innermost frames of every
Python thread (the solver thread and the lookahead producers), then prints
per-thread runs of identical stacks longer than 2 ms. Shows where the bind
and the producers wait.

    python scripts/stack_sample.py [reps]
"""
import os, sys, threading, time, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import SolverState, adasap_step

n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, "matern32", m, seed=0, lam=1e-2, device="cuda")
X, Y = np.ascontiguousarray(prob.X), np.ascontiguousarray(prob.Y)
cfg = sap.RunConfig(lam=1e-2, blocksize=b, nystrom_rank=r, residual_every=0, seed=0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
samples = []
stop = threading.Event()


def sampler():
    me = threading.get_ident()
    while not stop.is_set():
        now = time.perf_counter()
        for tid, fr in sys._current_frames().items():
            if tid == me:
                continue
            st = traceback.extract_stack(fr)[-4:]
            key = " < ".join(f"{os.path.basename(f.filename)}:{f.lineno}:{f.name}" for f in reversed(st))
            samples.append((now, tid, key))
        time.sleep(5e-4)


def one(tag):
    torch.cuda.synchronize()
    T0 = time.perf_counter()
    o = sap.KernelOracle(prob.spec(), X, 1e-2, device="cuda")
    accel = sap.resolve_accel(cfg, n, b)
    st = SolverState.zeros(n, m, accelerated=True)
    for _ in range(20):
        st, eta, _ = adasap_step(o, st, Y, cfg, accel)
    W = st.W
    torch.cuda.synchronize()
    T1 = time.perf_counter()
    st.iteration = st.iteration  # detach: releases the engine
    print(f"{tag}: {1e3 * (T1 - T0):.1f} ms", flush=True)
    return T0, T1


for k in range(reps - 1):
    one(f"rep {k}")
th = threading.Thread(target=sampler, daemon=True)
th.start()
T0, T1 = one("sampled rep")
stop.set()
th.join()
names = {t.ident: t.name for t in threading.enumerate()}
main_id = threading.main_thread().ident
by = {}
for now, tid, key in samples:
    if T0 <= now <= T1:
        by.setdefault(tid, []).append((now, key))
for tid, ss in sorted(by.items(), key=lambda kv: (kv[0] != main_id, kv[0])):
    print(f"--- thread {names.get(tid, tid)}")
    run_key, run_t0, last = None, None, None
    for now, key in ss + [(ss[-1][0] + 1, None)]:
        if key != run_key:
            if run_key is not None and last - run_t0 >= 2e-3:
                print(f"  {1e3 * (run_t0 - T0):8.1f} +{1e3 * (last - run_t0):6.1f} ms  {run_key}")
            run_key, run_t0 = key, now
        last = now
