"""Latency of a fresh lookahead's first plan (the step API's first step waits
for it), by phase: host draws, enqueue of the fast-stream work, device
completion of the phase-1 work and of the power iteration."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic, pipeline
n, d, b, m, r = 1_000_000, 9, 2000, 65, 100
prob = synthetic.make_problem(n, d, "matern32", m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
tcp = o.tc_points(0, n)
from paper_2505_13723_b200.parallel import current_shard
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    la = pipeline.Lookahead(o, current_shard(n), 0, b, r, 1e-2, None, 32, False, tcp=tcp)
    t1 = time.perf_counter()
    plan = la.get(0)
    t2 = time.perf_counter()
    torch.cuda.current_stream().wait_event(la.cur.ready)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"rep {rep}: Lookahead() {1e3*(t1-t0):.1f} ms, get(0) (producer done) {1e3*(t2-t1):.1f} ms, "
          f"device ready {1e3*(t3-t2):.1f} ms", flush=True)
    la.close()

# the producer's host time, by function (one batch of 1, in this thread)
import cProfile, pstats
la = pipeline.Lookahead(o, current_shard(n), 0, b, r, 1e-2, None, 32, False, tcp=tcp)
la.get(0)
slot = la.slots[1 % len(la.slots)]
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
la._produce(la.slots[-1], 100000, 1, la.sides[0])
t1 = time.perf_counter()
pr.disable()
print(f"_produce(count=1) host time {1e3*(t1-t0):.1f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
la.close()
