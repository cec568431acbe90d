"""Kernel timeline of steady-state ADASAP iterations (torch.profiler / CUPTI):
device busy fraction, idle gaps and what precedes/follows them."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2505_13723_b200 as sap
from paper_2505_13723_b200 import synthetic
from paper_2505_13723_b200.solvers import AdasapEngine
# config 3 by default; N=100000 D=11 B=1000 FAM=rbf for config 2
n, d, b = int(os.environ.get("N", "1000000")), int(os.environ.get("D", "9")), int(os.environ.get("B", "2000"))
m, r = 65, 100
prob = synthetic.make_problem(n, d, os.environ.get("FAM", "matern32"), m, seed=0, lam=1e-2, device="cuda", rhs="noise")
o = sap.KernelOracle(prob.spec(), prob.X, prob.lam)
WARM, NIT = int(os.environ.get("WARM", "64")), int(os.environ.get("NIT", "64"))
TOTAL = int(os.environ.get("TOTAL", str(WARM + NIT)))  # > WARM + NIT: production in the window
cfg = sap.RunConfig(lam=prob.lam, blocksize=b, nystrom_rank=r, residual_every=0,
                    max_iters=TOTAL)
eng = AdasapEngine(o, prob.Y, cfg, sap.resolve_accel(cfg, n, b), total=TOTAL)
for _ in range(WARM): eng.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(NIT): eng.step()
    torch.cuda.synchronize()
eng.close()
path = "/tmp/trace.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
busy, cur_end, gaps = 0.0, t0, []
for i, e in enumerate(ev):
    s, f = e["ts"], e["ts"] + e["dur"]
    if s > cur_end:
        gaps.append((s - cur_end, ev[i - 1]["name"][:50] if i else "", e["name"][:50]))
    busy += max(0.0, f - max(s, cur_end))
    cur_end = max(cur_end, f)
span = t1 - t0
print(f"span {span/NIT:.1f} us/iter, busy {busy/NIT:.1f} us/iter ({100*busy/span:.1f}%), kernels {len(ev)}")
gaps.sort(reverse=True)
tot = sum(g[0] for g in gaps)
print(f"idle {tot/NIT:.1f} us/iter in {len(gaps)} gaps; largest:")
for g in gaps[:15]:
    print(f"  {g[0]:8.1f} us  after {g[1]!r}  before {g[2]!r}")
streams = {}
for e in ev:
    streams.setdefault(e["args"].get("stream"), []).append(e)
for sid, es in streams.items():
    print(f"stream {sid}: {len(es)} kernels, {sum(e['dur'] for e in es)/NIT:.1f} us/iter")
# krows kernels: duration stats
kr = [e["dur"] for e in ev if "krows_tc2_kernel<" in e["name"] and ", 80," in e["name"]]
print("krows us:", [round(x) for x in kr[:NIT]])
# per-kernel totals per iteration, by stream
agg = {}
for e in ev:
    k = (e["args"].get("stream"), e["name"][:int(os.environ.get("NAMEW", "70"))])
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += e["dur"]
print("per-iteration kernel time by stream (us/iter, launches/iter):")
for (sid, name), (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(os.environ.get("TOPK", "40"))]:
    print(f"  s{sid} {t/NIT:8.1f} us  {c/NIT:5.2f}x  {name}")
# what separates consecutive block-row products: the interval from one krows
# kernel's end to the next one's start, and every kernel (any stream) that
# starts inside it, for a few sample intervals
krs = [e for e in ev if "krows_tc2_kernel<" in e["name"] and ", 80," in e["name"]]
ivs = [(a["ts"] + a["dur"], b["ts"]) for a, b in zip(krs, krs[1:])]
if ivs:
    w = sorted(f - s for s, f in ivs)
    print(f"krows->krows interval: median {w[len(w)//2]:.1f} us, mean {sum(w)/len(w):.1f} us, "
          f"max {w[-1]:.1f} us over {len(w)}")
    for s, f in ivs[:int(os.environ.get("SHOWIV", "4"))]:
        print(f"  interval {f - s:.1f} us:")
        for e in ev:
            if s - 1 <= e["ts"] < f:
                print(f"    +{e['ts'] - s:7.1f} {e['dur']:7.1f} us s{e['args'].get('stream')} {e['name'][:60]}")
