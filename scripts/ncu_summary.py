"""Summarise an ncu report: key metrics, per-opcode counts, stall hot spots.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [--top 25]
"""
import argparse, collections, csv, io, subprocess, sys

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--entries", type=float, default=2e9)
a = ap.parse_args()

def run(*args):
    return subprocess.run(["ncu", "-i", a.rep, *args], capture_output=True, text=True).stdout

raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "lts__t_bytes.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
print("== metrics")
print("== kernel", vals[hdr.index("Kernel Name")][:100] if "Kernel Name" in hdr else "")
for h, u, v in zip(hdr, units, vals):
    if h in want:
        print(f"  {h:70s} {v:>14s} {u}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
H = src[1]
# a report with several kernels repeats the title/header rows: keep the first kernel's block
D = []
for r in src[2:]:
    if r and (r[0] == "Kernel Name" or r[0] == H[0]):
        break
    D.append(r)
ix = {k: H.index(k) for k in H}
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in D)
stalls = [k for k in H if k.startswith("stall_") and "Not Issued" not in k]
print("== per-opcode executed warp instructions (per entry = x32 / entries)")
cnt = collections.Counter()
for r in D:
    ex = float(r[ix["Instructions Executed"]] or 0)
    s = r[ix["Source"]].strip()
    op = s.split()[1] if s.startswith("@") else (s.split()[0] if s else "?")
    cnt[op] += ex
for op, c in cnt.most_common(30):
    print(f"  {op:32s} {c:14.0f} {c * 32 / a.entries:7.3f}")
print("== stall reasons (all samples)")
agg = collections.Counter()
for r in D:
    for k in stalls:
        agg[k] += float(r[ix[k]] or 0)
for k, v in agg.most_common(10):
    print(f"  {k:28s} {v / tot * 100:5.1f}%")
print(f"== top {a.top} instructions by stall samples (total {tot:.0f})")
for r in sorted(D, key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:a.top]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((float(r[ix[k]] or 0), k[6:]) for k in stalls), reverse=True)[:3]
    why = ", ".join(f"{k}:{v / max(s, 1) * 100:.0f}%" for v, k in top if v > 0)
    print(f"  {s / tot * 100:5.1f}% exe={r[ix['Instructions Executed']]:>10} {r[ix['Source']][:60]:60s} {why}")
