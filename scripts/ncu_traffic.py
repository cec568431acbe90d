"""Per-launch DRAM traffic and duration of the block-row kernel from `ncu --set
full` reports of bench.py (one steady-state launch per family), written to
profiles/r02_krows_traffic.json for bench.py's roofline.traffic:

    python scripts/ncu_traffic.py matern32=gpurun_out/r02_krows_m32.ncu-rep \\
                                  rbf=gpurun_out/r02_krows_rbf.ncu-rep
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__registers_per_thread")


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for k in WANT:
        if k in hdr:
            i = hdr.index(k)
            res[k] = (vals[i], units[i])
    res["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""
    return res


def to_bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    out = {}
    for arg in sys.argv[1:]:
        fam, rep = arg.split("=", 1)
        m = raw_metrics(rep)
        rd = to_bytes(*m["dram__bytes_read.sum"])
        wr = to_bytes(*m["dram__bytes_write.sum"])
        out[fam] = {"bytes": int(rd + wr), "read": int(rd), "write": int(wr),
                    "duration": " ".join(m["gpu__time_duration.sum"]),
                    "metrics": {k: " ".join(v) for k, v in m.items() if k != "kernel"},
                    "kernel": m["kernel"][:120],
                    "source": os.path.relpath(rep, ROOT) + " (ncu --set full, one steady-state "
                              "launch of bench.py; serialised, cold-cache replay)"}
    path = os.path.join(ROOT, "profiles", "r02_krows_traffic.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
