"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
stall samples per opcode class and per code region.

    ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
    python scripts/ncu_stalls.py src.csv
"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
isrc = hdr.index("Source")
iexe = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {r: hdr.index(r) for r in reasons}
by_op = collections.defaultdict(lambda: collections.Counter())
for r in data:
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    for k in reasons:
        by_op[o][k] += int(r[idx[k]] or 0)
tot = collections.Counter()
for o, c in by_op.items():
    tot.update(c)
print("total", sum(tot.values()), dict(tot.most_common(8)))
for o, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:18]:
    s = sum(c.values())
    print(f"{o:10s} {s:7d}  " + " ".join(f"{k[6:]}={v}" for k, v in c.most_common(4)))
