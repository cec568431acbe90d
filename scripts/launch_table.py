"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections, csv, sys
path, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ik, iv, im, iu = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Name", "Metric Unit"))
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
per = collections.defaultdict(list)
for r in data:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    per[r[ik].split("(")[0][:70]].append(float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0))
tot = sum(sum(v) for v in per.values())
lines = [title, f"# total kernel time {tot:.3f} ms over {sum(len(v) for v in per.values())} launches", "",
         f"{'kernel':72s} {'launches':>8s} {'total ms':>9s} {'mean ms':>8s} {'share':>6s}"]
for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{name:72s} {len(v):8d} {sum(v):9.3f} {sum(v) / len(v):8.4f} {sum(v) / tot * 100:5.1f}%")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:25]))
