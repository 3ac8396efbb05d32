"""Summarize an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[hdr_i], rows[hdr_i + 1:]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
skip = sys.argv[2] if len(sys.argv) > 2 else None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) <= vi or (skip and skip in r[ki]):
        continue
    v = float(r[vi].replace(",", "")) / 1e3
    name = r[ki].split("(")[0][:60]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(a[1] for a in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"{t / 1e3:9.3f} ms {100 * t / tot:5.1f}% n={c:6d} avg={t / c:9.1f}us {k}")
print(f"total {tot / 1e3:.3f} ms over {sum(a[0] for a in agg.values())} launches")
