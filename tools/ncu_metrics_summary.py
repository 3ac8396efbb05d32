"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv log: launches, time, DRAM bytes, GB/s.
python tools/ncu_metrics_summary.py LOG.csv [top]"""
import csv
import re
import sys
from collections import defaultdict

rows = defaultdict(dict)
names = {}
with open(sys.argv[1]) as f:
    lines = [ln for ln in f if ln.startswith('"')]
for r in csv.DictReader(lines):
    i = int(r["ID"])
    names[i] = r["Kernel Name"]
    v = float(r["Metric Value"].replace(",", ""))
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    rows[i][r["Metric Name"]] = v * scale.get(r["Metric Unit"], 1.0) if "duration" in r["Metric Name"] else v  # us
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in rows.items():
    nm = re.sub(r"\(.*", "", names[i]).replace("void ", "")
    nm = re.sub(r"\(anonymous namespace\)::", "", nm)
    a = agg[nm]
    a[0] += 1
    t = m.get("gpu__time_duration.sum", 0.0)
    a[1] += t
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
print(f"launches {len(rows)}  kernel time {tot / 1e3:.2f} ms (serialized, cold-ish cache; shares only)")
print(f"{'kernel':60s} {'n':>6s} {'ms':>9s} {'share':>6s} {'DRAM GB':>8s} {'GB/s':>7s}")
for nm, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    gb = (a[2] + a[3]) / 1e9
    print(f"{nm[:60]:60s} {a[0]:6d} {a[1] / 1e3:9.2f} {100 * a[1] / tot:5.1f}% {gb:8.3f} {gb / (a[1] * 1e-6) if a[1] else 0:7.0f}")
