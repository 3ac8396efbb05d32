"""Per-launch grouped-GEMM efficiency: joins the RSC_GEMM_LOG lines of a run
(stderr) with the ncu gpu__time_duration of the same launches (in order).
python tools/gemm_launch_eff.py GEMMLOG.txt NCU.csv"""
import csv
import sys
from collections import defaultdict

logs = [ln.split() for ln in open(sys.argv[1]) if ln.startswith("GEMMLOG")]
lines = [ln for ln in open(sys.argv[2]) if ln.startswith('"')]
durs = []
for r in csv.DictReader(lines):
    if "gemm_grouped" in r["Kernel Name"] and "duration" in r["Metric Name"]:
        v = float(r["Metric Value"])
        durs.append(v * (1e-3 if r["Metric Unit"] in ("ns", "nsecond") else 1.0))  # us
print("log lines", len(logs), "ncu launches", len(durs))
n = min(len(logs), len(durs))
logs = logs[-n:]  # the profiled pass is the last one logged
edges = [0, 148, 444, 888, 1776, 3552, 10**9]
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
tot_t = tot_f = 0.0
for lg, us in zip(logs, durs[:n]):
    tiles, fl, pad = int(lg[5]), float(lg[9]), float(lg[11])
    for lo, hi in zip(edges[:-1], edges[1:]):
        if lo <= tiles < hi:
            a = agg[(lo, hi)]
            a[0] += 1; a[1] += us; a[2] += fl; a[3] += pad
    tot_t += us; tot_f += fl
for k in sorted(agg):
    a = agg[k]
    print(f"tiles {k[0]:5d}-{k[1]:<10d} launches {a[0]:5d} time {a[1]/1e3:8.2f} ms ({100*a[1]/tot_t:4.1f}%) "
          f"{a[2]/a[1]/1e6:6.2f} TF/s useful, {a[3]/a[1]/1e6:6.2f} TF/s padded, useful/padded {a[2]/a[3]:.2f}")
print(f"total {tot_t/1e3:.1f} ms  {tot_f/tot_t/1e6:.2f} TF/s")
