import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
data = rows[hi + 1:]
ki, ii, mi, vi = h.index('Kernel Name'), h.index('ID'), h.index('Metric Name'), h.index('Metric Value')
k = {}
for r in data:
    if len(r) <= vi:
        continue
    d = k.setdefault(r[ii], {'name': r[ki]})
    d[r[mi]] = float(r[vi].replace(',', ''))
L = list(k.values())
tot = sum(x['gpu__time_duration.sum'] for x in L)
print('launches', len(L), 'total ms', tot / 1e6)
byk = collections.defaultdict(lambda: [0, 0.0, 0.0])
for x in L:
    nm = x['name'].split('(')[0][-28:]
    g = x.get('launch__grid_size', 0)
    t = x['gpu__time_duration.sum']
    cls = 'grid<148' if g < 148 else ('grid<740' if g < 740 else 'grid>=740')
    byk[(nm, cls)][0] += 1
    byk[(nm, cls)][1] += t
    byk[(nm, cls)][2] += t * x.get('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active', 0)
for key, (n, t, w) in sorted(byk.items(), key=lambda z: -z[1][1])[:14]:
    print(f"{key[0]:30s} {key[1]:10s} n={n:5d} {t/1e6:7.2f} ms  avg {t/n/1e3:6.1f} us  dmma {w/max(t,1):5.1f}%")
