"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '')
    agg.setdefault(name, []).append(float(r[vi].replace(',', '')) / 1000.0)
nframes = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tot = 0.0
for k, v in agg.items():
    per = sum(v) / nframes
    tot += per if k.startswith('vrs::') else 0
    print(f"{k[:60]:60s} n={len(v):4d} mean={sum(v)/len(v):9.1f} us  per-frame={per:9.1f} us")
print(f"vrs kernels per frame: {tot:.1f} us")
