"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (per kernel mean us)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki][:70]].append(float(r[vi].replace(',', '')))
for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):5d} {sum(v)/len(v)/1000:10.2f} us  {n}")
