"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki = h.index('Kernel Name'); mi = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) <= mi: continue
    name = r[ki].split('(')[0]
    agg[name][0] += 1; agg[name][1] += float(r[mi].replace(',', ''))
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:44s} {v[0]:8d} {v[1]/1e3:10.1f} {v[1]/v[0]/1e3:9.2f} {v[1]/tot:6.3f}")
