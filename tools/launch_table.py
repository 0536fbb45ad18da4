"""Aggregate an ncu --metrics gpu__time_duration.sum launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if 'Kernel Name' in r)
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
agg = collections.OrderedDict()
for d in data:
    if d.get('Metric Name') == 'gpu__time_duration.sum':
        agg.setdefault(d['Kernel Name'][:70], []).append(float(d['Metric Value']))
tot = sum(sum(v) for v in agg.values())
print(f"{'n':>5} {'avg_us':>9} {'total_us':>10} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):5d} {sum(v)/len(v)/1e3:9.2f} {sum(v)/1e3:10.1f} {100*sum(v)/tot:5.1f}%  {k}")
