"""Sum ncu per-SASS 'Instructions Executed' and stall samples by CUDA source line
ranges (regions) -- usage: sass_regions.py <sass csv> <nvdisasm -g> <source> <region spec>
region spec: name:first-last,name:first-last,..."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
inst = [float(r[idx['Instructions Executed']] or 0) for r in data]
samp = [float(r[idx['Warp Stall Sampling (All Samples)']] or 0) for r in data]
lines, cur = [], None
for ln in open(sys.argv[2]):
    m = re.search(r'line (\d+)', ln)
    if ln.strip().startswith('//##') and m:
        cur = int(m.group(1))
        continue
    if re.search(r'/\*[0-9a-f]{4}\*/', ln):
        lines.append(cur)
regions = []
for spec in sys.argv[4].split(','):
    name, rng = spec.split(':')
    a, b = rng.split('-')
    regions.append((name, int(a), int(b)))
I, S = defaultdict(float), defaultdict(float)
for i in range(min(len(lines), len(inst))):
    l = lines[i] or 0
    name = next((n for n, a, b in regions if a <= l <= b), 'other')
    I[name] += inst[i]
    S[name] += samp[i]
ti, ts = sum(I.values()), sum(S.values())
for n in [r[0] for r in regions] + ['other']:
    print(f"{n:14s} inst {100 * I[n] / ti:5.1f}%   stall-samples {100 * S[n] / ts:5.1f}%")
print("total inst", ti)
