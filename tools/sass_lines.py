"""Attribute ncu per-SASS stall samples to CUDA source lines.

usage: sass_lines.py <ncu source --print-source sass csv> <nvdisasm -g output>
The two listings are aligned by instruction index within the kernel."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
samp = [float(r[idx['Warp Stall Sampling (All Samples)']] or 0) for r in rows[2:] if len(r) == len(hdr)]
inst = [float(r[idx['Instructions Executed']] or 0) for r in rows[2:] if len(r) == len(hdr)]
ops = [r[idx['Source']].strip() for r in rows[2:] if len(r) == len(hdr)]
lines = []
cur = None
for ln in open(sys.argv[2]):
    m = re.search(r'line (\d+)', ln)
    if ln.strip().startswith('//##') and m:
        cur = int(m.group(1))
        continue
    if re.search(r'/\*[0-9a-f]{4}\*/', ln):
        lines.append(cur)
n = min(len(lines), len(samp))
agg = defaultdict(float)
cnt = defaultdict(float)
for i in range(n):
    agg[lines[i]] += samp[i]
    cnt[lines[i]] += inst[i]
tot = sum(agg.values())
src = open(sys.argv[3]).read().splitlines() if len(sys.argv) > 3 else None
for l, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 30]:
    s = src[l - 1].strip()[:80] if (src and l) else ''
    print(f"{100 * v / tot:5.1f}%  inst {cnt[l]:12.0f}  L{l}: {s}")
