"""Summarise an ncu --page source --csv dump: stall totals and the hottest SASS lines."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
lines = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    s = 0
    for h in stall_cols:
        try:
            v = float(r[idx[h]] or 0)
        except ValueError:
            v = 0
        tot[h] += v
        s += v
    lines.append((s, r[idx["Source"]], {h: r[idx[h]] for h in stall_cols if r[idx[h]] not in ("", "0")}))
T = sum(tot.values())
print("total samples", T)
for h, v in tot.most_common(12):
    print(f"  {h:28s} {100 * v / T:6.1f}%")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for s, src, d in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{s:8.0f}  {src[:70]:70s} {d}")
