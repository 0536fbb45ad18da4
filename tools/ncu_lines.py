"""Per-CUDA-source-line totals (instructions executed, stall samples) from
`ncu -i X --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
hdr = None
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        try:
            samp = float(r[4] or 0)
            inst = float(r[7] or 0)
        except ValueError:
            continue
        out.append((inst, samp, f"{cur}:{r[0]}", r[1][:90]))
ti = sum(o[0] for o in out)
ts = sum(o[1] for o in out)
print(f"total warp instructions {ti:.0f}, samples {ts:.0f}")
for inst, samp, loc, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{100 * inst / ti:5.1f}% inst {100 * samp / ts:5.1f}% stall  {loc:22s} {src}")
