"""Per-source-line instruction / stall summary of one kernel from an ncu
report: SASS rows (ncu --page source --print-source sass) mapped to source
lines with the cubin's line table (nvdisasm -g).

    python tools/ncu_srcmap.py REPORT.ncu-rep LIB.so KERNEL_SUBSTRING [TOP]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
kshow = sys.argv[5] if len(sys.argv) > 5 else None   # substring of the demangled name in the report
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        sections.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = r
    elif cur is not None:
        cur[2].append(r)
sec = next(s_ for s_ in sections if kshow is None or kshow in s_[0])
hdr = sec[1]
data = [r for r in sec[2] if len(r) == len(hdr)]
A, I, S = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][A], 16)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
off2line = {}
for cub in os.listdir(tmp):
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    if kname not in dis:
        continue
    cur = None
    infn = False
    for ln in dis.splitlines():
        m = re.search(r"\.text\.(\S+):", ln)
        if m:
            infn = kname in m.group(1)
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            off2line[int(m.group(1), 16)] = cur
inst = collections.Counter()
samp = collections.Counter()
why = collections.defaultdict(collections.Counter)
for r in data:
    k = off2line.get(int(r[A], 16) - base, ("?", 0))
    inst[k] += float(r[I] or 0)
    samp[k] += float(r[S] or 0)
    for h in stalls:
        why[k][h] += float(r[hdr.index(h)] or 0)
ti, ts = sum(inst.values()), sum(samp.values())
print(f"instructions {ti:.0f}, samples {ts:.0f}")
for k, v in samp.most_common(top):
    w = ", ".join(f"{h[6:]} {100 * c / v:.0f}%" for h, c in why[k].most_common(3) if v)
    print(f"{100 * v / ts:5.1f}% samp  {100 * inst[k] / ti:5.1f}% inst  {k[0]}:{k[1]}  [{w}]")
