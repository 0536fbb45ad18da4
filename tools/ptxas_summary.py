"""Summarise ptxas -v logs: registers and spills per kernel (demangled-ish)."""
import glob
import os
import re
import sys

pat = sys.argv[1] if len(sys.argv) > 1 else "fdt_kernel"
rows = {}
for f in glob.glob(os.environ.get("PTXAS_GLOB", "build/smg/*.ptxas.log")):
    name = None
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"Function properties for (\S+)", line)
        if m:
            name = m.group(1)
            continue
        if name and pat in name:
            m = re.search(r"(\d+) bytes spill stores", line)
            if m:
                rows.setdefault(name, {})["spill"] = int(m.group(1))
            m = re.search(r"Used (\d+) registers", line)
            if m:
                rows.setdefault(name, {})["regs"] = int(m.group(1))
for n, d in sorted(rows.items()):
    m = re.search(r"ILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELb(\d)(?:ELi(\d+))?E", n)
    tag = "p=%s no=%s tile=%sx%s dm=%s lc=%s" % m.groups() if m else n[:60]
    print(f"{tag:40s} regs {d.get('regs', '?'):>4} spill {d.get('spill', 0)}")
