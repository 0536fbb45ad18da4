"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of
the C2 top-level kernels from an ncu report -> profiles/traffic_c2.json.

    python tools/ncu_traffic.py gpurun_out/X.ncu-rep [profiles/traffic_c2.json]"""
import csv
import json
import subprocess
import sys

rep = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic_c2.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]


def val(row, key):
    i = h.index(key)
    v = float(row[i].replace(",", ""))
    u = units[i].strip().lower()
    scale = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6,
             "msecond": 1e-3}.get(u, 1)
    return v * scale


res = {}
for row in rows[2:]:
    name = row[h.index("Kernel Name")]
    key = name.split("<")[0].split("(")[0].replace("void ", "").replace("smg::", "").strip()
    if key == "opw_kernel" and name.split("(")[0].rstrip(">").rstrip().endswith("1"):
        key = "opw_kernel_restr"   # opw_kernel<P, TX, TY, DOT, RESTR = 1>: residual restricted in place
    tr = val(row, "dram__bytes_read.sum") + val(row, "dram__bytes_write.sum")
    res.setdefault(key, {"bytes_per_launch": tr, "kernel": name[:90], "report": rep.split("/")[-1]})
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
