"""Key metrics per kernel from an ncu report (details page)."""
import csv
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'Executed Ipc Active', 'Issue Slots Busy',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Dynamic Shared Memory Per Block', 'Waves Per SM', 'Block Size',
        'Grid Size', 'Block Limit Registers', 'Block Limit Shared Mem']
out = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, ni, vi, ii, ui = (hdr.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'ID', 'Metric Unit'))
cur = None
for r in rows[1:]:
    if r[ni] in WANT:
        key = (r[ii], r[ki][:60])
        if key != cur:
            print(); print(key); cur = key
        print(f"    {r[ni]:34s} {r[vi]} {r[ui]}")
raw = subprocess.run(['ncu', '-i', sys.argv[1], '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units = rr[0], rr[1]
keys = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'gpu__time_duration.sum']
for row in rr[2:]:
    print('---', row[h.index('Kernel Name')][:60])
    for k in keys:
        if k in h:
            print(f"    {k:60s} {row[h.index(k)]} {units[h.index(k)]}")
