"""Brief view of one kernel in an ncu report: pipes, stalls, shared-memory wavefronts,
and the source lines with the most stall samples.  python tools/ncu_brief.py X.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, row = rr[0], rr[2]
print(row[h.index('Kernel Name')][:70])
for k in ['gpu__time_duration.sum', 'launch__registers_per_thread', 'launch__block_size', 'launch__grid_size',
          'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
          'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
          'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
          'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active',
          'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
          'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
          'sm__inst_executed.avg.per_cycle_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
          'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__cycles_elapsed.max']:
    if k in h:
        print(f"  {k:75s} {row[h.index(k)]}")
st = []
for i, k in enumerate(h):
    if 'issue_stalled' in k and k.endswith('per_issue_active.ratio'):
        st.append((float(row[i]), k[33:-23]))
print("  stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:9]))
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
cur = None
hdr = None
out = []


def f(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) > 20:
        out.append((f(r[4]), f(r[7]), f(r[19]), f(r[18]), f"{cur}:{r[0]}", r[1].strip()[:80]))
ts = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
tw = sum(o[2] for o in out) or 1
print(f"  source lines: {ti:.0f} warp instr, {tw:.0f} smem wavefronts ({sum(o[3] for o in out):.0f} excess)")
for s, i, w, e, loc, txt in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"  {100 * s / ts:5.1f}% stall {100 * i / ti:5.1f}% inst {100 * w / tw:5.1f}% wf  {loc:18s} {txt}")
