#!/bin/bash
# ncu --set full of the paired-line kernel and the default tiled kernel at 256^2, p = 16
O=gpurun_out
mkdir -p $O
N=${N:-256}; PP=${PP:-16}
for eng in pair dfma; do
  SMG_FD_ENGINE=$eng timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fd[tp]_kernel" -c 1 \
     -o $O/fd_${eng}_${PP} -f python tools/prof_kernels.py --n $N --p $PP --what fd --reps 2 > $O/ncu_${eng}.log 2>&1
  python tools/ncu_summary.py $O/fd_${eng}_${PP}.ncu-rep > $O/fd_${eng}_${PP}_summary.txt 2>&1
done
ls -la $O
