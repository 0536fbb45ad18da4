#!/bin/bash
O=gpurun_out
ENGINES=pair TAG=minb3 python tools/time_fd_sweep.py 256:16 64:16 > $O/pair_time2.log 2>&1
SMG_LIB=$PWD/paper_1512_02390_b200/libsmg_b2.so ENGINES=pair TAG=minb2 python tools/time_fd_sweep.py 256:16 64:16 >> $O/pair_time2.log 2>&1
SMG_FDP_TILE=42 ENGINES=pair TAG=t42 python tools/time_fd_sweep.py 256:16 64:16 >> $O/pair_time2.log 2>&1
SMG_FD_ENGINE=pair timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fd[tp]_kernel" -c 1 \
     -o $O/fd_pair_16 -f python tools/prof_kernels.py --n 256 --p 16 --what fd --reps 2 > $O/ncu_pair.log 2>&1
cat $O/pair_time2.log
