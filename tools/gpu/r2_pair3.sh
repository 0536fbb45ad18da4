#!/bin/bash
O=gpurun_out
python tools/pair_check.py 8 12 16 24 32 > $O/pair_check.log 2>&1; echo "rc $?" >> $O/pair_check.log
ENGINES=pair TAG=def python tools/time_fd_sweep.py 256:8 256:12 256:16 256:24 256:32 128:32 64:16 > $O/pair_time3.log 2>&1
SMG_FDP_TILE=42 ENGINES=pair TAG=t42 python tools/time_fd_sweep.py 256:32 128:32 256:16 >> $O/pair_time3.log 2>&1
SMG_FDP_TILE=22 ENGINES=pair TAG=t22 python tools/time_fd_sweep.py 256:24 >> $O/pair_time3.log 2>&1
for cfg in "128 32" "256 24"; do set -- $cfg
SMG_FD_ENGINE=pair timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fdp_kernel" -c 1 \
     -o $O/fdp_$2 -f python tools/prof_kernels.py --n $1 --p $2 --what fd --reps 2 > $O/ncu_pair_$2.log 2>&1
done
tail -3 $O/pair_check.log; cat $O/pair_time3.log
