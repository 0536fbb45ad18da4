#!/bin/bash
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"opdh_kernel" -c 1 -o $O/opdh_24 -f python tools/prof_kernels.py --n 256 --p 24 --what diff --reps 2 > $O/ncu_opdh24.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"opdh_kernel" -c 1 -o $O/opdh_32 -f python tools/prof_kernels.py --n 128 --p 32 --what op --reps 2 > $O/ncu_opdh32.log 2>&1
ls -la $O/opdh*
