#!/bin/bash
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"restrict_warp_kernel|restrict_fixup" -c 2 -o $O/rw_32 -f python tools/prof_kernels.py --n 128 --p 32 --what restrict --reps 1 > $O/ncu_rw32.log 2>&1
ls -la $O/rw_32.ncu-rep
