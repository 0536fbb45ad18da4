#!/bin/bash
# ncu captures of the kernels changed in the last pass of round 2: the p = 24 tensor-core diffusion
# residual, the p = 12 one, and the cooperative coarse PCG
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"opdh_kernel" -c 1 -o $O/opdh_24c -f python tools/prof_kernels.py --n 256 --p 24 --what diff --reps 2 > $O/ncu_opdh24c.log 2>&1
REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"pcg_coop" -c 1 -o $O/pcg_coop_c -f python tools/prof_coarse_c5.py > $O/ncu_pcgc2.log 2>&1
ls -la $O/opdh_24c* $O/pcg_coop_c*
