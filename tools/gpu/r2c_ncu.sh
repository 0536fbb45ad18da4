#!/bin/bash
# ncu captures of the kernels changed in the last pass of round 2: the p = 24 tensor-core diffusion
# residual, the p = 12 one, and the cooperative coarse PCG
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"opdh_kernel" -c 1 -o $O/opdh_24c -f python tools/prof_kernels.py --n 256 --p 24 --what diff --reps 2 > $O/ncu_opdh24c.log 2>&1
REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"pcg_coop" -c 1 -o $O/pcg_coop_c -f python tools/prof_coarse_c5.py > $O/ncu_pcgc2.log 2>&1
ls -la $O/opdh_24c* $O/pcg_coop_c*
# the residual restricted in place (p_f = 16 at C4 size) and the warp-per-element p = 12 diffusion residual (C5 level 12)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"opw_kernel" -c 1 -o $O/opw16_restr -f python tools/prof_rr.py 256 16 > $O/ncu_opw16r.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"opdw_kernel" -c 1 -o $O/opdw_12 -f python tools/prof_kernels.py --n 512 --p 12 --what diff --reps 2 > $O/ncu_opdw12.log 2>&1
ls -la $O/opw16_restr* $O/opdw_12*
