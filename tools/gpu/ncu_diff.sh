# ncu of the diffusion residual kernel at p = 24 (C5's top level, 256^2 elements here)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:op_kernel -c 1 -o $O/opdiff24_full python tools/prof_kernels.py --n 256 --p 24 --what diff --reps 2 > $O/ncu_opdiff.log 2>&1
