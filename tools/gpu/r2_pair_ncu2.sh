#!/bin/bash
O=gpurun_out
for cfg in "128 32" "256 24" "256 16"; do set -- $cfg
SMG_FD_ENGINE=pair timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fdp_kernel" -c 1 \
     -o $O/fdp_$2 -f python tools/prof_kernels.py --n $1 --p $2 --what fd --reps 2 > $O/ncu_pair_$2.log 2>&1
done
ls -la $O/*.ncu-rep
