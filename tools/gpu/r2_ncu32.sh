cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fdt_kernel" -c 1 -o /tmp/f32 python tools/prof_kernels.py --n 128 --p 32 --what fd --reps 2 > $O/ncu_f32.log 2>&1
python tools/ncu_summary.py /tmp/f32.ncu-rep > $O/f32_summary.txt 2>&1
ncu -i /tmp/f32.ncu-rep --page raw --csv > $O/f32_raw.csv 2>&1
ncu -i /tmp/f32.ncu-rep --page source --csv --print-source cuda,sass > $O/f32_source.csv 2>&1
ls -la $O/f32*
