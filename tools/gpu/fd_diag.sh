# Schwarz-kernel diagnostics at the smoother-microbench sizes + ncu of the p=24 kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python tools/fd_diag.py > $O/fd_diag.txt 2>&1
ENGINES=dfma timeout 600 ncu --set full --import-source on --clock-control none -k regex:fdt_kernel -c 1 -o $O/fdt24_full python tools/fd_diag.py 256:24 > $O/ncu_fdt24.log 2>&1
