cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mult_sweep -c 1 -o $O/mult_full python tools/time_mult.py > $O/ncu_mult.log 2>&1
