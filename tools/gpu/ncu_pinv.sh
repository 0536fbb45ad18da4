cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pinv_cluster -c 1 -o $O/pinv_full python tools/vcycle_time.py > $O/ncu_pinv.log 2>&1
