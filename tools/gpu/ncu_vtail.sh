cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:vtail_kernel -c 1 -o $O/vtail_full python tools/vtail_phases.py > $O/ncu_vtail.log 2>&1
