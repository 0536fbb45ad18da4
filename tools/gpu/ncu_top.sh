cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"op_kernel|fdt_kernel|fdt_fixup|restrict_kernel|prolong_kernel" -c 5 -o $O/top_full python tools/prof_c2_top.py > $O/ncu_top.log 2>&1
