# diffusion operator iteration: full GPU tests, C5 per-component breakdown (shared-memory vs constant-bank D)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/diff_tests.log 2>&1; echo "exit $?" >> $O/diff_tests.log
timeout 600 python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5.txt 2>&1
SMG_LIB=build/libsmg_dconst.so timeout 600 python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5_const.txt 2>&1
