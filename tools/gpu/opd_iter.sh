# DMMA diffusion residual: oracle check, full GPU tests, C5 breakdown, with and without (SMG_OPD=0)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python tools/diff_check.py > $O/diffcheck.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/opd_tests.log 2>&1; echo "exit $?" >> $O/opd_tests.log
timeout 600 python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5.txt 2>&1
SMG_OPD=0 timeout 600 python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5_noopd.txt 2>&1
