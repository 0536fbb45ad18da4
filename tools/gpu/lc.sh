cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pins_r2.py tests/test_gpu_determinism.py -x -q -m gpu > $O/lc_tests.log 2>&1; echo "exit $?" >> $O/lc_tests.log
tail -3 $O/lc_tests.log
SMG_FDT_LC=1 ENGINES=dfma,dmma_eo python tools/time_fd_sweep.py > $O/lc1.txt 2>&1
SMG_FDT_LC=2 ENGINES=dfma python tools/time_fd_sweep.py > $O/lc2.txt 2>&1
cat $O/lc1.txt $O/lc2.txt
