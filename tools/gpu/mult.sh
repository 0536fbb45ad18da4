cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_mult.py -x -q > $O/mult_tests.log 2>&1; echo "exit $?" >> $O/mult_tests.log
timeout 900 python tools/time_mult.py > $O/mult_time.txt 2>&1
