cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -x -q -m gpu > $O/rr_tests.log 2>&1; echo "exit $?" >> $O/rr_tests.log
tail -2 $O/rr_tests.log
(TAG=rrhoist python tools/vcycle_time.py; TAG=rrhoist python tools/vcycle_time.py; N=256 PP=16 TAG=rrhoist python tools/vcycle_time.py) > $O/rr_time.txt 2>&1; cat $O/rr_time.txt
