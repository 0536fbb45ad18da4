cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > $O/quick_tests.log 2>&1; echo "exit $?" >> $O/quick_tests.log
python tools/vcycle_breakdown.py > $O/breakdown.txt 2>&1
python tools/vcycle_time.py > $O/vtime5.txt 2>&1
