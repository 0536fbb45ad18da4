cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_strips.py -x -q -m gpu > $O/sg_tests.log 2>&1; echo "exit $?" >> $O/sg_tests.log
tail -3 $O/sg_tests.log
grep -E "Error|error" $O/sg_tests.log | head -5
