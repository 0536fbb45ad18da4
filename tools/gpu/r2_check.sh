# full GPU suite + contraction microbench (round 2)
cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
./tools/micro/contract2 > $O/contract2.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
tail -5 $O/gpu_tests.log
cat $O/contract2.log
