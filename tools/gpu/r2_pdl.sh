cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_solve_graph.py -x -q -m gpu > $O/pdl_tests.log 2>&1; echo "exit $?" >> $O/pdl_tests.log
tail -2 $O/pdl_tests.log
(TAG=pdlhoist python tools/vcycle_time.py; N=128 PP=32 TAG=pdlhoist python tools/vcycle_time.py; N=256 PP=16 TAG=pdlhoist python tools/vcycle_time.py) > $O/pdl_time.txt 2>&1
cat $O/pdl_time.txt
