cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py tests/test_pins_r2.py tests/test_gpu_determinism.py -x -q -m gpu > $O/dm_tests.log 2>&1; echo "exit $?" >> $O/dm_tests.log
tail -3 $O/dm_tests.log
ENGINES=dfma,dmma_eo TAG=dm2 python tools/time_fd_sweep.py 256:24 256:32 128:32 > $O/dm2.txt 2>&1
cat $O/dm2.txt
for c in 1 0; do SMG_CHAIN=$c TAG=chain$c python tools/vcycle_time.py; SMG_CHAIN=$c TAG=chain$c N=128 PP=32 python tools/vcycle_time.py; done > $O/chain_time.txt 2>&1
cat $O/chain_time.txt
