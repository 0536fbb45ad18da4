cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_chain.py -x -q -m gpu > $O/chain_tests.log 2>&1; echo "exit $?" >> $O/chain_tests.log
tail -2 $O/chain_tests.log
for c in 1 0; do SMG_CHAIN=$c TAG=chain$c python tools/vcycle_time.py; SMG_CHAIN=$c TAG=chain$c N=128 PP=32 python tools/vcycle_time.py; done > $O/chain_time.txt 2>&1
cat $O/chain_time.txt
CFG=c4 python tools/mgcg_breakdown.py > $O/mgcg_c4.txt 2>&1; cat $O/mgcg_c4.txt
CFG=c2 python tools/mgcg_breakdown.py > $O/mgcg_c2.txt 2>&1; cat $O/mgcg_c2.txt
