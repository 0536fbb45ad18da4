cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "exit $?" >> $O/gpu_tests.log
tail -3 $O/gpu_tests.log
CFG=c4 python tools/mgcg_breakdown.py > $O/mgcg_c4.txt 2>&1; head -1 $O/mgcg_c4.txt
CFG=c2 python tools/mgcg_breakdown.py > $O/mgcg_c2.txt 2>&1; head -1 $O/mgcg_c2.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-micro > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench exit $?"
tail -c 3000 $O/bench_n1.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref exit $?"
cut -c1-400 $O/bench_ref.json
