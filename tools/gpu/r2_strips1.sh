cd $GRAFT_REPO_ROOT
O=gpurun_out
SMG_BENCH_STRIPS=1 timeout -k 10 400 python bench.py --steps 5 --warmup 3 > $O/strips1.json 2> $O/strips1.err; echo "exit $?" >> $O/strips1.err
SMG_BENCH_STRIPS=1 SMG_HALO=torch timeout -k 10 400 python bench.py --steps 5 --warmup 3 >> $O/strips1.json 2>> $O/strips1.err; echo "exit $?" >> $O/strips1.err
