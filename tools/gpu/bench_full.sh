cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>> $O/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-micro --no-cpu > $O/ncu_bench.log 2>&1
python tools/launch_table.py $O/bench_launches.csv > $O/bench_launch_table.txt 2>&1
