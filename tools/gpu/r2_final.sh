cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/final_smi.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_full.json 2> $O/bench_full.err; echo "bench $?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2>> $O/bench_full.err; echo "ref $?"
for c in c1 c2 c3 c4 c5; do timeout 600 python tools/run_config.py $c; done > $O/configs_b200.jsonl 2> $O/configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-micro --no-cpu > $O/ncu_bench.log 2>&1
python tools/launch_table.py $O/bench_launches.csv > $O/bench_launch_table.txt 2>&1
gzip -f $O/bench_launches.csv
head -30 $O/bench_launch_table.txt
cat $O/configs_b200.jsonl | cut -c1-300
