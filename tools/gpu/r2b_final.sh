#!/bin/bash
# round-2 (second half) evidence: bench, reference arm, configs, launch list, top-kernel ncu + traffic
cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench_full.json 2> $O/bench_full.err; echo "bench $?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_ref.json 2>> $O/bench_full.err; echo "ref $?"
for c in c1 c2 c3 c4 c5; do timeout 600 python tools/run_config.py $c; done > $O/configs_b200.jsonl 2> $O/configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-micro --no-cpu > $O/ncu_bench.log 2>&1
python tools/launch_table.py $O/bench_launches.csv > $O/bench_launch_table.txt 2>&1
gzip -f $O/bench_launches.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"opw_kernel|fdp_kernel|fdt_fixup|restrict_blk_kernel|restrict_fixup|prolong_warp_kernel" -c 7 -f -o $O/top_full python tools/prof_c2_top.py > $O/ncu_top.log 2>&1
python tools/ncu_traffic.py $O/top_full.ncu-rep $O/traffic_c2.json > /dev/null 2>&1
python tools/ncu_summary.py $O/top_full.ncu-rep > $O/c2_top_kernels_ncu.txt 2>&1
head -24 $O/bench_launch_table.txt
cut -c1-250 $O/configs_b200.jsonl
