# Full GPU test suite, smoke, bench (ours + reference arm), launch list, ncu of the top-level kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_full.json 2> $O/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>> $O/bench_full.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-micro --no-cpu > $O/ncu_bench.log 2>&1
python tools/launch_table.py $O/bench_launches.csv > $O/bench_launch_table.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"opw_kernel|fdt_kernel|fdt_fixup|restrict_blk|prolong_warp" -c 5 -o $O/top_full python tools/prof_c2_top.py > $O/ncu_top.log 2>&1
