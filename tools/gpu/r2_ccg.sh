# one-CTA coarse CG: tests, timings vs the grid path, default bench
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_coarse_cta.py tests/test_gpu_parity.py tests/test_pins_r2.py tests/test_gpu_determinism.py -x -q > $O/ccg_tests.log 2>&1; echo "exit $?" >> $O/ccg_tests.log
timeout 300 python tools/coarse_cta_time.py > $O/ccg_time.txt 2>&1
SMG_CCG_CTA=0 timeout 300 python tools/coarse_cta_time.py >> $O/ccg_time.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
