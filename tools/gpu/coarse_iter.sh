# coarse FFT pseudo-inverse iteration: full GPU tests, coarse timings, C5/C4 breakdowns
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/coarse_tests.log 2>&1; echo "exit $?" >> $O/coarse_tests.log
python tools/time_coarse.py 512 > $O/coarse_t.txt 2>&1; python tools/time_coarse.py 256 >> $O/coarse_t.txt 2>&1
timeout 600 python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5.txt 2>&1
timeout 600 python tools/vcycle_breakdown_cfg.py c4 > $O/bd_c4.txt 2>&1
