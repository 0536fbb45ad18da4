cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout -k 10 200 python -m pytest tests/test_gpu_halo.py -x -q -o faulthandler_timeout=150 > $O/halo2.log 2>&1; echo "exit $?" >> $O/halo2.log
timeout -k 10 400 python -m pytest tests/test_gpu_strips.py tests/test_gpu_coarse_cta.py -x -q >> $O/halo2.log 2>&1; echo "exit $?" >> $O/halo2.log
