cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout -k 10 400 python -m pytest tests/test_gpu_coarse_cta.py -x -q > $O/cta2.log 2>&1; echo "exit $?" >> $O/cta2.log
