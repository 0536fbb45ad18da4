cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -x -q -m gpu > $O/opd_tests.log 2>&1; echo "exit $?" >> $O/opd_tests.log
tail -2 $O/opd_tests.log
TAG=sfrag python tools/time_op.py 512:24:diffusion 256:24:diffusion > $O/op_time.txt 2>&1; cat $O/op_time.txt
