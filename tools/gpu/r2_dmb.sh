cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
(TAG=dmb2 ENGINES=dmma_eo python tools/time_fd_sweep.py 256:32 128:32; SMG_LIB=$PWD/paper_1512_02390_b200/libsmg_dmb3.so TAG=dmb3 ENGINES=dmma_eo python tools/time_fd_sweep.py 256:32 128:32) > $O/dmb.txt 2>&1
SMG_LIB=$PWD/paper_1512_02390_b200/libsmg_dmb3.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "microbench or sweeps or c3" > $O/dmb3_tests.log 2>&1; echo "exit $?" >> $O/dmb3_tests.log
cat $O/dmb.txt; tail -2 $O/dmb3_tests.log
