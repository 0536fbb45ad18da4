# Shared-memory factor build (SMG_FDT_SMEMF) vs default: timings + parity, then the default GPU suite and smoke
cd $GRAFT_REPO_ROOT
O=gpurun_out
L=paper_1512_02390_b200/libsmg_smemf.so
timeout 300 python tools/time_fd_sweep.py > $O/smemf_time.txt 2>&1
SMG_LIB=$PWD/$L timeout 300 python tools/time_fd_sweep.py >> $O/smemf_time.txt 2>&1
timeout 300 python tools/time_fd_sweep.py >> $O/smemf_time.txt 2>&1
SMG_LIB=$PWD/$L timeout 300 python tools/time_fd_sweep.py >> $O/smemf_time.txt 2>&1
SMG_LIB=$PWD/$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -x -q > $O/smemf_parity.log 2>&1; echo "exit $?" >> $O/smemf_parity.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
