# DMMA Schwarz variant with 16 warps per CTA (build -DSMG_FDT_DMW=16) vs the default 8: timings + parity
cd $GRAFT_REPO_ROOT
O=gpurun_out
L=$PWD/paper_1512_02390_b200/libsmg_dmw16.so
for i in 1 2; do
  timeout 300 python tools/time_fd_sweep.py > /dev/null 2>&1  # warm
  echo "# default engines" >> $O/dmw_time.txt
  timeout 300 python tools/time_fd_sweep.py >> $O/dmw_time.txt 2>&1
  SMG_LIB=$L timeout 300 python tools/time_fd_sweep.py >> $O/dmw_time.txt 2>&1
  echo "# SMG_FD_ENGINE=dmma_eo" >> $O/dmw_time.txt
  SMG_FD_ENGINE=dmma_eo timeout 300 python tools/time_fd_sweep.py >> $O/dmw_time.txt 2>&1
  SMG_FD_ENGINE=dmma_eo SMG_LIB=$L timeout 300 python tools/time_fd_sweep.py >> $O/dmw_time.txt 2>&1
done
SMG_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py -x -q > $O/dmw_parity.log 2>&1; echo "exit $?" >> $O/dmw_parity.log
SMG_FD_ENGINE=dmma_eo SMG_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fd or schwarz or smooth" > $O/dmw_parity_eo.log 2>&1; echo "exit $?" >> $O/dmw_parity_eo.log
