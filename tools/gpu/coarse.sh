cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "coarse or v_cycle or c1_solver or c2_full" > $O/coarse_tests.log 2>&1; echo "exit $?" >> $O/coarse_tests.log
python tools/vcycle_breakdown.py > $O/breakdown.txt 2>&1
SMG_PINV_CLUSTER=0 python tools/vcycle_breakdown.py 2>&1 | tail -1 >> $O/breakdown.txt
python tools/vcycle_time.py > $O/vtime3.txt 2>&1
