cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/fused_tests.log 2>&1; echo "exit $?" >> $O/fused_tests.log
python tools/vcycle_breakdown.py > $O/breakdown.txt 2>&1
python tools/vcycle_time.py > $O/vtime4.txt 2>&1
SMG_FDT_FUSED=0 TAG=unfused python tools/vcycle_time.py >> $O/vtime4.txt 2>&1
