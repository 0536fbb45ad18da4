cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/quick_tests.log 2>&1; echo "exit $?" >> $O/quick_tests.log
python tools/vcycle_breakdown.py > $O/breakdown.txt 2>&1
python tools/vcycle_time.py > $O/vtime5.txt 2>&1
SMG_LVL_FUSED=0 TAG=lvl0 python tools/vcycle_time.py >> $O/vtime5.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/vlaunch.csv python tools/vcycle_time.py > $O/ncu_v.log 2>&1
python tools/launch_table.py $O/vlaunch.csv > $O/vlaunch_table.txt 2>&1
