cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_vtail.py -x -q > $O/vtail_tests.log 2>&1; echo "exit $?" >> $O/vtail_tests.log
python tools/vcycle_time.py > $O/vtime2.txt 2>&1
SMG_VTAIL=1 TAG=tail python tools/vcycle_time.py >> $O/vtime2.txt 2>&1
python tools/vtail_phases.py > $O/vtail_phases.txt 2>&1
