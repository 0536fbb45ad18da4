cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
./tools/micro/contract2 > $O/contract2.log 2>&1
timeout 900 python -m pytest tests/test_pins_r2.py -x -q -m gpu > $O/pins_r2.log 2>&1; echo "exit $?" >> $O/pins_r2.log
tail -3 $O/pins_r2.log
cat $O/contract2.log
