cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/r2_tests.log 2>&1; echo "exit $?" >> $O/r2_tests.log
tail -3 $O/r2_tests.log
python tools/vcycle_breakdown_cfg.py c3 > $O/bd_c3.txt 2>&1; cat $O/bd_c3.txt
python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5.txt 2>&1; tail -7 $O/bd_c5.txt
(TAG=r2 python tools/vcycle_time.py; N=128 PP=32 TAG=r2 python tools/vcycle_time.py; SMG_RESTRICT2=0 N=128 PP=32 TAG=norestrict2 python tools/vcycle_time.py) > $O/vc_time.txt 2>&1; cat $O/vc_time.txt
