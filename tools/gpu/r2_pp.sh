cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/pp_tests.log 2>&1; echo "exit $?" >> $O/pp_tests.log
tail -2 $O/pp_tests.log
python tools/vcycle_breakdown_cfg.py c3 > $O/bd_c3.txt 2>&1; cat $O/bd_c3.txt
python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5.txt 2>&1; tail -7 $O/bd_c5.txt
(N=128 PP=32 TAG=pp python tools/vcycle_time.py; SMG_TR_PP=0 N=128 PP=32 TAG=nopp python tools/vcycle_time.py) > $O/vc_time.txt 2>&1; cat $O/vc_time.txt
