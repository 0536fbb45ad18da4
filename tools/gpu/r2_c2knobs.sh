cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_pins_r2.py -x -q -m gpu > $O/r_tests.log 2>&1; echo "exit $?" >> $O/r_tests.log
tail -2 $O/r_tests.log
python tools/vcycle_breakdown_cfg.py c3 > $O/bd_c3.txt 2>&1; cat $O/bd_c3.txt
python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5.txt 2>&1; cat $O/bd_c5.txt
(TAG=base python tools/vcycle_time.py
for t in 41 22 21 44; do SMG_FDT_TILE=$t SMG_FDT_TILE_P=16 TAG=tile$t python tools/vcycle_time.py; done
SMG_PDL=0 TAG=nopdl python tools/vcycle_time.py
SMG_FDT_MIN_TILES=1000 TAG=mintiles1000 python tools/vcycle_time.py) > $O/c2knobs.txt 2>&1
cat $O/c2knobs.txt
