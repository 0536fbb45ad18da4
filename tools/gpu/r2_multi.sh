# Functional check of the N > 1 bench path on ONE GPU: 2 ranks over gloo
# (host-staged halos) -- not a measurement; the NCCL path needs 2 devices.
cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py tests/test_pins_r2.py tests/test_integration_stub.py -x -q -m gpu > $O/tr_tests.log 2>&1; echo "exit $?" >> $O/tr_tests.log
tail -2 $O/tr_tests.log
python tools/vcycle_breakdown_cfg.py c3 > $O/bd_c3.txt 2>&1; cat $O/bd_c3.txt
python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5.txt 2>&1; tail -7 $O/bd_c5.txt
(TAG=tr python tools/vcycle_time.py; N=128 PP=32 TAG=tr python tools/vcycle_time.py) > $O/vc_time.txt 2>&1; cat $O/vc_time.txt
SMG_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > $O/bench_n2_gloo.json 2> $O/bench_n2_gloo.err; echo "n2 exit $?"
tail -c 1500 $O/bench_n2_gloo.json; tail -3 $O/bench_n2_gloo.err
# ncu: every kernel of one eager C2 V-cycle, summarised on the box (the report is large)
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -o /tmp/c2vc python tools/vcycle_once.py > $O/ncu_c2vc.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py /tmp/c2vc.ncu-rep > $O/c2_vcycle_ncu_summary.txt 2>&1
ncu -i /tmp/c2vc.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active > $O/c2_vcycle_ncu_raw.csv 2>&1
CFG=c4 timeout 600 ncu --set full --clock-control none -k regex:"dot_kernel|cg_update_kernel|dot2_kernel|cg_direction_kernel" -c 4 -o /tmp/blas python tools/mgcg_breakdown.py > $O/ncu_blas.log 2>&1; echo "ncu blas exit $?"
python tools/ncu_summary.py /tmp/blas.ncu-rep > $O/blas_c4_ncu_summary.txt 2>&1
du -sh $O
