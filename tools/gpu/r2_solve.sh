cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solve_graph.py tests/test_gpu_parity.py tests/test_gpu_determinism.py -x -q -m gpu > $O/solve_tests.log 2>&1; echo "exit $?" >> $O/solve_tests.log
tail -3 $O/solve_tests.log
CFG=c4 python tools/mgcg_breakdown.py > $O/mgcg_c4.txt 2>&1; head -1 $O/mgcg_c4.txt
CFG=c2 python tools/mgcg_breakdown.py > $O/mgcg_c2.txt 2>&1; head -1 $O/mgcg_c2.txt
CFG=c5 python tools/mgcg_breakdown.py > $O/mgcg_c5.txt 2>&1; cat $O/mgcg_c5.txt
python tools/vcycle_breakdown_cfg.py c5 > $O/bd_c5.txt 2>&1; cat $O/bd_c5.txt
python tools/vcycle_breakdown_cfg.py c3 > $O/bd_c3.txt 2>&1; cat $O/bd_c3.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"opd_kernel" -c 1 -o $O/opd24_full python tools/prof_kernels.py --n 256 --p 24 --what diff --reps 2 > $O/ncu_opd24.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"restrict" -c 1 -o $O/restrict32_full python tools/prof_kernels.py --n 128 --p 32 --what restrict --reps 2 > $O/ncu_r32.log 2>&1
ls $O/*.ncu-rep
