cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/blas_tests.log 2>&1; echo "exit $?" >> $O/blas_tests.log
tail -2 $O/blas_tests.log
CFG=c4 python tools/mgcg_breakdown.py > $O/mgcg_c4.txt 2>&1; cat $O/mgcg_c4.txt
CFG=c5 python tools/mgcg_breakdown.py > $O/mgcg_c5.txt 2>&1; cat $O/mgcg_c5.txt
