cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu > $O/inline_tests.log 2>&1; echo "exit $?" >> $O/inline_tests.log
tail -3 $O/inline_tests.log
(for c in 1 0; do SMG_FDT_INLINE=$c TAG=inline$c python tools/vcycle_time.py; SMG_FDT_INLINE=$c TAG=inline$c N=128 PP=32 python tools/vcycle_time.py; SMG_FDT_INLINE=$c TAG=inline$c N=256 PP=16 python tools/vcycle_time.py; done) > $O/inline_time.txt 2>&1
cat $O/inline_time.txt
