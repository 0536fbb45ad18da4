cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/fd_engine.txt
for v in "TAG=dfma" "SMG_FD_ENGINE=dmma_eo TAG=dmma_eo" "SMG_FD_ENGINE=dmma TAG=dmma_dense"; do
  echo "== $v" >> $O/fd_engine.txt
  env $v python tools/vcycle_breakdown.py 2>&1 | head -5 >> $O/fd_engine.txt
  env $v python tools/vcycle_time.py >> $O/fd_engine.txt 2>&1
done
