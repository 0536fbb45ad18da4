cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/variants.txt
for v in "TAG=default" "SMG_RR_FUSED=0 TAG=rr0" "SMG_RR_FUSED=3 TAG=rr3" "SMG_TR_BLK=0 TAG=blk0"; do
  env $v python tools/vcycle_time.py >> $O/variants.txt 2>&1
done
