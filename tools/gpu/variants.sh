cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/variants.txt
for v in "TAG=default" "SMG_RR_FUSED=0 TAG=rr0" "SMG_RR_FUSED=3 TAG=rr3" "SMG_TR_WARP=0 TAG=trw0" "SMG_PDL=0 TAG=pdl0" "SMG_RR_FUSED=3 SMG_PDL=0 TAG=rr3pdl0"; do
  env $v python tools/vcycle_time.py >> $O/variants.txt 2>&1
done
