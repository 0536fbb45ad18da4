# C2 V-cycle with the p=16 Schwarz tile forced (graph replay, L2 flushed)
cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/c2_tiles.txt
for t in 0 42 41 22 21; do
  echo "== p16 tile $t" >> $O/c2_tiles.txt
  SMG_FDT_TILE=$t SMG_FDT_TILE_P=16 timeout 300 python tools/vcycle_time.py >> $O/c2_tiles.txt 2>&1
done
