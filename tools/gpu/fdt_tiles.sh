cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/fdt_tiles.txt
for v in "TAG=default" "SMG_FDT_TILE=21" "SMG_FDT_TILE=11" "SMG_FDT_MIN_TILES=300" "SMG_FDT_MIN_TILES=600" "SMG_FDT_MIN_TILES=1000"; do
  echo "== $v" >> $O/fdt_tiles.txt
  env $v python tools/vcycle_breakdown.py 2>&1 | head -5 >> $O/fdt_tiles.txt
  env $v python tools/vcycle_time.py >> $O/fdt_tiles.txt 2>&1
done
