# Schwarz kernel: tile-shape variants at p = 24, 32
cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/fd_tiles.txt
for t in 0 21 11; do
  echo "== SMG_FDT_TILE=$t" >> $O/fd_tiles.txt
  SMG_FDT_TILE=$t timeout 300 python tools/fd_diag.py 256:24 256:32 128:32 >> $O/fd_tiles.txt 2>&1
done
