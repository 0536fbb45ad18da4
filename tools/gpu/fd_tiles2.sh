# Schwarz kernel: tile-shape variants at p = 16, 24, 32 (DFMA), and the default engines
cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/fd_tiles2.txt
for t in 0 41 22 21; do
  echo "== SMG_FDT_TILE=$t" >> $O/fd_tiles2.txt
  SMG_FDT_TILE=$t ENGINES=dfma timeout 300 python tools/fd_diag.py 256:16 64:16 256:24 256:32 >> $O/fd_tiles2.txt 2>&1
done
