# quick variant probes: C2 V-cycle vs fused residual+restriction tile; p=32 DMMA tiles
cd $GRAFT_REPO_ROOT
O=gpurun_out
: > $O/qv.txt
for m in 148 512 1024 4096; do echo "== SMG_RR_MIN_CTAS=$m" >> $O/qv.txt; SMG_RR_MIN_CTAS=$m timeout 300 python tools/vcycle_time.py >> $O/qv.txt 2>&1; done
for t in 0 41 21; do echo "== p32 dmma_eo tile $t" >> $O/qv.txt; SMG_FDT_TILE=$t SMG_FDT_TILE_P=32 ENGINES=dmma_eo timeout 300 python tools/fd_diag.py 256:32 128:32 2>&1 | grep -v skip=1 >> $O/qv.txt; done
