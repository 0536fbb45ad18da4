cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
(for c in 1 0; do SMG_FDT_INLINE=$c TAG=inline$c python tools/time_fd_sweep.py 64:8 64:4 64:2 64:16 32:16; done) > $O/inline_fd.txt 2>&1
cat $O/inline_fd.txt
(for c in 1 0; do SMG_PDL=0 SMG_FDT_INLINE=$c TAG=nopdl_inline$c python tools/vcycle_time.py; done) > $O/inline_nopdl.txt 2>&1
cat $O/inline_nopdl.txt
