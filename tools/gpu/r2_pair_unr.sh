#!/bin/bash
O=gpurun_out
: > $O/pair_unr.log
for U in 1 3 4 32; do
SMG_LIB=$PWD/paper_1512_02390_b200/libsmg_u$U.so ENGINES=pair TAG=unr$U python tools/time_fd_sweep.py 256:8 256:12 256:16 256:24 256:32 >> $O/pair_unr.log 2>&1
done
cat $O/pair_unr.log
