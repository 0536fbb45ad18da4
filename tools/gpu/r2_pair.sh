#!/bin/bash
# paired-line Schwarz engine: parity against the default engine and the oracle, then timing
set -x
python tools/pair_check.py 8 12 16 24 32 > gpurun_out/pair_check.log 2>&1; echo "rc $?" >> gpurun_out/pair_check.log
ENGINES=dfma,dmma_eo,pair TAG=r2 python tools/time_fd_sweep.py 256:8 256:12 256:16 256:24 256:32 128:32 64:16 > gpurun_out/pair_time.log 2>&1
cat gpurun_out/pair_check.log gpurun_out/pair_time.log
