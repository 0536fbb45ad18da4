#!/bin/bash
# paired-line Schwarz engine: parity against the default engine and the oracle, then timing
set -x
python tools/pair_check.py 16 > gpurun_out/pair_check.log 2>&1; echo "rc $?" >> gpurun_out/pair_check.log
ENGINES=dfma,pair TAG=r2 python tools/time_fd_sweep.py 256:16 64:16 128:16 > gpurun_out/pair_time.log 2>&1
cat gpurun_out/pair_check.log gpurun_out/pair_time.log
