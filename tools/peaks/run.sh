nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/peaks/fp64_peaks > gpurun_out/peaks.log 2>&1
kill $SMI
nproc >> gpurun_out/peaks.log; lscpu | head -20 >> gpurun_out/peaks.log
cat gpurun_out/peaks.log
# DMMA and DFMA pipes together (one datapath: any mix sums to ~37 TF)
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/peaks/fp64_mixed tools/peaks/fp64_mixed.cu && ./tools/peaks/fp64_mixed > gpurun_out/fp64_mixed.log 2>&1
