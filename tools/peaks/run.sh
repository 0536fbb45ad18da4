nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./tools/peaks/fp64_peaks > gpurun_out/peaks.log 2>&1
kill $SMI
nproc >> gpurun_out/peaks.log; lscpu | head -20 >> gpurun_out/peaks.log
cat gpurun_out/peaks.log
