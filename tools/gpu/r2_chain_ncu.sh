cd $GRAFT_REPO_ROOT
O=gpurun_out
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py -x -q -m gpu > $O/chain_tests.log 2>&1; echo "exit $?" >> $O/chain_tests.log
tail -3 $O/chain_tests.log
for c in 1 0; do SMG_CHAIN=$c TAG=chain$c python tools/vcycle_time.py; SMG_CHAIN=$c TAG=chain$c N=128 PP=32 python tools/vcycle_time.py; done > $O/chain_time.txt 2>&1
cat $O/chain_time.txt
# ncu: p=32 DMMA Schwarz (C3 top level) and p=16 DFMA at 256^2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fdt_kernel" -c 1 -o $O/fdt32_full python tools/prof_kernels.py --n 128 --p 32 --what fd --reps 2 > $O/ncu_fdt32.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"fdt_kernel" -c 1 -o $O/fdt16_full python tools/prof_kernels.py --n 256 --p 16 --what fd --reps 2 > $O/ncu_fdt16.log 2>&1
ls -la $O/*.ncu-rep
