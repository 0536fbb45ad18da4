# native NCCL halos (smg_halo_*) on one GPU + coarse CTA CG tests
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_strips.py tests/test_gpu_coarse_cta.py -x -q > $O/halo_tests.log 2>&1; echo "exit $?" >> $O/halo_tests.log
