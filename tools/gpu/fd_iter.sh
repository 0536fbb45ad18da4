# Schwarz-kernel iteration: parity subset, timings, phase profile (profile build)
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/iter_tests.log 2>&1; echo "exit $?" >> $O/iter_tests.log
ENGINES=dfma timeout 600 python tools/fd_diag.py 256:16 256:24 256:32 128:32 64:16 > $O/iter_diag.txt 2>&1
SMG_LIB=build/libsmg_prof.so SMG_FD_ENGINE=dfma timeout 300 python tools/fdt_phases.py 256:16 256:24 256:32 > $O/iter_phases.txt 2>&1
