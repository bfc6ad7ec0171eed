cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_smoother.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gal.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_gal.log
[ $rc -eq 0 ] || exit 0
timeout 600 python scripts/kbench.py > gpurun_out/kbench.log 2>&1; echo "rc=$?" >> gpurun_out/kbench.log
