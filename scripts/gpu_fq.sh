# quick fused-smoother iteration: bitwise tests + kernel timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_smoother.py -x -q > gpurun_out/pytest_smoother.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_smoother.log
[ $rc -eq 0 ] || exit 0
timeout 600 python scripts/kbench.py ${KB_ARGS:-} > gpurun_out/kbench.log 2>&1; echo "rc=$?" >> gpurun_out/kbench.log
