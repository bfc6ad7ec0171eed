# fused-smoother check: bitwise tests first, then all GPU tests, kernel timings, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_smoother.py -x -q > gpurun_out/pytest_smoother.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_smoother.log
[ $rc -eq 0 ] || exit 0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/kbench.py > gpurun_out/kbench.log 2>&1; echo "rc=$?" >> gpurun_out/kbench.log
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
