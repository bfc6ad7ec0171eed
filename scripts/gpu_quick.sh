# GPU tests + one paper-scale bench line (default flags)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_gpu.log
[ $rc -eq 0 ] || exit 0
timeout 900 python bench.py ${BENCH_ARGS:---steps 3 --warmup 3} > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
