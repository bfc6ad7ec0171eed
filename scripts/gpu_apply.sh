cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_gpu.log
[ $rc -eq 0 ] || exit 0
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:apply_kernel -s 1 -c 1 -o gpurun_out/prof_apply $CMD > gpurun_out/ncu_apply.log 2>&1
echo "done rc=$?" >> gpurun_out/plain.log
