# GPU tests, then (only if they pass) the bench command plain, its ncu launch list,
# and one --set full capture each of the level-0 GS phase and the assembly/residual kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "rc=$rc" >> gpurun_out/pytest_gpu.log
[ $rc -eq 0 ] || exit 0
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gs_phase_kernel -s 4 -c 1 -o gpurun_out/prof_gs $CMD > gpurun_out/ncu_gs.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"assemble_kernel|apply_kernel" -c 2 -o gpurun_out/prof_asm $CMD > gpurun_out/ncu_asm.log 2>&1
echo "done rc=$?" >> gpurun_out/plain.log
