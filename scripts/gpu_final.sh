# round-end style check: smoke, GPU tests, reference arm, bench, launch list, ncu capture of the top kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --warm 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gs_fused_kernel -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_tma_kernel -c 1 -o gpurun_out/prof_apply $CMD > gpurun_out/ncu_apply.log 2>&1
# the residual variant of the fused sweep (first sweep of a cycle in wd_solve)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:gs_fused_kernel<.bool.1>' -c 1 -o gpurun_out/prof_fused_res $CMD > gpurun_out/ncu_fused_res.log 2>&1
echo done >> gpurun_out/smoke.log
