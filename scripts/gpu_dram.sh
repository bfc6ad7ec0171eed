# per-launch DRAM bytes + duration of every kernel of one bench step (ncu; serialized, cold)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --warm 0"
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/dram.csv $CMD > gpurun_out/ncu_dram.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_dram.log
# the residual variant of the fused sweep (first sweep of a cycle in wd_solve)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:gs_fused_kernel<.bool.1>' -c 1 -o gpurun_out/prof_fused_res $CMD > gpurun_out/ncu_fused_res.log 2>&1
