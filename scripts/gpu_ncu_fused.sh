# one --set full capture of the fused sweep (level 0, paper scale) + phased phase for comparison
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/kbench.py --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gs_fused_kernel -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_fused.log
