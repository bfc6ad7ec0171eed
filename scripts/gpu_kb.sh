cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/kbench.py ${KB_ARGS:-} > gpurun_out/kbench.log 2>&1; echo "rc=$?" >> gpurun_out/kbench.log
CMD="python scripts/kbench.py --only gs_sweep --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gs_fused_kernel -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_fused.log 2>&1
