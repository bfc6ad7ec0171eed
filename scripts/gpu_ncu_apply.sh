cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python scripts/kbench.py --reps 2"
timeout 600 $CMD > gpurun_out/kb_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:apply_tma_kernel -s 2 -c 1 -o gpurun_out/prof_apply_tma $CMD > gpurun_out/ncu_apply.log 2>&1
echo "rc=$?" >> gpurun_out/kb_plain.log
