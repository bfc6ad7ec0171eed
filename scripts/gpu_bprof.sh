# bench (default) + ncu full capture of prolong_kernel level 0
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
CMD="python scripts/kbench.py --only prolong,restrict --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prolong_kernel" -c 1 -o gpurun_out/prof_prolong $CMD > gpurun_out/ncu_prolong.log 2>&1
