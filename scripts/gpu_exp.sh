cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for e in 1 0 1; do
  echo "pair=$e" >> gpurun_out/exp.log
  WD_GS_PAIR=$e timeout 300 python -m pytest tests/test_gpu_smoother.py tests/test_gpu_dist.py -x -q 2>&1 | tail -1 >> gpurun_out/exp.log
  WD_GS_PAIR=$e timeout 300 python scripts/kbench.py --only gs_sweep,vcycle >> gpurun_out/exp.log 2>&1
done
