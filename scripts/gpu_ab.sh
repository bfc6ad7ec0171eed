# quick A/B: smoother tests + level-0 sweep timing (twice)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_smoother.py tests/test_gpu_dist.py -x -q 2>&1 | tail -1 >> gpurun_out/exp.log
timeout 300 python scripts/kbench.py --only gs_sweep,vcycle >> gpurun_out/exp.log 2>&1
timeout 300 python scripts/kbench.py --only gs_sweep,vcycle >> gpurun_out/exp.log 2>&1
