cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_smoother.py tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q 2>&1 | tail -1 >> gpurun_out/exp.log
timeout 300 python scripts/kbench.py > gpurun_out/kb.log 2>&1
grep galerkin gpurun_out/kb.log >> gpurun_out/exp.log
