# quick A/B: parity tests + assembly / sweep timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -1 >> gpurun_out/exp.log
timeout 300 python scripts/kbench.py --only assemble,gs_sweep >> gpurun_out/exp.log 2>&1
