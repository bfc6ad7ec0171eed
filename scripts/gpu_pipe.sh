cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q > gpurun_out/pytest_pipe.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pipe.log
