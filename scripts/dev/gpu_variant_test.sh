# parity of one library variant (dev experiment): VARIANT=exp_libs/libwd_vN.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp $VARIANT paper_2101_08453_b200/libwd.so
timeout 900 python -m pytest tests/test_gpu_smoother.py tests/test_gpu_dist.py -x -q 2>&1 | tail -3 >> gpurun_out/variants.log
