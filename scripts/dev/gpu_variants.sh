# time level-0 fused sweep for each library variant in exp_libs/ (dev experiment)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2101_08453_b200/libwd.so /tmp/libwd_orig.so
for f in ${VARIANTS:-$(ls exp_libs/*.so)} exp_libs/libwd_v0.so; do
  cp $f paper_2101_08453_b200/libwd.so
  echo "== $f" >> gpurun_out/variants.log
  timeout 300 python scripts/kbench.py --only ${KERNELS:-gs_sweep} --reps 20 >> gpurun_out/variants.log 2>&1
done
cp /tmp/libwd_orig.so paper_2101_08453_b200/libwd.so
