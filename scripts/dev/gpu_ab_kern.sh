# A/B of library builds on selected level-0 kernels (dev tool): args = lib tags
cp paper_2101_08453_b200/libwd.so /tmp/libwd_cur.so
for v in "$@"; do
  cp exp_libs/libwd_$v.so paper_2101_08453_b200/libwd.so
  for r in 1 2; do
    timeout 300 python scripts/kbench.py --config paper --only ${KERNELS:-gs_sweep,gs_sweep_res} --reps 20 > gpurun_out/kb_${v}_$r.jsonl 2>&1
  done
done
cp /tmp/libwd_cur.so paper_2101_08453_b200/libwd.so
