# A/B of library builds on the per-level breakdown (dev tool)
cp paper_2101_08453_b200/libwd.so /tmp/libwd_cur.so
for v in "$@"; do
  cp exp_libs/libwd_$v.so paper_2101_08453_b200/libwd.so
  timeout 300 python scripts/kbench.py --config paper --breakdown --reps 20 > gpurun_out/bd_$v.jsonl 2>&1
done
cp /tmp/libwd_cur.so paper_2101_08453_b200/libwd.so
