cp paper_2101_08453_b200/libwd.so /tmp/libwd_cur.so
for v in "$@"; do
  cp exp_libs/libwd_$v.so paper_2101_08453_b200/libwd.so
  for c in small medium; do timeout 300 python scripts/kbench.py --config $c --breakdown --reps 20 > gpurun_out/bd_${v}_$c.jsonl 2>&1; done
done
cp /tmp/libwd_cur.so paper_2101_08453_b200/libwd.so
