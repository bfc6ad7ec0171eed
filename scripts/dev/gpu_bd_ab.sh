cp paper_2101_08453_b200/libwd.so /tmp/libwd_cur.so
for v in rp0 rpz; do
  cp exp_libs/libwd_$v.so paper_2101_08453_b200/libwd.so
  for c in paper medium; do timeout 300 python scripts/kbench.py --config $c --breakdown --reps 20 > gpurun_out/bd_${v}_$c.jsonl 2>&1; done
done
cp /tmp/libwd_cur.so paper_2101_08453_b200/libwd.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_smoother.py tests/test_gpu_edge.py tests/test_gpu_variants.py tests/test_gpu_dist.py -q -x 2>&1 | tail -2
