# run a python script against several experimental library builds (dev tool):
#   bash scripts/dev/gpu_ab_script.sh "<script and args>" tag1 tag2 ...
cmd="$1"; shift
cp paper_2101_08453_b200/libwd.so /tmp/libwd_cur.so
for v in "$@"; do
  cp exp_libs/libwd_$v.so paper_2101_08453_b200/libwd.so
  echo "$v $(timeout 300 python $cmd 2>&1 | tail -1)"
done
cp /tmp/libwd_cur.so paper_2101_08453_b200/libwd.so
