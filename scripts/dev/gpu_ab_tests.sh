# run a test selection against an experimental library build (dev tool): $1 = lib tag, rest = pytest args
cp paper_2101_08453_b200/libwd.so /tmp/libwd_cur.so
cp exp_libs/libwd_$1.so paper_2101_08453_b200/libwd.so
shift
timeout 900 python -m pytest "$@" 2>&1 | tail -3
cp /tmp/libwd_cur.so paper_2101_08453_b200/libwd.so
