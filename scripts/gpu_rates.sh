cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python scripts/rate_study.py > gpurun_out/rate_study.jsonl 2> gpurun_out/rate_study.err; echo "rc=$?" >> gpurun_out/rate_study.err
