cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/kbench.py ${KB_ARGS:---apply-variants 0,1,2,3} > gpurun_out/kbench.log 2>&1; echo "rc=$?" >> gpurun_out/kbench.log
