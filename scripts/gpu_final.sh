# round-end style runs, one part per gpurun call (at most one ncu per call):
#   bash scripts/gpu_final.sh check     smoke, pytest -m gpu, reference arm, default bench line
#   bash scripts/gpu_final.sh launches  ncu launch list (+ DRAM bytes) of one bench step
#   bash scripts/gpu_final.sh plain     ncu --set full of the level-0 fused sweep (plain)
#   bash scripts/gpu_final.sh res       ncu --set full of its residual variant
#   bash scripts/gpu_final.sh apply     ncu --set full of the TMA residual
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --warm 0"
case "$1" in
check)
    timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
    timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
    timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
    timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
    ;;
launches)
    timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
    timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
    echo "rc=$?" >> gpurun_out/ncu_launch.log
    ;;
plain)
    timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:gs_fused2_kernel<.int.0' -c 1 -o gpurun_out/prof_plain $CMD > gpurun_out/ncu_plain.log 2>&1
    echo "rc=$?" >> gpurun_out/ncu_plain.log
    ;;
res)
    timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k 'regex:gs_fused2_kernel<.int.1' -c 1 -o gpurun_out/prof_res $CMD > gpurun_out/ncu_res.log 2>&1
    echo "rc=$?" >> gpurun_out/ncu_res.log
    ;;
apply)
    timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on \
        -k regex:apply_tma_kernel -c 1 -o gpurun_out/prof_apply $CMD > gpurun_out/ncu_apply.log 2>&1
    echo "rc=$?" >> gpurun_out/ncu_apply.log
    ;;
esac
