for c in paper medium small; do for m in -1 0 1 2; do
  echo "cfg=$c lf=$m" >> gpurun_out/perlevel.txt
  timeout 600 python bench.py --config $c --line-from=$m --steps 3 --warmup 3 --no-e2e --no-cpu --warm 0 2>/dev/null | grep '^{' | tail -1 >> gpurun_out/perlevel.txt
done; done
