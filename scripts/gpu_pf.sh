cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for pf in 1 2 0; do
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-eval --prefetch $pf > gpurun_out/pf$pf.json 2> gpurun_out/pf$pf.err
done
GGB_PREFETCH_PRIORITY=same timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-eval --prefetch 2 > gpurun_out/pf2same.json 2> gpurun_out/pf2same.err
