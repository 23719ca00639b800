# Quick A/B: bench lines (no CPU baseline, no eval) under env settings given as args.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/tune.txt
for setting in "$@"; do
  env $setting timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-eval > gpurun_out/tune_one.json 2> gpurun_out/tune_one.err
  echo "== $setting rc=$?" >> gpurun_out/tune.txt
  python scripts/show_bench.py gpurun_out/tune_one.json >> gpurun_out/tune.txt 2>&1
done
cat gpurun_out/tune.txt
