# every tensor-core GEMM launch of one timed step (skip the warm-up step's 14), full set
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-eval --prefetch 0"
ncu --set full --clock-control none --import-source on -k regex:"k_gemm" -s 14 -c 14 \
    -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_gemm.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_gemm.log
