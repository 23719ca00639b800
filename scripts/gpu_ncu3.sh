cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --prefetch 0"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_spmm_pipe" -s 6 -c 4 -o gpurun_out/prof_spmm $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" > gpurun_out/ncu_rc.txt
