cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --prefetch 0"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches2.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" > gpurun_out/ncu_rc.txt
ncu --set full --clock-control none --import-source on -k regex:"k_fwd_row|k_bwd_row|k_gemm_kmajor|k_ce_row|k_gemm_wgrad" -s 12 -c 12 -o gpurun_out/prof_c2b $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_rc.txt
