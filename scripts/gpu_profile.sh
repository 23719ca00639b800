# Round profile capture: plain run, launch list, full capture of the top kernels (1 GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" > gpurun_out/ncu_rc.txt
ncu --set full --clock-control none --import-source on -k regex:"k_spmm_pipe|k_gemm_kmajor|k_fwd_row|k_bwd_row|k_gemm_wgrad|k_extract_fill|k_ce_row" -s 40 -c 16 -o gpurun_out/prof_r01 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_rc.txt
