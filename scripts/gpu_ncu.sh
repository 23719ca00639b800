cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" > gpurun_out/ncu_rc.txt
ncu --set full --clock-control none --import-source on -k regex:"k_spmm|k_gemm_kmajor|k_fwd_apply|k_bwd_apply|k_extract" -s 10 -c 12 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_rc.txt
