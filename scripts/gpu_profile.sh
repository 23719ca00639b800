# Round profile capture: plain run, launch list, one full capture per hot kernel (1 GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R=${ROUND:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-eval"
[ -z "$ONLY" ] && $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" > gpurun_out/ncu_rc.txt
# ncu matches base names (no template args): per step the SpMM pipe runs fwd fp32 x2
# (layers 2, 3; layer 1 is pre-aggregated) then bwd bf16 x2; per step 6 fwd + 4 dX
# k_gemm_kmajor and 6 k_gemm_wgrad. Skip the warm-up step's launches of each
# kernel, capture one of the timed ones
for spec in "spmm_fwd:k_spmm_pipe:4" "spmm_bwd:k_spmm_pipe:6" "gemm_fwd:k_gemm_kmajor:12" "gemm_dx:k_gemm_kmajor:17" \
            "gemm_wgrad:k_gemm_wgrad:7" "fwd_row:k_fwd_row:4" "bwd_row:k_bwd_row:4" "extract:k_extract_fill:2" \
            "gather:k_gather_x:2" "cross_entropy:k_ce_row:1"; do
  name=${spec%%:*}; rest=${spec#*:}; kre=${rest%:*}; skip=${rest##*:}
  if [ -n "$ONLY" ] && ! echo " $ONLY " | grep -q " $name "; then continue; fi
  ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 \
      -o gpurun_out/prof_${R}_$name $CMD > gpurun_out/ncu_full_$name.log 2>&1
  echo "$name rc=$?" >> gpurun_out/ncu_rc.txt
done
