# launch list only (ncu gpu__time_duration per launch) of the default bench step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
R=${ROUND:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-eval"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?" > gpurun_out/ncu_rc.txt
