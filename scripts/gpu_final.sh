# Final HEAD validation on one 4-GPU box: every GPU test (multi-GPU included),
# smoke, the driver's bench commands (1 GPU, reference arm, DP 2 and 4).
cd $GRAFT_REPO_ROOT
O=gpurun_out/final
mkdir -p $O
rm -f $O/rc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
export GGB_COMM_TIMEOUT_MS=30000
timeout 1800 python -m pytest tests -m gpu -v --timeout 600 > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/rc.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench n1 rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?" >> $O/rc.txt
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2956$N \
    bench.py --gpus $N --steps 20 --warmup 5 > $O/bench_n$N.json 2> $O/bench_n$N.err; echo "bench n$N rc=$?" >> $O/rc.txt
done
cat $O/rc.txt; grep -E "passed|failed" $O/gpu_tests.log | tail -2
