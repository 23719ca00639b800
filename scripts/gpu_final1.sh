# Final 1-GPU driver-like check + DP 2/4 bench lines (4-GPU box, GPU 0 for the 1-GPU parts).
cd $GRAFT_REPO_ROOT
O=gpurun_out/final1
mkdir -p $O; rm -f $O/rc.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -k "not multigpu and not sharded_grid" > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/rc.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench n1 rc=$?" >> $O/rc.txt
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2958$N \
    bench.py --gpus $N --steps 20 --warmup 5 > $O/bench_n$N.json 2> $O/bench_n$N.err; echo "bench n$N rc=$?" >> $O/rc.txt
done
nvidia-smi > $O/smi_after.txt 2>&1
cat $O/rc.txt; tail -1 $O/gpu_tests.log
