# Multi-GPU check of HEAD: the multi-rank parity tests, then bench.py under
# torchrun (default DP grid) at N = 2 and N = all GPUs of the box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export GGB_WATCHDOG_S=120
N=$(nvidia-smi -L | wc -l)
rm -f gpurun_out/mgc_rc.txt
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x --timeout 400 > gpurun_out/mgc_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/mgc_rc.txt
for W in 2 $N; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr=127.0.0.1 --master-port=29536 \
    bench.py --gpus $W --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/mgc_bench_n$W.json 2> gpurun_out/mgc_bench_n$W.err
  echo "bench n=$W rc=$?" >> gpurun_out/mgc_rc.txt
done
cat gpurun_out/mgc_rc.txt; tail -2 gpurun_out/mgc_tests.log
