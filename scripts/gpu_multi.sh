cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export GGB_WATCHDOG_S=120
N=$(nvidia-smi -L | wc -l)
rm -f gpurun_out/mg_rc.txt
for gp in ${MG_GRIDS:-2x1x1x1:0 1x1x1x2:0 1x2x1x1:0 1x1x2x1:1 1x2x2x1:0 1x1x2x2:1 2x1x1x2:0 4x1x1x1:0 1x2x1x1:2 1x2x2x1:2 1x2x2x2:0 2x2x2x1:0}; do
  g=${gp%%:*}; p=${gp##*:}
  W=$(echo $g | tr 'x' '\n' | awk 'BEGIN{p=1}{p*=$1}END{print p}')
  if [ $W -gt $N ]; then continue; fi
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr=127.0.0.1 --master-port=29533 \
    tests/mgpu_worker.py $g $p > gpurun_out/mg_$g.log 2>&1
  echo "$g prec=$p rc=$? $(grep '^{' gpurun_out/mg_$g.log | tail -1)" >> gpurun_out/mg_rc.txt
done
# the driver's scaling run: bench.py under torchrun on all GPUs of the box (default DP grid)
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29534 \
  bench.py --gpus $N --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
echo "bench n=$N rc=$?" >> gpurun_out/mg_rc.txt
