cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export NCCL_DEBUG=WARN GGB_WATCHDOG_S=100
for g in 2x1x1x1 1x1x1x2; do
  timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 \
    --redirects 3 --log-dir gpurun_out/tr_$g tests/mgpu_worker.py $g 0 > gpurun_out/mg_$g.log 2>&1
  echo "$g rc=$?" >> gpurun_out/mg_rc.txt
done
