cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
  --master-port=29536 scripts/nccl_probe.py > gpurun_out/nccl_probe.log 2>&1
echo "probe rc=$?" > gpurun_out/nccl_rc.txt
