# C2 on PMM grids with the per-rank timeline trace (GGB_PROF_TRACE) + NCCL probe.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/trace
rm -f gpurun_out/trace/*
for g in ${GRIDS:-1x2x2x1 2x1x2x1}; do
  W=$(echo $g | tr 'x' '\n' | awk 'BEGIN{p=1}{p*=$1}END{print p}')
  mkdir -p gpurun_out/trace/$g
  GGB_PROF_TRACE=gpurun_out/trace/$g timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr=127.0.0.1 --master-port=29551 \
    bench.py --gpus $W --grid $g --steps 10 --warmup 3 --no-cpu-baseline --no-eval $EXTRA > gpurun_out/trace/c2g_$g.json 2> gpurun_out/trace/c2g_$g.err
  echo "$g rc=$?"
done
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29552 scripts/nccl_probe.py > gpurun_out/trace/nccl2.json 2>&1
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29553 scripts/nccl_probe.py > gpurun_out/trace/nccl4.json 2>&1
nvidia-smi topo -m > gpurun_out/trace/topo.txt
