# Peer-memory all-reduce + reshard: multi-GPU parity + C2 PMM-grid A/B against NCCL.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/peer
rm -rf gpurun_out/peer/*
export GGB_COMM_TIMEOUT_MS=20000
timeout 1200 python -m pytest tests/test_multigpu.py -x -q --timeout 600 > gpurun_out/peer/mgpu_tests.log 2>&1
echo "mgpu tests rc=$?" > gpurun_out/peer/rc.txt
tail -3 gpurun_out/peer/mgpu_tests.log >> gpurun_out/peer/rc.txt
timeout 300 python -m pytest tests/test_gpu_train.py -x -q -k "async_loss" > gpurun_out/peer/async.log 2>&1
echo "async test rc=$?" >> gpurun_out/peer/rc.txt
for v in ${PEER_AB:-"1x2x2x1|fp32|GGB_PEER=0" "1x2x2x1|fp32|GGB_PEER=1" "1x2x2x1|bf16comm|GGB_PEER=1" "1x1x1x2|bf16comm|GGB_PEER=1" "1x2x1x1|bf16comm|GGB_PEER=1" "1x1x2x2|bf16comm|GGB_PEER=1"}; do
  IFS='|' read -r g prec envs <<< "$v"
  W=$(echo $g | tr 'x' '\n' | awk 'BEGIN{p=1}{p*=$1}END{print p}')
  name=${g}_${prec}_${envs#GGB_PEER=}
  mkdir -p gpurun_out/peer/$name
  env $envs GGB_PROF_TRACE=gpurun_out/peer/$name timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr=127.0.0.1 --master-port=29551 \
    bench.py --gpus $W --grid $g --precision $prec --steps 10 --warmup 3 --no-cpu-baseline --no-eval > gpurun_out/peer/$name.json 2> gpurun_out/peer/$name.err
  echo "$name rc=$? $(python scripts/show_bench.py gpurun_out/peer/$name.json 2>&1 | head -1)" >> gpurun_out/peer/rc.txt
done
cat gpurun_out/peer/rc.txt
