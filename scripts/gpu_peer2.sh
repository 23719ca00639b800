# Chunked producer / peer-reduction overlap: parity with chunks, then A/B of the chunk count.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/peer2
rm -rf gpurun_out/peer2/*
export GGB_COMM_TIMEOUT_MS=20000
GGB_PEER_CHUNKS=4 timeout 1200 python -m pytest tests/test_multigpu.py -x -q --timeout 600 -k "not timeout" > gpurun_out/peer2/mgpu_tests.log 2>&1
echo "mgpu tests (4 chunks) rc=$?" > gpurun_out/peer2/rc.txt
tail -2 gpurun_out/peer2/mgpu_tests.log >> gpurun_out/peer2/rc.txt
for v in ${PEER_AB:-"1x2x2x1|bf16comm|GGB_PEER_CHUNKS=1" "1x2x2x1|bf16comm|GGB_PEER_CHUNKS=2" "1x2x2x1|bf16comm|GGB_PEER_CHUNKS=4" "1x2x2x1|bf16comm|GGB_PEER_CHUNKS=4 GGB_PEER_RESERVE=8" "1x2x2x1|bf16comm|GGB_PEER_CHUNKS=4 GGB_PEER_RESERVE=32" "1x2x2x1|fp32|GGB_PEER_CHUNKS=4"}; do
  IFS='|' read -r g prec envs <<< "$v"
  W=$(echo $g | tr 'x' '\n' | awk 'BEGIN{p=1}{p*=$1}END{print p}')
  name=${g}_${prec}_$(echo $envs | tr ' =' '_-')
  env $envs timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr=127.0.0.1 --master-port=29551 \
    bench.py --gpus $W --grid $g --precision $prec --steps 10 --warmup 3 --no-cpu-baseline --no-eval > gpurun_out/peer2/$name.json 2> gpurun_out/peer2/$name.err
  echo "$name rc=$? $(python scripts/show_bench.py gpurun_out/peer2/$name.json 2>&1 | head -1)" >> gpurun_out/peer2/rc.txt
done
cat gpurun_out/peer2/rc.txt
