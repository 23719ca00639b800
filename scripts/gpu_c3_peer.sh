# C3 (Reddit-shaped) on 1 and 4 B200 with the peer-memory collectives (and NCCL for comparison).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/c3p
rm -rf gpurun_out/c3p/*
export GGB_COMM_TIMEOUT_MS=20000
for v in ${C3_AB:-"1x1x1x1|fp32|X=1" "1x2x2x1|fp32|GGB_PEER=0" "1x2x2x1|fp32|GGB_PEER=1" "1x2x2x1|bf16comm|GGB_PEER=1" "1x1x2x2|fp32|GGB_PEER=1" "1x1x2x2|bf16comm|GGB_PEER=1" "2x1x2x1|bf16comm|GGB_PEER=1" "4x1x1x1|fp32|X=1"}; do
  IFS='|' read -r g prec envs <<< "$v"
  W=$(echo $g | tr 'x' '\n' | awk 'BEGIN{p=1}{p*=$1}END{print p}')
  name=${g}_${prec}_$(echo $envs | tr ' =' '_-')
  env $envs timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr=127.0.0.1 --master-port=29551 \
    bench.py --config C3 --gpus $W --grid $g --precision $prec --steps 10 --warmup 3 --no-cpu-baseline --no-eval > gpurun_out/c3p/$name.json 2> gpurun_out/c3p/$name.err
  echo "$name rc=$? $(python scripts/show_bench.py gpurun_out/c3p/$name.json 2>&1 | head -1)" >> gpurun_out/c3p/rc.txt
done
cat gpurun_out/c3p/rc.txt
