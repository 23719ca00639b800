# PMM collectives overlap: parity on every multi-GPU grid, then C3 timings for
# chunk counts / NCCL CTA budgets (4 GPUs).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_multi.sh > /dev/null 2>&1
cat gpurun_out/mg_rc.txt | cut -c1-60
for v in "GGB_COMM_CHUNKS=1" "GGB_COMM_CHUNKS=4" "GGB_COMM_CHUNKS=8" "GGB_COMM_CHUNKS=4 GGB_COMM_CTAS=32"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29541 \
    bench.py --config C3 --gpus 4 --grid 1x2x2x1 --steps 10 --warmup 3 --no-cpu-baseline --no-eval > gpurun_out/ov_$tag.json 2> gpurun_out/ov_$tag.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ov_$tag.json').read().splitlines()[-1]); k=d['kernels']
print('$v', round(d['ms_per_step'],3), {n: round(v['ms_per_step'],3) for n,v in k.items() if n in ('collectives','spmm_fwd','spmm_bwd','gemm_fwd','gemm_dx')})"
done
