# DP e2e vs the host-gather grid (4 and 2 GPUs).
cd $GRAFT_REPO_ROOT
O=gpurun_out/dpg; mkdir -p $O; rm -f $O/*
for N in 4 2; do for B in 16 32 64; do
  GGB_HOST_GATHER_BLOCKS=$B timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2957$N \
    bench.py --gpus $N --steps 20 --warmup 5 --no-cpu-baseline --no-eval > $O/n${N}_b$B.json 2> $O/n${N}_b$B.err
  python - $O/n${N}_b$B.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'step', round(d['ms_per_step'], 3), 'e2e', round(d['e2e']['ms_per_step'], 3), d['e2e_step_ms_rank0'][:6])
PY
done; done
