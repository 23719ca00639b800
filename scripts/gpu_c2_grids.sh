# C2 epoch time on the SURVEY 8(e) grid shapes that fit 4 GPUs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/c2g_rc.txt
for g in ${C2_GRIDS:-1x1x1x2 2x1x1x1 1x2x1x1 4x1x1x1 1x2x2x1 2x1x1x2 2x1x2x1}; do
  W=$(echo $g | tr 'x' '\n' | awk 'BEGIN{p=1}{p*=$1}END{print p}')
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$W --master-addr=127.0.0.1 --master-port=29551 \
    bench.py --gpus $W --grid $g --steps 10 --warmup 3 --no-cpu-baseline --no-eval $EXTRA > gpurun_out/c2g_$g.json 2> gpurun_out/c2g_$g.err
  echo "$g rc=$?" >> gpurun_out/c2g_rc.txt
  python -c "
import json; d=json.loads(open('gpurun_out/c2g_$g.json').read().splitlines()[-1]); k=d['kernels']
print('$g', round(d['value'],5), round(d['ms_per_step'],3), 'coll', round(k.get('collectives',{}).get('ms_per_step',0),3), 'e2e', round(d['e2e']['value'],5))" >> gpurun_out/c2g_rc.txt 2>&1
done
cat gpurun_out/c2g_rc.txt
