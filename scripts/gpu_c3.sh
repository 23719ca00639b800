# C3 (Reddit-shaped) at 1 GPU and on 4 GPUs: data parallel vs 3D-PMM grids.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/c3_rc.txt
[ -z "$SKIP1" ] && timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-eval > gpurun_out/c3_n1.json 2> gpurun_out/c3_n1.err
echo "n1 rc=$?" >> gpurun_out/c3_rc.txt
for g in $GRIDS; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29541 \
    bench.py --config C3 --gpus 4 --grid $g --steps 10 --warmup 3 --no-cpu-baseline --no-eval $EXTRA > gpurun_out/c3_$g$TAG.json 2> gpurun_out/c3_$g$TAG.err
  echo "$g rc=$?" >> gpurun_out/c3_rc.txt
done
cat gpurun_out/c3_rc.txt
for f in gpurun_out/c3_*.json; do python scripts/show_bench.py $f 2>/dev/null | head -1; done
