# bench.py under torchrun on N GPUs (default DP grid), prefetch variants, and a PMM grid
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
rm -f gpurun_out/sc_rc.txt
run() {  # name, extra args
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=29535 \
    bench.py --gpus $N --steps 20 --warmup 3 --no-cpu-baseline --no-eval $2 > gpurun_out/sc_$1.json 2> gpurun_out/sc_$1.err
  echo "$1 rc=$?" >> gpurun_out/sc_rc.txt
}
run n${N}_pf1 ""
GGB_PREFETCH_PRIORITY=low run n${N}_pf1low ""
run n${N}_pf0 "--prefetch 0"
[ -n "$PMM" ] && run n${N}_pmm "--grid $PMM"
[ -n "$PMM" ] && run n${N}_pmm_w10 "--grid $PMM --warmup 10"
