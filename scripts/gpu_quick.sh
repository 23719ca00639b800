cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/rc.txt
timeout 400 python -m pytest tests/test_gpu_train.py -q --timeout 150 > gpurun_out/tq.log 2>&1; echo "t rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --prefetch 0 > gpurun_out/bench_c2_nopf.json 2> gpurun_out/bench_c2_nopf.err; echo "c2nopf rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 30 --warmup 5 --compute fast --no-cpu-baseline > gpurun_out/bench_c2_fast.json 2> gpurun_out/bench_c2_fast.err; echo "c2f rc=$?" >> gpurun_out/rc.txt
