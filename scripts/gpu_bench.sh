cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 300 python bench.py --config C1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?" >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 20 --warmup 3 --compute fast --no-cpu-baseline > gpurun_out/bench_c2_fast.json 2> gpurun_out/bench_c2_fast.err; echo "c2f rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt
