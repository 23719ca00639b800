cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 200 python -m pytest tests/test_gpu_kernels.py -q --timeout 60 > gpurun_out/k.log 2>&1; echo "rc=$?" >> gpurun_out/k.log
timeout 400 python -m pytest tests/test_gpu_sampler.py -q --timeout 150 > gpurun_out/s.log 2>&1; echo "rc=$?" >> gpurun_out/s.log
timeout 400 python -m pytest tests/test_gpu_train.py tests/test_gpu_eval.py tests/test_cpp_dropin.py -q --timeout 300 > gpurun_out/t.log 2>&1; echo "rc=$?" >> gpurun_out/t.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
for f in gpurun_out/*.log; do tail -n 3 $f; done
