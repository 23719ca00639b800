#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over small instances of
# every hot kernel: the smoke step (sampler, SpMM pipes, tcgen05 GEMMs, row
# kernels, cross-entropy, Adam) and the kernel tests' small shapes.
mkdir -p gpurun_out/sanitize
SEL='test_gemm_bf16 and 129 or test_gemm_wgrad and 3000 or test_spmm_f32_rows and 777 or test_spmm_skewed_rows and 128-1 or test_gemm_split and 77'
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --target-processes all \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize/smoke_$tool.log 2>&1
  echo "smoke $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/smoke_$tool.log | tail -1)"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --target-processes all \
    python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "$SEL" > gpurun_out/sanitize/kernels_$tool.log 2>&1
  echo "kernels $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize/kernels_$tool.log | tail -1) $(tail -1 gpurun_out/sanitize/kernels_$tool.log)"
done
