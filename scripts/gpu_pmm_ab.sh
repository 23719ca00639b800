# 4 GPUs: multi-GPU parity, then C2 PMM grids with the gradient all-reduces inline vs async
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests/test_multigpu.py -q -m gpu 2>&1 | tail -3
for v in 1 0; do
  echo "== GGB_ASYNC_GRAD=$v"
  GGB_ASYNC_GRAD=$v C2_GRIDS="1x2x2x1 1x1x1x2 2x1x2x1" bash scripts/gpu_c2_grids.sh 2>&1 | grep -v rc=
done
