#!/bin/bash
# A/B of run-time switches on one box: each line "name|ENV=... ENV2=...|extra bench args"
# prints ms_per_step, e2e ms_per_step, dominant kernel class per variant.
mkdir -p gpurun_out/ab
while IFS='|' read -r name envs extra; do
  [ -z "$name" ] && continue
  env $envs python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-eval $extra \
      > gpurun_out/ab/$name.json 2> gpurun_out/ab/$name.err
  python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab/{n}.json").read().strip().splitlines()[-1])
    k = d["kernels"]
    print(f"{n:24s} step {d['ms_per_step']:.3f} ms  e2e {d['e2e']['ms_per_step']:.3f} ms  clk {d['clocks']['sm_mhz']} "
          + " ".join(f"{c}={v['ms_per_step']:.2f}" for c, v in sorted(k.items(), key=lambda kv: -kv[1]['ms_per_step'])))
except Exception as e:
    print(n, "FAILED", e, open(f"gpurun_out/ab/{n}.err").read()[-500:])
PY
done
