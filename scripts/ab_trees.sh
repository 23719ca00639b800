#!/bin/bash
# A/B of two source trees on one box: the current tree and old_tree/ (a git worktree)
mkdir -p gpurun_out/ab
for i in 1 2; do
  for t in . old_tree; do
    (cd $t && python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-eval $EXTRA) > gpurun_out/ab/tree_${t//\//_}_$i.json 2>/dev/null
    python - "$t" "$i" <<'PY'
import json, sys
t, i = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/ab/tree_{t.replace('/', '_')}_{i}.json").read().strip().splitlines()[-1])
k = d["kernels"]
print(f"{t:10s} {i} step {d['ms_per_step']:.3f} e2e {d['e2e']['ms_per_step']:.3f} " + " ".join(f"{c}={v['ms_per_step']:.2f}" for c, v in sorted(k.items(), key=lambda kv: -kv[1]['ms_per_step'])[:6]))
PY
  done
done
