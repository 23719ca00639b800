"""Probe: the reference (oracle/_ref) on the full C2 batch on this host —
step time and peak RSS per grid (informs the reference arm of bench.py)."""
import os, resource, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O

R = O.Ref()
t0 = time.time()
h = R.dataset_synthetic(2_450_000, 50.53, 100, 47, 7)
print("dataset", time.time() - t0, "s; maxrss GB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, flush=True)
mcfg = O.ModelConfig(layers=3, d_in=100, d_h=256, d_out=47, dropout_rate=0.1)
for dims in [tuple(int(x) for x in g.split("x")) for g in sys.argv[1:]]:
    t0 = time.time()
    ms, phase = R.bench(h, dims, mcfg, 612_500, 1, 0, 1)
    print(dims, "step ms", list(ms), "phase", list(phase), "wall", time.time() - t0,
          "maxrss GB", resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, flush=True)
