"""Probe (not product code): time the host vs device synthetic dataset build at C2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_02651_b200 import gridgnn as gg
ctx = gg.Context()
for name, fn in [("device", gg.Graph.generate_synthetic_device), ("host", gg.Graph.generate_synthetic)]:
    t0 = time.time()
    g = fn(ctx, 2450000, 50.53, 100, 47, 7, 3)
    ctx.synchronize()
    print(name, "%.2f s" % (time.time() - t0), "nnz", g.nnz, flush=True)
    if name == "device":
        t0 = time.time()
        g2 = fn(ctx, 2450000, 50.53, 100, 47, 7, 3)
        ctx.synchronize()
        print(name, "(warm) %.2f s" % (time.time() - t0), flush=True)
        del g2
    del g
