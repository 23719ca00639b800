"""Probe (not product code): time one C2 batch build with HBM-resident vs
host-resident features, alone on the device."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_02651_b200 import gridgnn as gg

ctx = gg.Context()
g = gg.Graph.generate_synthetic(ctx, 2450000, 50.53, 100, 47, 7, 3)
b = 612500
bt = None
def timed(label):
    global bt
    for t in range(2):
        bt = gg.build_step_batch(ctx, g, b, 1, t, reuse=bt)
    ctx.synchronize()
    t0 = time.perf_counter()
    for t in range(5):
        bt = gg.build_step_batch(ctx, g, b, 1, t, reuse=bt)
    ctx.synchronize()
    print(label, "%.3f ms/build" % ((time.perf_counter() - t0) / 5 * 1e3), flush=True)
timed("hbm features")
g.features_to_host()
timed("host features")
