"""Probe (not product code): time the tcgen05 GEMMs alone at the C2 shapes
through the C ABI (ggb_gemm_bf16 / ggb_gemm_split_bf16), CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_02651_b200 import gridgnn as gg

_s = torch.cuda.Stream()
torch.cuda.set_stream(_s)
ctx = gg.Context(stream=_s.cuda_stream)
L = gg.lib()
M = 612500
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(_s)
    for _ in range(reps): fn()
    b.record(_s); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
for (n, k, split, out) in [(256, 256, 0, "bf16"), (256, 256, 0, "f32"), (256, 256, 1, "f32"), (256, 104, 1, "f32"),
                           (256, 48, 0, "f32"), (48, 256, 1, "f32")]:
    A = torch.randn(M, k, device="cuda").to(torch.bfloat16)
    Al = torch.randn(M, k, device="cuda").to(torch.bfloat16)
    B = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    Bl = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, n, device="cuda")
    Cb = torch.empty(M, n, device="cuda", dtype=torch.bfloat16)
    if split:
        f = lambda: gg.check(L.ggb_gemm_split_bf16(ctx.h, M, n, k, A.data_ptr(), Al.data_ptr(), k, B.data_ptr(),
                                                   Bl.data_ptr(), k, C.data_ptr(), n))
    elif out == "bf16":
        f = lambda: gg.check(L.ggb_gemm_bf16(ctx.h, M, n, k, A.data_ptr(), k, B.data_ptr(), k, None, 0,
                                             Cb.data_ptr(), n))
    else:
        f = lambda: gg.check(L.ggb_gemm_bf16(ctx.h, M, n, k, A.data_ptr(), k, B.data_ptr(), k, C.data_ptr(), n,
                                             None, 0))
    us = t(f)
    byts = M * k * 2 * (1 + split) + M * n * (2 if out == "bf16" else 4)
    print(f"n={n} k={k} split={split} out={out}: {us:7.1f} us  {byts / us / 1e3:6.0f} GB/s", flush=True)
