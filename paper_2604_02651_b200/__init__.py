"""B200-native (sm_100a) mini-batch GCN training step of ScaleGNN (arxiv 2604.02651).

The compute path is libggb.so (CUDA kernels + NCCL behind the C ABI in
include/ggb.h); ``gridgnn`` mirrors the reference's hot-path API on top of it.
"""
from . import gridgnn  # noqa: F401
from ._lib import LIBPATH, build, lib  # noqa: F401
