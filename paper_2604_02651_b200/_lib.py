"""ctypes binding of libggb.so (include/ggb.h).

The CUDA library is the only compute path: importing this module loads the
in-tree ``libggb.so`` and raises if it is missing. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.path.join(HERE, "libggb.so")

I32, I64, U64, F64, P = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p

GGB_OK, GGB_EINVAL, GGB_ECONTRACT, GGB_ETIMEOUT, GGB_ECUDA, GGB_ENCCL = 0, 1, 2, 3, 4, 5
FP32, BF16_WIRE, BF16_SUM = 0, 1, 2
SGD, ADAM = 0, 1
COMPUTE_ACCURATE, COMPUTE_FAST = 0, 1


class ModelConfigC(C.Structure):
    """ggb_model_config == ModelConfig (model.hpp:26-43)."""

    _fields_ = [("layers", I32), ("d_in", I64), ("d_h", I64), ("d_out", I64),
                ("dropout_rate", F64), ("use_rmsnorm", I32), ("use_dropout", I32),
                ("use_residual", I32)]


class BlockC(C.Structure):
    """ggb_block == one rank's block of a ShardedTensor (tensor.hpp:75-86)."""

    _fields_ = [("row_axis", I32), ("col_axis", I32), ("g_rows", I64), ("g_cols", I64), ("row_off", P),
                ("col_off", P), ("data", P), ("ld", I64)]


class CsrBlockC(C.Structure):
    """ggb_csr_block == one rank's block of a ShardedSparse (tensor.hpp:88-96)."""

    _fields_ = [("row_axis", I32), ("col_axis", I32), ("g_rows", I64), ("g_cols", I64), ("row_off", P),
                ("col_off", P), ("row_ptr", P), ("col", P), ("val", P)]


# (name, restype, argtypes)
_SIGS = [
    ("ggb_last_error", C.c_char_p, []),
    ("ggb_version", C.c_int, []),
    ("ggb_get_unique_id", C.c_int, [P]),
    ("ggb_device_count", C.c_int, [P]),
    ("ggb_ctx_create", C.c_int, [P, I32, I32, P, P, P]),
    ("ggb_ctx_destroy", C.c_int, [P]),
    ("ggb_ctx_set_stream", C.c_int, [P, P]),
    ("ggb_ctx_synchronize", C.c_int, [P]),
    ("ggb_ctx_set_comm_timeout", C.c_int, [P, I64]),
    ("ggb_ctx_counters", C.c_int, [P, P]),
    ("ggb_ctx_comm_stats", C.c_int, [P, I32, I32, P]),
    ("ggb_ctx_profile", C.c_int, [P, I32]),
    ("ggb_ctx_profile_read", C.c_int, [P, P, P, P, P, I32]),
    ("ggb_sample_vertices", C.c_int, [P, I64, I64, U64, U64, P]),
    ("ggb_graph_create", C.c_int, [P, I64, P, P, P, I32, I64, P, I64, P, I32, P]),
    ("ggb_graph_generate_synthetic", C.c_int, [P, I64, F64, I64, I64, U64, I32, P]),
    ("ggb_graph_generate_synthetic_device", C.c_int, [P, I64, F64, I64, I64, U64, I32, P]),
    ("ggb_graph_export", C.c_int, [P, P, P, P, P, P, P]),
    ("ggb_dataset_load", C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, P]),
    ("ggb_dataset_generate_synthetic", C.c_int, [I64, F64, I64, I64, U64, P]),
    ("ggb_rmat_edges", C.c_int, [P, I32, I64, F64, F64, F64, U64, P]),
    ("ggb_dataset_generate_rmat", C.c_int, [P, I32, I64, F64, F64, F64, I64, I64, U64, P]),
    ("ggb_dataset_info", C.c_int, [P, P]),
    ("ggb_dataset_export", C.c_int, [P, P, P, P, P, P, P, P]),
    ("ggb_dataset_save", C.c_int, [P, C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p]),
    ("ggb_graph_from_dataset", C.c_int, [P, P, I32, P]),
    ("ggb_dataset_destroy", C.c_int, [P]),
    ("ggb_graph_set_split", C.c_int, [P, P]),
    ("ggb_graph_destroy", C.c_int, [P]),
    ("ggb_graph_info", C.c_int, [P, P]),
    ("ggb_graph_features_to_host", C.c_int, [P]),
    ("ggb_build_step_batch", C.c_int, [P, P, I64, U64, U64, P]),
    ("ggb_batch_destroy", C.c_int, [P]),
    ("ggb_prefetch_create", C.c_int, [P, P, I64, U64, U64, U64, I32, I64, F64, P]),
    ("ggb_prefetch_next", C.c_int, [P, P]),
    ("ggb_prefetch_destroy", C.c_int, [P]),
    ("ggb_batch_info", C.c_int, [P, P]),
    ("ggb_batch_sample", C.c_int, [P, P]),
    ("ggb_batch_offsets", C.c_int, [P, I32, P]),
    ("ggb_batch_plane", C.c_int, [P, I32, I32, P, P, P, P]),
    ("ggb_batch_x_in", C.c_int, [P, P]),
    ("ggb_batch_labels", C.c_int, [P, P]),
    ("ggb_state_create", C.c_int, [P, P, U64, P]),
    ("ggb_state_destroy", C.c_int, [P]),
    ("ggb_state_set_compute", C.c_int, [P, I32]),
    ("ggb_state_num_params", C.c_int, [P]),
    ("ggb_state_param_info", C.c_int, [P, I32, P]),
    ("ggb_state_param_get", C.c_int, [P, I32, I32, P]),
    ("ggb_state_param_set", C.c_int, [P, I32, I32, P]),
    ("ggb_train_step", C.c_int, [P, P, P, I32, U64, U64, F64, P]),
    ("ggb_last_loss_device", C.c_int, [P, P]),
    ("ggb_state_logits", C.c_int, [P, P, P]),
    ("ggb_forward", C.c_int, [P, P, P, I32, I32, U64, U64, F64]),
    ("ggb_evaluate_full_graph", C.c_int, [P, P, P, P, C.c_int32, C.c_double, P]),
    ("ggb_dp_sync", C.c_int, [P, P]),
    ("ggb_optimizer_step", C.c_int, [P, P, I32, F64]),
    ("ggb_gemm_bf16", C.c_int, [P, I64, I64, I64, P, I64, P, I64, P, I64, P, I64]),
    ("ggb_gemm_split_bf16", C.c_int, [P, I64, I64, I64, P, P, I64, P, P, I64, P, I64]),
    ("ggb_gemm_wgrad_bf16", C.c_int, [P, I64, I64, I64, P, I64, P, I64, P, I64]),
    ("ggb_spmm_csr", C.c_int, [P, I64, P, P, P, P, I64, I64, P, I64, P, I64, I32]),
    ("ggb_sample_vertices_test_reject", C.c_int, [P, I64, I64, U64, U64, U64, P]),
    ("ggb_spmm_csr_f32", C.c_int, [P, I64, P, P, P, P, I64, I64, P, I64, P, P, I64, I32]),
    ("ggb_contract", C.c_int, [P, P, P, P, I32]),
    ("ggb_spmm", C.c_int, [P, P, P, P, I32]),
    ("ggb_transposed", C.c_int, [P, P, P]),
    ("ggb_gather_full", C.c_int, [P, P, P, I64]),
    ("ggb_reshard", C.c_int, [P, P, P]),
    ("ggb_rmsnorm_fwd", C.c_int, [P, P, P, F64, P, P]),
    ("ggb_rmsnorm_bwd", C.c_int, [P, P, P, P, P, P, P]),
    ("ggb_fused_elementwise_fwd", C.c_int, [P, P, P, F64, U64, I32, P, P]),
    ("ggb_fused_elementwise_bwd", C.c_int, [P, P, P, C.c_float, P]),
    ("ggb_mask_words", I64, [I64]),
    ("ggb_cross_entropy", C.c_int, [P, P, P, P, P]),
    ("ggb_batch_csr_block", C.c_int, [P, I32, I32, P]),
    ("ggb_loss", C.c_int, [P, P, P, P]),
    ("ggb_loss_to_host_async", C.c_int, [P, P, P]),
    ("ggb_backward", C.c_int, [P, P, P, I32]),
    ("ggb_device_alloc", C.c_int, [P, C.c_size_t, P]),
    ("ggb_device_free", C.c_int, [P, P]),
    ("ggb_memcpy_h2d", C.c_int, [P, P, P, C.c_size_t]),
    ("ggb_memcpy_d2h", C.c_int, [P, P, P, C.c_size_t]),
]

EXPORTED = [name for name, _, _ in _SIGS]


def build() -> None:
    """Compile libggb.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIBPATH):
            raise RuntimeError(f"{LIBPATH} is missing: build it with paper_2604_02651_b200._lib.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIBPATH)
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class GgbError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(GgbError, ValueError):
    """std::invalid_argument in the reference."""


class CommContract(GgbError):
    """gridgnn::CommContract (comm.hpp:44-46)."""


class CommTimeout(GgbError):
    """gridgnn::CommTimeout (comm.hpp:41-43)."""


def check(rc: int) -> None:
    if rc == GGB_OK:
        return
    msg = lib().ggb_last_error().decode(errors="replace")
    if rc == GGB_EINVAL:
        raise InvalidArgument(rc, msg)
    if rc == GGB_ECONTRACT:
        raise CommContract(rc, msg)
    if rc == GGB_ETIMEOUT:
        raise CommTimeout(rc, msg)
    raise GgbError(rc, msg)
