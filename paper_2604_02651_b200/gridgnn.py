"""Python mirror of the reference's hot-path API (namespace gridgnn, /root/reference/proj)
over the C ABI of libggb.so. Names, argument meaning and error behaviour follow
the reference so parity tests read like the reference's own tests:

    sample_vertices            sampling.hpp:33
    block_partition            shardsample.hpp:14
    sample_partition           shardsample.hpp:118
    Dataset / RankContext      dataset.hpp:16-29, model.hpp:212-234  -> Graph
    build_step_batch           model.hpp:250-309                     -> StepBatch
    init_state                 model.hpp:175-208                     -> ModelState
    forward / train_step       model.hpp:335-478
    dp_sync / optimizer_step   model.hpp:423-456
    steps_per_epoch            model.hpp:539-542

Errors raise InvalidArgument (std::invalid_argument), CommContract and
CommTimeout like the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import (ADAM, BF16_SUM, BF16_WIRE, BlockC, CsrBlockC, COMPUTE_ACCURATE, COMPUTE_FAST, FP32, SGD, CommContract, CommTimeout, GgbError,  # noqa: F401
                   InvalidArgument, ModelConfigC, check, lib)

P = C.c_void_p
AXIS_D, AXIS_X, AXIS_Y, AXIS_Z = 0, 1, 2, 3


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(P)


# ---- host-side layout algebra (grid.hpp, shardsample.cpp:8-17, pmm.hpp:31-63) -------

# Graph500 R-MAT quadrant probabilities (d = 1 - a - b - c = 0.05)
RMAT_A, RMAT_B, RMAT_C = 0.57, 0.19, 0.19


def rmat_edges(ctx: "Context", scale: int, edges: int, seed: int, a: float = RMAT_A, b: float = RMAT_B,
               c: float = RMAT_C) -> np.ndarray:
    """The raw R-MAT edge list (edges x 2, int64) drawn on the GPU."""
    out = np.empty((edges, 2), np.int64)
    check(lib().ggb_rmat_edges(ctx.h, scale, edges, a, b, c, seed, _ptr(out)))
    return out


def block_partition(n: int, g: int) -> np.ndarray:
    if g < 1:
        raise InvalidArgument(1, "block_partition: g must be >= 1")
    base, extra = divmod(n, g)
    sizes = [base + (1 if k < extra else 0) for k in range(g)]
    return np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)


def sample_partition(s: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    return np.searchsorted(np.asarray(s), np.asarray(offsets), side="left").astype(np.int64)


def steps_per_epoch(n: int, b: int, gd: int) -> int:
    per = b * gd
    return (n + per - 1) // per


def adjacency_layout(layer: int) -> tuple[int, int]:
    return [(AXIS_Z, AXIS_X), (AXIS_Y, AXIS_Z), (AXIS_X, AXIS_Y)][(layer - 1) % 3]


def feature_layout(layer: int) -> tuple[int, int]:
    return [(AXIS_X, AXIS_Y), (AXIS_Z, AXIS_X), (AXIS_Y, AXIS_Z)][(layer - 1) % 3]


@dataclass(frozen=True)
class DeviceGrid:
    """4D grid (g_d, g_x, g_y, g_z), lexicographic rank numbering (grid.hpp:18-73)."""

    gd: int = 1
    gx: int = 1
    gy: int = 1
    gz: int = 1

    def __post_init__(self):
        if min(self.dims) < 1:
            raise InvalidArgument(1, "DeviceGrid: dims must be >= 1")

    @property
    def dims(self) -> tuple[int, int, int, int]:
        return (self.gd, self.gx, self.gy, self.gz)

    def total(self) -> int:
        return self.gd * self.gx * self.gy * self.gz

    def coord_of(self, rank: int) -> tuple[int, int, int, int]:
        z = rank % self.gz
        rank //= self.gz
        y = rank % self.gy
        rank //= self.gy
        x = rank % self.gx
        return (rank // self.gx, x, y, z)

    def rank_of(self, c) -> int:
        return ((c[0] * self.gx + c[1]) * self.gy + c[2]) * self.gz + c[3]

    def dp_group(self, rank: int) -> int:
        return self.coord_of(rank)[0]

    @staticmethod
    def parse(s: str) -> "DeviceGrid":
        """'GdxGxxGyxGz' as the reference CLI (gridgnn_main.cpp:57-66)."""
        parts = [int(x) for x in s.lower().split("x")]
        if len(parts) != 4:
            raise InvalidArgument(1, "grid must be GdxGxxGyxGz")
        return DeviceGrid(*parts)


# ---- context ---------------------------------------------------------------------------

def get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().ggb_get_unique_id(buf))
    return bytes(buf)


class Context:
    """One rank on one GPU: replaces Communicator + RankComm (comm.hpp:203-408).

    ``nccl_uid`` (from get_unique_id() on rank 0, broadcast by the caller)
    creates NCCL communicators for the grid axes. Without it the context is
    virtual: sampling and single-rank work run, multi-rank collectives raise
    CommContract.
    """

    def __init__(self, grid: DeviceGrid = DeviceGrid(), rank: int = 0, device: int = 0,
                 nccl_uid: bytes | None = None, stream: int | None = None):
        self.grid = grid
        self.rank = rank
        self.coord = grid.coord_of(rank)
        dims = (C.c_int32 * 4)(*grid.dims)
        uid = (C.c_uint8 * 128).from_buffer_copy(nccl_uid) if nccl_uid else None
        h = P()
        check(lib().ggb_ctx_create(dims, rank, device, uid, stream, C.byref(h)))
        self.h = h

    def set_stream(self, stream: int | None):
        check(lib().ggb_ctx_set_stream(self.h, stream))

    def set_comm_timeout(self, ms: int):
        """CommConfig::timeout (comm.hpp:195-198): collective watchdog deadline."""
        check(lib().ggb_ctx_set_comm_timeout(self.h, ms))

    def synchronize(self):
        check(lib().ggb_ctx_synchronize(self.h))

    def counters(self) -> dict:
        c = (C.c_uint64 * 3)()
        check(lib().ggb_ctx_counters(self.h, c))
        return {"launches": int(c[0]), "h2d_bytes": int(c[1]), "d2h_bytes": int(c[2])}

    AXES = ("D", "X", "Y", "Z")
    PHASES = ("sampling", "forward", "backward", "dp_sync", "other")

    def comm_stats(self, grid_total: bool = False, reset: bool = False) -> dict:
        """CommStats (comm.hpp:75-117): the reference's byte accounting of the
        logical collectives, {"bytes": {axis: {phase: n}}, "allreduce_calls":
        {axis: n}, "allgather_calls": {axis: n}}. grid_total sums over every
        rank (Communicator::snapshot; every rank must call it)."""
        c = (C.c_uint64 * 28)()
        check(lib().ggb_ctx_comm_stats(self.h, int(grid_total), int(reset), c))
        return {
            "bytes": {a: {p: int(c[i * 5 + j]) for j, p in enumerate(self.PHASES)} for i, a in enumerate(self.AXES)},
            "allreduce_calls": {a: int(c[20 + i]) for i, a in enumerate(self.AXES)},
            "allgather_calls": {a: int(c[24 + i]) for i, a in enumerate(self.AXES)},
        }

    def launches(self) -> int:
        return self.counters()["launches"]

    PROF_CLASSES = ["sampling", "spmm_fwd", "spmm_bwd", "gemm_fwd", "gemm_dx", "gemm_wgrad", "elementwise",
                    "optimizer", "collectives", "fwd_row", "bwd_row", "cross_entropy"]

    def profile(self, enable: bool):
        """Per-kernel-class CUDA-event timing on the context's stream."""
        check(lib().ggb_ctx_profile(self.h, int(enable)))

    def profile_read(self, reset: bool = True) -> dict:
        k = len(self.PROF_CLASSES)
        ms, by, fl = (np.zeros(k) for _ in range(3))
        cnt = np.zeros(k, np.int64)
        check(lib().ggb_ctx_profile_read(self.h, _ptr(ms), _ptr(by), _ptr(fl), _ptr(cnt), int(reset)))
        return {name: {"ms": float(ms[i]), "bytes": float(by[i]), "flops": float(fl[i]), "launches": int(cnt[i])}
                for i, name in enumerate(self.PROF_CLASSES)}

    def close(self):
        if getattr(self, "h", None):
            lib().ggb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx


@dataclass
class SampleSet:
    vertices: np.ndarray
    batch_size: int
    graph_size: int
    seed: int
    step: int


def sample_vertices(n: int, b: int, seed: int, step: int, ctx: Context | None = None) -> SampleSet:
    """sampling.hpp:33, sampled on the GPU (bit-exact with the reference)."""
    ctx = ctx or default_context()
    if b <= 0 or b > n:
        raise InvalidArgument(1, "sample_vertices: need 1 <= b <= n")
    out = np.empty(b, np.int64)
    check(lib().ggb_sample_vertices(ctx.h, n, b, seed, step, _ptr(out)))
    return SampleSet(out, b, n, seed, step)


# ---- graph (Dataset + RankContext resident in HBM) ----------------------------------------

class Graph:
    def __init__(self, ctx: Context, h):
        self.ctx = ctx
        self.h = h
        self._info()

    def _info(self):
        info = np.zeros(7, np.int64)
        check(lib().ggb_graph_info(self.h, _ptr(info)))
        (self.n, self.nnz, self.d_in, self.n_classes, self.distinct_shards, self.device_bytes,
         host) = (int(x) for x in info)
        self.features_on_host = bool(host)

    def features_to_host(self) -> None:
        """Move the feature slice to mapped pinned host memory (the reference's
        host-resident Dataset); batch builds then gather x_in rows over PCIe."""
        check(lib().ggb_graph_features_to_host(self.h))
        self._info()

    @staticmethod
    def from_csr(ctx: Context, n: int, row_ptr, col_idx, values, features, labels, n_classes: int,
                 layers: int, symmetric: bool = True, split=None) -> "Graph":
        rp = np.ascontiguousarray(row_ptr, np.int64)
        ci = np.ascontiguousarray(col_idx, np.int64)
        va = np.ascontiguousarray(values, np.float64)
        fe = np.ascontiguousarray(features, np.float32)
        la = np.ascontiguousarray(labels, np.int32)
        h = P()
        check(lib().ggb_graph_create(ctx.h, n, _ptr(rp), _ptr(ci), _ptr(va), int(symmetric),
                                     fe.shape[1] if fe.ndim == 2 else 1, _ptr(fe), n_classes, _ptr(la),
                                     layers, C.byref(h)))
        g = Graph(ctx, h)
        if split is not None:
            g.set_split(split)
        return g

    def set_split(self, split) -> None:
        """Split tags per vertex (Dataset::split: 0 train, 1 val, 2 test, 3 unused)."""
        sp = np.ascontiguousarray(split, np.uint8)
        if sp.shape != (self.n,):
            raise InvalidArgument(1, f"split: expected {self.n} tags, got shape {sp.shape}")
        check(lib().ggb_graph_set_split(self.h, _ptr(sp)))

    @staticmethod
    def generate_synthetic(ctx: Context, n: int, avg_degree: float, d_in: int, n_classes: int,
                           seed: int, layers: int) -> "Graph":
        """generate_synthetic (dataset.cpp:85-131), built natively then uploaded."""
        h = P()
        check(lib().ggb_graph_generate_synthetic(ctx.h, n, avg_degree, d_in, n_classes, seed, layers,
                                                 C.byref(h)))
        return Graph(ctx, h)

    @staticmethod
    def generate_synthetic_device(ctx: Context, n: int, avg_degree: float, d_in: int, n_classes: int,
                                  seed: int, layers: int) -> "Graph":
        """generate_synthetic built on the GPU (edges, CSR, labels, split bit-identical)."""
        h = P()
        check(lib().ggb_graph_generate_synthetic_device(ctx.h, n, avg_degree, d_in, n_classes, seed, layers,
                                                        C.byref(h)))
        return Graph(ctx, h)

    def export(self, csr: bool = True, features: bool = True):
        """Host copies: (row_ptr, col_idx, values) | None, features | None, labels, split."""
        rp = ci = va = fe = None
        if csr:
            rp = np.empty(self.n + 1, np.int64)
            ci = np.empty(self.nnz, np.int64)
            va = np.empty(self.nnz, np.float64)
        if features:
            fe = np.empty((self.n, self.d_in), np.float32)
        la = np.empty(self.n, np.int32)
        sp = np.empty(self.n, np.uint8)
        check(lib().ggb_graph_export(self.h, _ptr(rp), _ptr(ci), _ptr(va), _ptr(fe), _ptr(la), _ptr(sp)))
        return ((rp, ci, va) if csr else None), fe, la, sp

    def close(self):
        if getattr(self, "h", None):
            lib().ggb_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Dataset:
    """Host Dataset (dataset.hpp:16-29) with its raw edge list: the reference's
    file formats (load_dataset / save_*, dataset.cpp:152-280) and generator.
    No GPU needed except for to_graph."""

    def __init__(self, h):
        self.h = h
        info = np.zeros(5, np.int64)
        check(lib().ggb_dataset_info(h, _ptr(info)))
        self.n, self.nnz, self.d_in, self.n_classes, self.n_edges = (int(x) for x in info)

    @staticmethod
    def load(edges, features, labels, split) -> "Dataset":
        h = P()
        check(lib().ggb_dataset_load(*(str(x).encode() for x in (edges, features, labels, split)), C.byref(h)))
        return Dataset(h)

    @staticmethod
    def generate_synthetic(n: int, avg_degree: float, d_in: int, n_classes: int, seed: int) -> "Dataset":
        h = P()
        check(lib().ggb_dataset_generate_synthetic(n, avg_degree, d_in, n_classes, seed, C.byref(h)))
        return Dataset(h)

    @staticmethod
    def generate_rmat(ctx: "Context", scale: int, edges: int, d_in: int, n_classes: int, seed: int,
                      a: float = RMAT_A, b: float = RMAT_B, c: float = RMAT_C) -> "Dataset":
        """R-MAT graph (Graph500 parameters by default; edges drawn on the GPU)
        with generate_synthetic's features, labels and split."""
        h = P()
        check(lib().ggb_dataset_generate_rmat(ctx.h, scale, edges, a, b, c, d_in, n_classes, seed, C.byref(h)))
        return Dataset(h)

    def save(self, edges=None, features=None, labels=None, split=None) -> None:
        enc = lambda x: None if x is None else str(x).encode()
        check(lib().ggb_dataset_save(self.h, enc(edges), enc(features), enc(labels), enc(split)))

    def arrays(self):
        """((row_ptr, col_idx, values), features, labels, split, edges_uv)"""
        rp, ci, va = np.empty(self.n + 1, np.int64), np.empty(self.nnz, np.int64), np.empty(self.nnz, np.float64)
        fe, la, sp = np.empty((self.n, self.d_in), np.float32), np.empty(self.n, np.int32), np.empty(self.n, np.uint8)
        uv = np.empty((self.n_edges, 2), np.int64)
        check(lib().ggb_dataset_export(self.h, _ptr(rp), _ptr(ci), _ptr(va), _ptr(fe), _ptr(la), _ptr(sp), _ptr(uv)))
        return (rp, ci, va), fe, la, sp, uv

    def to_graph(self, ctx: "Context", layers: int) -> "Graph":
        h = P()
        check(lib().ggb_graph_from_dataset(ctx.h, self.h, layers, C.byref(h)))
        return Graph(ctx, h)

    def close(self):
        if getattr(self, "h", None):
            lib().ggb_dataset_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    r0: int = 0
    r1: int = 0
    c0: int = 0
    c1: int = 0

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0


class StepBatch:
    """StepBatch (model.hpp:238-246) resident in HBM; exports are host copies."""

    def __init__(self, graph: Graph, h):
        self.graph = graph
        self.h = h

    def info(self):
        v = np.zeros(9, np.int64)
        check(lib().ggb_batch_info(self.h, _ptr(v)))
        return v

    @property
    def b(self) -> int:
        return int(self.info()[0])

    @property
    def planes(self) -> int:
        return int(self.info()[2])

    @property
    def nnz_extracted(self) -> int:
        return int(self.info()[7])

    @property
    def nnz_kept(self) -> int:
        return int(self.info()[8])

    @property
    def sample(self) -> np.ndarray:
        out = np.empty(self.b, np.int64)
        check(lib().ggb_batch_sample(self.h, _ptr(out)))
        return out

    def batch_off(self, axis: int) -> np.ndarray:
        out = np.empty(self.graph.ctx.grid.dims[axis] + 1, np.int64)
        check(lib().ggb_batch_offsets(self.h, axis, _ptr(out)))
        return out

    def _plane(self, p: int, t: int) -> Csr:
        dims = np.zeros(7, np.int64)
        check(lib().ggb_batch_plane(self.h, p, t, _ptr(dims), None, None, None))
        rp = np.empty(dims[0] + 1, np.int64)
        col = np.empty(dims[2], np.int64)
        val = np.empty(dims[2], np.float64)
        check(lib().ggb_batch_plane(self.h, p, t, _ptr(dims), _ptr(rp), _ptr(col), _ptr(val)))
        return Csr(int(dims[0]), int(dims[1]), rp, col, val, *(int(x) for x in dims[3:7]))

    def a(self, p: int) -> Csr:
        return self._plane(p, 0)

    def a_t(self, p: int) -> Csr:
        return self._plane(p, 1)

    @property
    def x_in(self) -> tuple[tuple[int, int, int, int], np.ndarray]:
        i = self.info()
        r0, r1, c0, c1 = (int(x) for x in i[3:7])
        out = np.empty((r1 - r0, c1 - c0), np.float32)
        check(lib().ggb_batch_x_in(self.h, _ptr(out)))
        return (r0, r1, c0, c1), out

    @property
    def labels(self) -> np.ndarray:
        out = np.empty(self.b, np.int32)
        check(lib().ggb_batch_labels(self.h, _ptr(out)))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib().ggb_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StaleBatch(GgbError):
    """A prefetched batch used after the next Prefetcher.next() or close():
    its slot may already hold a later batch."""

    def __init__(self, msg: str):
        super().__init__(1, msg)  # GGB_EINVAL


class _BorrowedBatch(StepBatch):
    """A batch owned by a Prefetcher slot (never destroyed from Python). Valid
    until the prefetcher's next next() or close(); the reference's
    PrefetchQueue hands batches out by value, so a later use raises
    StaleBatch instead of reading a slot the producer refills."""

    def __init__(self, pf: "Prefetcher", h):
        self._pf, self._gen = pf, pf._gen
        super().__init__(pf.graph, h)

    @property
    def h(self):
        if self._h is not None and (self._pf.h is None or self._pf._gen != self._gen):
            raise StaleBatch("prefetched batch used after the next Prefetcher.next() or close()")
        return self._h

    @h.setter
    def h(self, v):
        self._h = v

    def close(self):
        self._h = None


class Prefetcher:
    """Sampling/training overlap (the train_run producer thread + PrefetchQueue,
    model.hpp:556-581): a native producer thread samples step t+1 on its own
    stream while step t trains; next() returns the batch of the following step."""

    def __init__(self, ctx: Context, graph: Graph, b: int, group_seed: int, first_step: int = 0,
                 run_seed: int = 0, cfg: "ModelConfig | None" = None):
        """With cfg (and its dropout on), the producer also evaluates the
        dropout keep-bits of every layer for the step ahead (keyed by run_seed)."""
        self.ctx, self.graph = ctx, graph
        layers = cfg.layers if (cfg is not None and cfg.use_dropout) else 0
        rate = cfg.dropout_rate if cfg is not None else 0.0
        d_h = cfg.d_h if cfg is not None else 0
        h = P()
        check(lib().ggb_prefetch_create(ctx.h, graph.h, b, group_seed, first_step, run_seed, layers, d_h, rate,
                                        C.byref(h)))
        self.h = h
        self._gen = 0

    def next(self) -> StepBatch:
        bh = P()
        check(lib().ggb_prefetch_next(self.h, C.byref(bh)))
        self._gen += 1
        return _BorrowedBatch(self, bh)

    def close(self):
        if getattr(self, "h", None):
            lib().ggb_prefetch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_step_batch(ctx: Context, graph: Graph, b: int, group_seed: int, step: int,
                     reuse: StepBatch | None = None) -> StepBatch:
    """model.hpp:250-309: the rank-local batch; communication-free."""
    h = P(reuse.h.value if reuse is not None else None)
    check(lib().ggb_build_step_batch(ctx.h, graph.h, b, group_seed, step, C.byref(h)))
    if reuse is not None:
        return reuse
    return StepBatch(graph, h)


# ---- model ------------------------------------------------------------------------------

@dataclass
class ModelConfig:
    layers: int = 2
    d_in: int = 0
    d_h: int = 64
    d_out: int = 0
    dropout_rate: float = 0.1
    use_rmsnorm: bool = True
    use_dropout: bool = True
    use_residual: bool = True

    def c(self) -> ModelConfigC:
        return ModelConfigC(self.layers, self.d_in, self.d_h, self.d_out, self.dropout_rate,
                            int(self.use_rmsnorm), int(self.use_dropout), int(self.use_residual))

    def param_names(self) -> list[str]:
        out = ["win"]
        for l in range(1, self.layers + 1):
            out.append(f"w{l}")
            if self.use_rmsnorm:
                out.append(f"gamma{l}")
        out.append("wout")
        return out


@dataclass
class ParamBlock:
    name: str
    g_rows: int
    g_cols: int
    r0: int
    r1: int
    c0: int
    c1: int
    is_vec: bool = False


class ModelState:
    """ModelState (model.hpp:87-105) resident in HBM (fp32 master weights,
    gradients and Adam moments; bf16 operand copies for the tensor cores)."""

    def __init__(self, ctx: Context, cfg: ModelConfig, seed: int, compute: int = COMPUTE_ACCURATE):
        self.ctx = ctx
        self.cfg = cfg
        h = P()
        c = cfg.c()
        check(lib().ggb_state_create(ctx.h, C.byref(c), seed, C.byref(h)))
        self.h = h
        self.set_compute(compute)
        self.blocks: list[ParamBlock] = []
        for i, name in enumerate(cfg.param_names()):
            info = np.zeros(6, np.int64)
            check(lib().ggb_state_param_info(h, i, _ptr(info)))
            self.blocks.append(ParamBlock(name, *(int(x) for x in info), is_vec=name.startswith("gamma")))

    def set_compute(self, mode: int):
        """COMPUTE_ACCURATE (fp32 forward activations, split-bf16 GEMMs) or COMPUTE_FAST (bf16)."""
        check(lib().ggb_state_set_compute(self.h, mode))
        self.compute = mode

    def _get(self, i: int, which: int) -> np.ndarray:
        b = self.blocks[i]
        shape = (b.c1 - b.c0,) if b.is_vec else (b.r1 - b.r0, b.c1 - b.c0)
        out = np.empty(shape, np.float32)
        check(lib().ggb_state_param_get(self.h, i, which, _ptr(out)))
        return out

    def weights(self) -> list[np.ndarray]:
        return [self._get(i, 0) for i in range(len(self.blocks))]

    def grads(self) -> list[np.ndarray]:
        return [self._get(i, 1) for i in range(len(self.blocks))]

    def moments(self) -> tuple[list[np.ndarray], list[np.ndarray]]:
        return ([self._get(i, 2) for i in range(len(self.blocks))],
                [self._get(i, 3) for i in range(len(self.blocks))])

    def set_weight(self, i: int, w: np.ndarray):
        w = np.ascontiguousarray(w, np.float32)
        check(lib().ggb_state_param_set(self.h, i, 0, _ptr(w)))

    def logits(self) -> tuple[tuple[int, int, int, int], np.ndarray]:
        dims = np.zeros(4, np.int64)
        check(lib().ggb_state_logits(self.h, _ptr(dims), None))
        out = np.empty((dims[1] - dims[0], dims[3] - dims[2]), np.float32)
        check(lib().ggb_state_logits(self.h, _ptr(dims), _ptr(out)))
        return tuple(int(x) for x in dims), out

    def loss_device_ptr(self) -> int:
        p = P()
        check(lib().ggb_last_loss_device(self.h, C.byref(p)))
        return int(p.value)

    def close(self):
        if getattr(self, "h", None):
            lib().ggb_state_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_state(ctx: Context, cfg: ModelConfig, seed: int, compute: int = COMPUTE_ACCURATE) -> ModelState:
    return ModelState(ctx, cfg, seed, compute)


def forward(ctx: Context, st: ModelState, batch: StepBatch, prec: int, training: bool, run_seed: int,
            global_step: int, rmsnorm_eps: float = 1e-6) -> None:
    check(lib().ggb_forward(ctx.h, st.h, batch.h, prec, int(training), run_seed, global_step, rmsnorm_eps))


def train_step(ctx: Context, st: ModelState, batch: StepBatch, prec: int, run_seed: int, global_step: int,
               rmsnorm_eps: float = 1e-6, sync_loss: bool = True) -> float | None:
    """forward + cross-entropy + backward; gradients left un-synced (model.hpp:459-478)."""
    loss = C.c_float()
    check(lib().ggb_train_step(ctx.h, st.h, batch.h, prec, run_seed, global_step, rmsnorm_eps,
                               C.byref(loss) if sync_loss else None))
    return float(loss.value) if sync_loss else None


def loss_to_host_async(ctx: Context, st: ModelState, host_dst_ptr: int) -> None:
    """Enqueue the D2H copy of the last train_step's loss into pinned host
    memory at host_dst_ptr without waiting (read it after a later wait)."""
    check(lib().ggb_loss_to_host_async(ctx.h, st.h, C.c_void_p(host_dst_ptr)))


@dataclass
class EvalCounts:
    """EvalCounts (model.hpp:480-490): index 0 train, 1 val, 2 test."""
    correct: tuple
    total: tuple

    def accuracy(self, split: int) -> float:
        return 0.0 if self.total[split] == 0 else self.correct[split] / self.total[split]


def build_eval_batch(ctx: Context, graph: Graph, run_seed: int) -> StepBatch:
    """train_run's eval batch: build_step_batch(b = n, seed, step 0) (model.hpp:625)."""
    return build_step_batch(ctx, graph, graph.n, run_seed, 0)


def evaluate_full_graph(ctx: Context, st: ModelState, eval_batch: StepBatch, graph: Graph,
                        precision: int = FP32, rmsnorm_eps: float = 1e-6) -> EvalCounts:
    """evaluate_full_graph (model.hpp:493-537): dropout-off forward over every vertex,
    argmax (ties to the lowest class id), per-split counts summed over the grid."""
    c = np.zeros(6, np.uint64)
    check(lib().ggb_evaluate_full_graph(ctx.h, st.h, eval_batch.h, graph.h, precision, rmsnorm_eps, _ptr(c)))
    return EvalCounts(tuple(int(x) for x in c[:3]), tuple(int(x) for x in c[3:]))


def dp_sync(ctx: Context, st: ModelState) -> None:
    check(lib().ggb_dp_sync(ctx.h, st.h))


def optimizer_step(ctx: Context, st: ModelState, optimizer: int = ADAM, lr: float = 1e-3) -> None:
    check(lib().ggb_optimizer_step(ctx.h, st.h, optimizer, lr))


def hash_combine(a: int, b: int) -> int:
    """rng.hpp:17-19 (host-side seed derivation, e.g. group seeds model.hpp:620-621)."""
    m = (1 << 64) - 1

    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & m
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
        return x ^ (x >> 31)

    return sm((a ^ ((0x9E3779B97F4A7C15 + ((b << 6) & m) + (b >> 2)) & m)) & m)


# ---- layer operators (pmm.hpp:76-401) over device blocks -----------------------

@dataclass
class DeviceBlock:
    """One rank's block of a ShardedTensor (tensor.hpp:75-86) in HBM: ordered
    layout (grid axes X=1, Y=2, Z=3), global shape, explicit partition
    offsets, the block at device pointer `ptr` with leading dimension `ld`."""
    layout: tuple[int, int]
    g_rows: int
    g_cols: int
    row_off: np.ndarray
    col_off: np.ndarray
    ptr: int
    ld: int

    def c(self) -> BlockC:
        self._ro = np.ascontiguousarray(self.row_off, np.int64)
        self._co = np.ascontiguousarray(self.col_off, np.int64)
        return BlockC(self.layout[0], self.layout[1], self.g_rows, self.g_cols, self._ro.ctypes.data,
                      self._co.ctypes.data, self.ptr, self.ld)


def _pb(x):
    return C.byref(x) if x is not None else None


def contract(ctx: Context, a: DeviceBlock, b: DeviceBlock, out: DeviceBlock, prec: int = FP32) -> None:
    ca, cb, cc = a.c(), b.c(), out.c()
    check(lib().ggb_contract(ctx.h, C.byref(ca), C.byref(cb), C.byref(cc), prec))


def spmm(ctx: Context, a: CsrBlockC, f: DeviceBlock, out: DeviceBlock, prec: int = FP32) -> None:
    cf, co = f.c(), out.c()
    check(lib().ggb_spmm(ctx.h, C.byref(a), C.byref(cf), C.byref(co), prec))


def transposed(ctx: Context, t: DeviceBlock, out: DeviceBlock) -> None:
    ct, co = t.c(), out.c()
    check(lib().ggb_transposed(ctx.h, C.byref(ct), C.byref(co)))


def gather_full(ctx: Context, t: DeviceBlock, full_ptr: int, ld_full: int) -> None:
    ct = t.c()
    check(lib().ggb_gather_full(ctx.h, C.byref(ct), full_ptr, ld_full))


def reshard(ctx: Context, src: DeviceBlock, dst: DeviceBlock) -> None:
    cs, cd = src.c(), dst.c()
    check(lib().ggb_reshard(ctx.h, C.byref(cs), C.byref(cd)))


def rmsnorm_fwd(ctx: Context, x: DeviceBlock, gamma_ptr: int, eps: float, y: DeviceBlock, rms_ptr: int) -> None:
    cx, cy = x.c(), y.c()
    check(lib().ggb_rmsnorm_fwd(ctx.h, C.byref(cx), gamma_ptr, eps, C.byref(cy), rms_ptr))


def rmsnorm_bwd(ctx: Context, x: DeviceBlock, gamma_ptr: int, rms_ptr: int, dy: DeviceBlock, dx: DeviceBlock,
                dgamma_ptr: int) -> None:
    cx, cdy, cdx = x.c(), dy.c(), dx.c()
    check(lib().ggb_rmsnorm_bwd(ctx.h, C.byref(cx), gamma_ptr, rms_ptr, C.byref(cdy), C.byref(cdx), dgamma_ptr))


def fused_elementwise_fwd(ctx: Context, x: DeviceBlock, h_prev: DeviceBlock | None, rate: float, mask_key: int,
                          training: bool, out: DeviceBlock, keep_bits_ptr: int | None) -> None:
    cx, co = x.c(), out.c()
    ch = h_prev.c() if h_prev is not None else None
    check(lib().ggb_fused_elementwise_fwd(ctx.h, C.byref(cx), _pb(ch), rate, mask_key, int(training), C.byref(co),
                                          keep_bits_ptr))


def keep_scale(rate: float, training: bool) -> float:
    """The fp32 scale of a kept element (pmm.hpp:311)."""
    return float(np.float32(1.0 / (1.0 - rate))) if training and rate > 0 else 1.0


def fused_elementwise_bwd(ctx: Context, dy: DeviceBlock, keep_bits_ptr: int, scale: float, dx: DeviceBlock) -> None:
    cdy, cdx = dy.c(), dx.c()
    check(lib().ggb_fused_elementwise_bwd(ctx.h, C.byref(cdy), keep_bits_ptr, scale, C.byref(cdx)))


def mask_words(cols: int) -> int:
    return int(lib().ggb_mask_words(cols))


def cross_entropy(ctx: Context, logits: DeviceBlock, labels_ptr: int, loss_ptr: int, grad: DeviceBlock) -> None:
    cl, cg = logits.c(), grad.c()
    check(lib().ggb_cross_entropy(ctx.h, C.byref(cl), labels_ptr, loss_ptr, C.byref(cg)))


def batch_csr_block(batch: StepBatch, plane: int, transposed: bool = False) -> CsrBlockC:
    out = CsrBlockC()
    check(lib().ggb_batch_csr_block(batch.h, plane, int(transposed), C.byref(out)))
    out._batch = batch  # the pointers live as long as the batch
    return out


def loss(ctx: Context, st: "ModelState", batch: StepBatch) -> float:
    """parallel_cross_entropy on the last forward's logits (train_step's seam)."""
    out = C.c_float()
    check(lib().ggb_loss(ctx.h, st.h, batch.h, C.byref(out)))
    return out.value


def backward(ctx: Context, st: "ModelState", batch: StepBatch, prec: int = FP32) -> None:
    check(lib().ggb_backward(ctx.h, st.h, batch.h, prec))
