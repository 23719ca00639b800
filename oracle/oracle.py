"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the mini-batch GCN step.

Two layers:

* ``liboracle.so`` (oracle.c): our C restatement of the bit-exact parts
  (RNG, partial Fisher-Yates sampler, Alg. 2 shard extraction, dataset
  generation). Wrapped by the ``orc_*`` helpers below.
* ``serial_train_step`` / ``adam_step``: a numpy fp32 restatement of the
  serial (1x1x1x1) training step, citing the reference lines it follows.

Plus ``Ref``: ctypes access to the UNMODIFIED reference compiled in place
(oracle/_ref/libgridgnn_ref.so via oracle/ref_shim.cpp), used to pin the
restatement and as the CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. The product path never
does.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIBORACLE = os.path.join(HERE, "liboracle.so")
_LIBREF = os.path.join(HERE, "_ref", "libgridgnn_ref.so")

U64 = C.c_uint64
I64 = C.c_int64
P = C.c_void_p


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so (always) and _ref (when /root/reference exists)."""
    targets = ["oracle"]
    if ref is None:
        ref = os.path.isdir("/root/reference/proj")
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(P)


_orc = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(_LIBORACLE):
            build(ref=False)
        L = C.CDLL(_LIBORACLE)
        L.orc_splitmix64.restype = U64
        L.orc_splitmix64.argtypes = [U64]
        L.orc_hash_combine.restype = U64
        L.orc_hash_combine.argtypes = [U64, U64]
        L.orc_element_unit.restype = C.c_double
        L.orc_element_unit.argtypes = [U64, U64, U64]
        L.orc_bf16_round.restype = C.c_float
        L.orc_bf16_round.argtypes = [C.c_float]
        L.orc_dropout_key.restype = U64
        L.orc_dropout_key.argtypes = [U64, C.c_int, U64, C.c_int]
        L.orc_sample_vertices.argtypes = [I64, I64, U64, U64, P]
        L.orc_block_partition.argtypes = [I64, C.c_int, P]
        L.orc_sample_partition.argtypes = [P, I64, P, I64, P]
        L.orc_local_minibatch.argtypes = [I64, P, P, P, I64, I64, I64, I64, I64, U64, U64, P,
                                          P, P, P, P, P, P]
        L.orc_synthetic_edges.restype = I64
        L.orc_synthetic_edges.argtypes = [I64, C.c_double, U64, P]
        L.orc_sample_vertices_reject.argtypes = [I64, I64, U64, U64, U64, P]
        L.orc_rmat_edges.argtypes = [C.c_int, I64, C.c_double, C.c_double, C.c_double, U64, P]
        L.orc_normalize_adjacency.restype = I64
        L.orc_normalize_adjacency.argtypes = [P, I64, I64, P, P, P]
        L.orc_features.argtypes = [I64, I64, U64, P]
        L.orc_labels.argtypes = [I64, P, I64, P]
        L.orc_split.argtypes = [I64, U64, P]
        L.orc_fill_weight.argtypes = [I64, I64, U64, P]
        L.orc_dropout_keep.argtypes = [U64, I64, I64, I64, I64, C.c_double, P]
        _orc = L
    return _orc


# ---- bit-exact restatement (C) ------------------------------------------------

def splitmix64(x: int) -> int:
    return orc().orc_splitmix64(x)


def hash_combine(a: int, b: int) -> int:
    return orc().orc_hash_combine(a, b)


def element_unit(k: int, i: int, j: int) -> float:
    return orc().orc_element_unit(k, i, j)


def bf16_round(x: float) -> float:
    return orc().orc_bf16_round(x)


def dropout_key(seed: int, dp: int, gstep: int, layer: int) -> int:
    return orc().orc_dropout_key(seed, dp, gstep, layer)


def sample_vertices(n: int, b: int, seed: int, step: int) -> np.ndarray:
    out = np.empty(b, np.int64)
    if orc().orc_sample_vertices(n, b, seed, step, _ptr(out)) != 0:
        raise ValueError("sample_vertices: need 1 <= b <= n")
    return out


def sample_vertices_reject(n: int, b: int, seed: int, step: int, reject_mod: int) -> np.ndarray:
    """sample_vertices with the test-only extra rejection rule (x % reject_mod == 0)."""
    out = np.empty(b, np.int64)
    orc().orc_sample_vertices_reject(n, b, seed, step, reject_mod, _ptr(out))
    return out


def block_partition(n: int, g: int) -> np.ndarray:
    out = np.empty(g + 1, np.int64)
    if orc().orc_block_partition(n, g, _ptr(out)) != 0:
        raise ValueError("block_partition: g must be >= 1")
    return out


def sample_partition(s: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(s, np.int64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    out = np.empty(len(offsets), np.int64)
    orc().orc_sample_partition(_ptr(s), len(s), _ptr(offsets), len(offsets), _ptr(out))
    return out


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        for r in range(self.n_rows):
            lo, hi = self.row_ptr[r], self.row_ptr[r + 1]
            d[r, self.col_idx[lo:hi]] = self.values[lo:hi]
        return d


@dataclass
class LocalShard:
    row_lo: int
    row_hi: int
    col_lo: int
    col_hi: int
    nnz_extracted: int
    nnz_kept: int
    a: Csr
    a_t: Csr


def local_minibatch(adj: Csr, r0: int, r1: int, c0: int, c1: int, b: int, seed: int,
                    step: int) -> LocalShard:
    """build_local_minibatch on the static shard rows [r0,r1) x cols [c0,c1)."""
    L = orc()
    meta = np.zeros(6, np.int64)
    args = [adj.n_rows, _ptr(adj.row_ptr), _ptr(adj.col_idx), _ptr(adj.values), r0, r1, c0, c1,
            b, seed, step, _ptr(meta)]
    if L.orc_local_minibatch(*args, None, None, None, None, None, None) != 0:
        raise ValueError("local_minibatch: bad arguments")
    nr, nc, kept = int(meta[1] - meta[0]), int(meta[3] - meta[2]), int(meta[5])
    arp, acol, aval = np.empty(nr + 1, np.int64), np.empty(kept, np.int64), np.empty(kept)
    trp, tcol, tval = np.empty(nc + 1, np.int64), np.empty(kept, np.int64), np.empty(kept)
    L.orc_local_minibatch(*args, _ptr(arp), _ptr(acol), _ptr(aval), _ptr(trp), _ptr(tcol),
                          _ptr(tval))
    return LocalShard(int(meta[0]), int(meta[1]), int(meta[2]), int(meta[3]), int(meta[4]), kept,
                      Csr(nr, nc, arp, acol, aval), Csr(nc, nr, trp, tcol, tval))


@dataclass
class Dataset:
    n: int
    d_in: int
    n_classes: int
    adj: Csr
    features: np.ndarray  # n x d_in float32
    labels: np.ndarray  # int32
    split: np.ndarray  # uint8


def synthetic_edges(n: int, avg_degree: float, seed: int) -> np.ndarray:
    L = orc()
    m = L.orc_synthetic_edges(n, avg_degree, seed, None)
    uv = np.empty((m, 2), np.int64)
    L.orc_synthetic_edges(n, avg_degree, seed, _ptr(uv))
    return uv


def rmat_edges(scale: int, m: int, seed: int, a: float = 0.57, b: float = 0.19, c: float = 0.19) -> np.ndarray:
    """R-MAT edge list (oracle.c orc_rmat_edges; restates gendata.cu k_rmat)."""
    uv = np.empty((m, 2), np.int64)
    orc().orc_rmat_edges(scale, m, a, b, c, seed, _ptr(uv))
    return uv


def normalize_adjacency(uv: np.ndarray, n: int) -> Csr:
    L = orc()
    uv = np.ascontiguousarray(uv, np.int64)
    nnz = L.orc_normalize_adjacency(_ptr(uv), len(uv), n, None, None, None)
    if nnz < 0:
        raise ValueError("normalize_adjacency: vertex id out of range")
    rp, col, val = np.empty(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
    L.orc_normalize_adjacency(_ptr(uv), len(uv), n, _ptr(rp), _ptr(col), _ptr(val))
    return Csr(n, n, rp, col, val)


def dataset_from_edges(n: int, uv: np.ndarray, d_in: int, n_classes: int, seed: int) -> Dataset:
    """generate_synthetic (dataset.cpp:85-131) for a given edge list."""
    L = orc()
    adj = normalize_adjacency(uv, n)
    feats = np.empty((n, d_in), np.float32)
    L.orc_features(n, d_in, seed, _ptr(feats))
    labels = np.empty(n, np.int32)
    L.orc_labels(n, _ptr(adj.row_ptr), n_classes, _ptr(labels))
    split = np.empty(n, np.uint8)
    L.orc_split(n, seed, _ptr(split))
    return Dataset(n, d_in, n_classes, adj, feats, labels, split)


def generate_synthetic(n: int, avg_degree: float, d_in: int, n_classes: int, seed: int) -> Dataset:
    return dataset_from_edges(n, synthetic_edges(n, avg_degree, seed), d_in, n_classes, seed)


def fill_weight(rows: int, cols: int, key: int) -> np.ndarray:
    out = np.empty((rows, cols), np.float32)
    orc().orc_fill_weight(rows, cols, key, _ptr(out))
    return out


def dropout_keep(key: int, r0: int, c0: int, rows: int, cols: int, rate: float) -> np.ndarray:
    out = np.empty((rows, cols), np.uint8)
    orc().orc_dropout_keep(key, r0, c0, rows, cols, rate, _ptr(out))
    return out.astype(bool)


# ---- numpy fp32 restatement of the serial training step ------------------------

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

    def arrays(self):
        mc = np.array([self.layers, self.d_in, self.d_h, self.d_out, int(self.use_rmsnorm),
                       int(self.use_dropout), int(self.use_residual)], np.int64)
        md = np.array([self.dropout_rate], np.float64)
        return mc, md

    def param_shapes(self) -> list[tuple[str, tuple[int, ...]]]:
        """param_views order (model.hpp:107-133)."""
        out = [("win", (self.d_in, self.d_h))]
        for l in range(self.layers):
            out.append((f"w{l + 1}", (self.d_h, self.d_h)))
            if self.use_rmsnorm:
                out.append((f"gamma{l + 1}", (self.d_h,)))
        out.append(("wout", (self.d_h, self.d_out)))
        return out


def init_params(cfg: ModelConfig, seed: int) -> list[np.ndarray]:
    """init_state (model.hpp:175-208) on the serial grid."""
    ps = [fill_weight(cfg.d_in, cfg.d_h, hash_combine(seed, 101))]
    for l in range(1, cfg.layers + 1):
        ps.append(fill_weight(cfg.d_h, cfg.d_h, hash_combine(seed, 200 + l)))
        if cfg.use_rmsnorm:
            ps.append(np.ones(cfg.d_h, np.float32))
    ps.append(fill_weight(cfg.d_h, cfg.d_out, hash_combine(seed, 102)))
    return ps


def _split_params(cfg: ModelConfig, ps):
    win, wout = ps[0], ps[-1]
    wl, gm = [], []
    k = 1
    for _ in range(cfg.layers):
        wl.append(ps[k])
        k += 1
        if cfg.use_rmsnorm:
            gm.append(ps[k])
            k += 1
    return win, wl, gm, wout


@dataclass
class StepResult:
    loss: float
    logits: np.ndarray
    grads: list[np.ndarray]


def serial_train_step(cfg: ModelConfig, ps: list[np.ndarray], ds: Dataset, b: int, seed: int,
                      step: int, eps: float = 1e-6, training: bool = True,
                      group_seed: int | None = None) -> StepResult:
    """forward + parallel_cross_entropy + backward on the 1x1x1x1 grid.

    Restates build_step_batch (model.hpp:250-309; at 1x1x1x1 every plane is
    the full batch adjacency), forward (model.hpp:335-376), the fused
    element-wise op (pmm.hpp:299-341), RMSNorm (pmm.hpp:214-287), the
    cross-entropy (pmm.hpp:352-401) and backward (model.hpp:378-420), in fp32.
    """
    import scipy.sparse as sp

    if group_seed is None:
        group_seed = hash_combine(seed, 0)
    f32 = np.float32
    n = ds.n
    lb = local_minibatch(ds.adj, 0, n, 0, n, b, group_seed, step)
    s = sample_vertices(n, b, group_seed, step)
    A = sp.csr_matrix((lb.a.values.astype(f32), lb.a.col_idx, lb.a.row_ptr), shape=(b, b))
    x_in = ds.features[s].astype(f32)
    labels = ds.labels[s].astype(np.int64)
    win, wl, gm, wout = _split_params(cfg, ps)
    H = cfg.d_h
    rate = cfg.dropout_rate if cfg.use_dropout else 0.0
    drop = training and rate > 0.0
    keep_scale = f32(1.0 / (1.0 - rate)) if drop else f32(1.0)

    xs = [x_in @ win]
    cache = []
    for l in range(1, cfg.layers + 1):
        hagg = (A @ xs[-1]).astype(f32)
        xw = hagg @ wl[l - 1]
        if cfg.use_rmsnorm:
            ss = np.sum(xw * xw, axis=1, dtype=f32)
            rms = np.sqrt(ss / f32(H) + f32(eps)).astype(f32)
            xn = gm[l - 1][None, :] * xw * (f32(1.0) / rms)[:, None]
        else:
            rms, xn = None, xw
        sc = (xn > 0).astype(f32)
        if drop:
            keep = dropout_keep(dropout_key(seed, 0, step, l), 0, 0, b, H, rate)
            sc = np.where(keep, sc * keep_scale, f32(0.0)).astype(f32)
        out = xn * sc
        if cfg.use_residual:
            out = out + xs[-1]
        cache.append((hagg, xw, rms, sc))
        xs.append(out.astype(f32))
    logits = xs[-1] @ wout

    # cross-entropy, mean over the batch rows
    mx = logits.max(axis=1)
    e = np.exp(logits - mx[:, None])
    z = e.sum(axis=1, dtype=f32)
    lse = mx + np.log(z)
    loss = float(np.mean((lse - logits[np.arange(b), labels]).astype(np.float64)))
    g = e / z[:, None]
    g[np.arange(b), labels] -= f32(1.0)
    dlogits = (g * f32(1.0 / b)).astype(f32)

    gw_out = xs[-1].T @ dlogits
    dxh = dlogits @ wout.T
    g_wl = [None] * cfg.layers
    g_gm = [None] * cfg.layers
    AT = A.T.tocsr()
    for l in range(cfg.layers, 0, -1):
        hagg, xw, rms, sc = cache[l - 1]
        dxn = dxh * sc
        dres = dxh if cfg.use_residual else None
        if cfg.use_rmsnorm:
            gam = gm[l - 1]
            srow = np.sum(dxn * gam[None, :] * xw, axis=1, dtype=f32)
            inv = f32(1.0) / rms
            coef = srow / (f32(H) * rms * rms * rms)
            dxw = gam[None, :] * dxn * inv[:, None] - xw * coef[:, None]
            g_gm[l - 1] = np.sum(dxn * xw * inv[:, None], axis=0, dtype=f32)
        else:
            dxw = dxn
        g_wl[l - 1] = hagg.T @ dxw
        dhagg = dxw @ wl[l - 1].T
        dxh = (AT @ dhagg).astype(f32)
        if dres is not None:
            dxh = dxh + dres
    gw_in = x_in.T @ dxh
    grads = [gw_in]
    for l in range(cfg.layers):
        grads.append(g_wl[l])
        if cfg.use_rmsnorm:
            grads.append(g_gm[l])
    grads.append(gw_out)
    return StepResult(loss, logits, [np.asarray(x, f32) for x in grads])


def adam_step(ps, grads, ms, vs, t: int, lr: float = 1e-3):
    """optimizer_step, Adam branch (model.hpp:444-455): fp64 math, fp32 store."""
    b1, b2, eps = 0.9, 0.999, 1e-8
    bc1 = 1.0 - math.pow(b1, t)
    bc2 = 1.0 - math.pow(b2, t)
    for k in range(len(ps)):
        g = grads[k].astype(np.float64)
        m = b1 * ms[k].astype(np.float64) + (1.0 - b1) * g
        v = b2 * vs[k].astype(np.float64) + (1.0 - b2) * g * g
        ms[k] = m.astype(np.float32)
        vs[k] = v.astype(np.float32)
        ps[k] = ps[k] - (lr * (m / bc1) / (np.sqrt(v / bc2) + eps)).astype(np.float32)


# ---- the unmodified reference (oracle/_ref) ---------------------------------------

class Ref:
    """ctypes view of oracle/_ref/libgridgnn_ref.so (reference compiled in place)."""

    def __init__(self):
        if not os.path.exists(_LIBREF):
            if os.path.isdir("/root/reference/proj"):
                build(ref=True)
            else:
                raise FileNotFoundError(f"{_LIBREF} missing and /root/reference unavailable")
        L = C.CDLL(_LIBREF)
        L.ref_last_error.restype = C.c_char_p
        L.ref_sample_vertices.argtypes = [I64, I64, U64, U64, P]
        L.ref_splitmix64.restype = U64
        L.ref_splitmix64.argtypes = [U64]
        L.ref_hash_combine.restype = U64
        L.ref_hash_combine.argtypes = [U64, U64]
        L.ref_element_unit.restype = C.c_double
        L.ref_element_unit.argtypes = [U64, U64, U64]
        L.ref_bf16_round.restype = C.c_float
        L.ref_bf16_round.argtypes = [C.c_float]
        L.ref_dropout_key.restype = U64
        L.ref_dropout_key.argtypes = [U64, C.c_int, U64, C.c_int]
        L.ref_block_partition.argtypes = [I64, C.c_int, P]
        L.ref_dataset_synthetic.restype = P
        L.ref_dataset_synthetic.argtypes = [I64, C.c_double, I64, I64, U64]
        L.ref_dataset_from_edges.restype = P
        L.ref_dataset_from_edges.argtypes = [I64, P, I64, I64, P, I64, P, P]
        L.ref_dataset_free.argtypes = [P]
        L.ref_dataset_load.restype = P
        L.ref_dataset_load.argtypes = [C.c_char_p] * 4
        L.ref_save_synthetic.argtypes = [I64, C.c_double, I64, I64, U64] + [C.c_char_p] * 4
        L.ref_dataset_info.argtypes = [P, P]
        L.ref_dataset_export.argtypes = [P, P, P, P, P, P, P]
        L.ref_synthetic_edges.restype = I64
        L.ref_synthetic_edges.argtypes = [I64, C.c_double, U64, P]
        L.ref_step_batch.restype = P
        L.ref_step_batch.argtypes = [P, P, C.c_int, C.c_int, I64, U64, U64]
        L.ref_batch_free.argtypes = [P]
        L.ref_batch_sample.argtypes = [P, P]
        L.ref_batch_counters.argtypes = [P, P]
        L.ref_batch_offsets.argtypes = [P, C.c_int, P]
        L.ref_batch_num_planes.argtypes = [P]
        L.ref_batch_plane.argtypes = [P, C.c_int, C.c_int, P, P, P, P]
        L.ref_batch_x_in.argtypes = [P, P, P]
        L.ref_batch_labels.argtypes = [P, P]
        L.ref_param_total.restype = I64
        L.ref_param_total.argtypes = [P, P]
        L.ref_train.argtypes = [P, P, P, P, I64, U64, U64, C.c_int, C.c_int, C.c_int,
                                C.c_double, C.c_double, P, P, P, P]
        L.ref_init_weights.argtypes = [P, P, U64, P]
        L.ref_train_eval.argtypes = [P, P, P, P, I64, U64, C.c_int, C.c_int, C.c_int, C.c_double,
                                     C.c_double, P, P]
        L.ref_bench.argtypes = [P, P, P, P, I64, U64, C.c_int, C.c_int, C.c_int, P, P]
        L.ref_comm_stats.argtypes = [P, P, P, P, I64, U64, C.c_int, C.c_int, C.c_int, P]
        L.ref_contract.argtypes = [I64, I64, I64, P, P, C.c_int, P]
        L.ref_spmm.argtypes = [I64, I64, P, P, P, P, I64, C.c_int, P]
        L.ref_rmsnorm.argtypes = [I64, I64, P, P, C.c_float, P, P, P, P, P]
        L.ref_fused.argtypes = [I64, I64, P, P, C.c_double, U64, C.c_int, P, P, P, P]
        L.ref_cross_entropy.argtypes = [I64, I64, P, P, P, P]
        self.L = L

    def _check(self, rc: int):
        if rc != 0:
            msg = self.L.ref_last_error().decode()
            raise (ValueError if rc == 1 else RuntimeError)(msg)

    def sample_vertices(self, n, b, seed, step):
        out = np.empty(b, np.int64)
        self._check(self.L.ref_sample_vertices(n, b, seed, step, _ptr(out)))
        return out

    # datasets are opaque handles owned by the caller
    def dataset_synthetic(self, n, avg_degree, d_in, n_classes, seed):
        h = self.L.ref_dataset_synthetic(n, avg_degree, d_in, n_classes, seed)
        if not h:
            raise ValueError(self.L.ref_last_error().decode())
        return h

    def load_files(self, edges, features, labels, split):
        """load_dataset (dataset.cpp:178-239) in a numpy-free child interpreter
        (see save_synthetic): ((row_ptr, col_idx, values), features, labels,
        split, n_classes); raises ValueError with the reference's message."""
        import tempfile
        with tempfile.TemporaryDirectory() as td:
            code = ("import ctypes as C, sys, os\n"
                    f"L = C.CDLL({_LIBREF!r})\n"
                    "L.ref_last_error.restype = C.c_char_p\n"
                    "L.ref_dataset_load.restype = C.c_void_p\n"
                    "L.ref_dataset_load.argtypes = [C.c_char_p] * 4\n"
                    "L.ref_dataset_info.argtypes = [C.c_void_p, C.c_void_p]\n"
                    "L.ref_dataset_export.argtypes = [C.c_void_p] * 7\n"
                    f"h = L.ref_dataset_load(*[a.encode() for a in {[str(x) for x in (edges, features, labels, split)]!r}])\n"
                    "if not h:\n"
                    "    sys.stderr.write(L.ref_last_error().decode()); sys.exit(1)\n"
                    "info = (C.c_int64 * 4)(); L.ref_dataset_info(h, info)\n"
                    "n, nnz, d, k = info\n"
                    "bufs = [(C.c_int64 * (n + 1))(), (C.c_int64 * nnz)(), (C.c_double * nnz)(),"
                    " (C.c_float * (n * d))(), (C.c_int32 * n)(), (C.c_uint8 * n)()]\n"
                    "L.ref_dataset_export(h, *[C.addressof(b) for b in bufs])\n"
                    f"td = {td!r}\n"
                    "open(os.path.join(td, 'info'), 'w').write('%d %d %d %d' % (n, nnz, d, k))\n"
                    "for i, b in enumerate(bufs): open(os.path.join(td, 'a%d' % i), 'wb').write(bytes(b))\n")
            r = subprocess.run(["python3", "-c", code], capture_output=True, text=True)
            if r.returncode != 0:
                raise (ValueError if r.returncode == 1 else RuntimeError)(r.stderr.strip())
            n, nnz, d, k = (int(x) for x in open(os.path.join(td, "info")).read().split())
            rd = lambda i, dt: np.fromfile(os.path.join(td, "a%d" % i), dt)
            return ((rd(0, np.int64), rd(1, np.int64), rd(2, np.float64)), rd(3, np.float32).reshape(n, d),
                    rd(4, np.int32), rd(5, np.uint8), k)

    def save_synthetic(self, n, avg_degree, d_in, n_classes, seed, edges, features, labels, split):
        """The CLI's gen command (gridgnn_main.cpp:313-324). Run in a child
        interpreter that never imports numpy: with numpy loaded, the
        reference's std::ofstream writers crash in this image (the readers and
        everything else are unaffected)."""
        code = ("import ctypes as C, sys\n"
                f"L = C.CDLL({_LIBREF!r})\n"
                "L.ref_last_error.restype = C.c_char_p\n"
                "L.ref_save_synthetic.argtypes = [C.c_int64, C.c_double, C.c_int64, C.c_int64, C.c_uint64]"
                " + [C.c_char_p] * 4\n"
                f"rc = L.ref_save_synthetic({int(n)}, {float(avg_degree)!r}, {int(d_in)}, {int(n_classes)}, "
                f"{int(seed)}, *[a.encode() for a in {[str(x) for x in (edges, features, labels, split)]!r}])\n"
                "sys.stderr.write(L.ref_last_error().decode())\n"
                "sys.exit(rc)\n")
        r = subprocess.run(["python3", "-c", code], capture_output=True, text=True)
        if r.returncode != 0:
            raise (ValueError if r.returncode == 1 else RuntimeError)(r.stderr.strip())

    def dataset_from(self, ds: Dataset, uv: np.ndarray):
        uv = np.ascontiguousarray(uv, np.int64)
        h = self.L.ref_dataset_from_edges(ds.n, _ptr(uv), len(uv), ds.d_in, _ptr(ds.features),
                                          ds.n_classes, _ptr(ds.labels), _ptr(ds.split))
        if not h:
            raise ValueError(self.L.ref_last_error().decode())
        return h

    def dataset_export(self, h) -> Dataset:
        info = np.zeros(4, np.int64)
        self.L.ref_dataset_info(h, _ptr(info))
        n, nnz, d_in, ncls = (int(x) for x in info)
        rp, col, val = np.empty(n + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        feats, labels = np.empty((n, d_in), np.float32), np.empty(n, np.int32)
        split = np.empty(n, np.uint8)
        self.L.ref_dataset_export(h, _ptr(rp), _ptr(col), _ptr(val), _ptr(feats), _ptr(labels),
                                  _ptr(split))
        return Dataset(n, d_in, ncls, Csr(n, n, rp, col, val), feats, labels, split)

    def free_dataset(self, h):
        self.L.ref_dataset_free(h)

    def step_batch(self, h, dims, rank, layers, b, group_seed, step) -> dict:
        d = np.asarray(dims, np.int32)
        bh = self.L.ref_step_batch(h, _ptr(d), rank, layers, b, group_seed, step)
        if not bh:
            raise ValueError(self.L.ref_last_error().decode())
        try:
            out = {"sample": np.empty(b, np.int64)}
            self.L.ref_batch_sample(bh, _ptr(out["sample"]))
            cnt = np.zeros(2, np.uint64)
            self.L.ref_batch_counters(bh, _ptr(cnt))
            out["counters"] = cnt
            offs = {}
            for ax in (1, 2, 3):
                buf = np.empty(int(dims[ax]) + 1, np.int64)
                self.L.ref_batch_offsets(bh, ax, _ptr(buf))
                offs[ax] = buf
            out["batch_off"] = offs
            planes = []
            for p in range(self.L.ref_batch_num_planes(bh)):
                pair = []
                for t in (0, 1):
                    dm = np.zeros(7, np.int64)
                    self.L.ref_batch_plane(bh, p, t, _ptr(dm), None, None, None)
                    rp, col = np.empty(dm[0] + 1, np.int64), np.empty(dm[2], np.int64)
                    val = np.empty(dm[2])
                    self.L.ref_batch_plane(bh, p, t, _ptr(dm), _ptr(rp), _ptr(col), _ptr(val))
                    pair.append({"dims": dm.copy(), "csr": Csr(int(dm[0]), int(dm[1]), rp, col, val)})
                planes.append(pair)
            out["planes"] = planes
            xd = np.zeros(4, np.int64)
            self.L.ref_batch_x_in(bh, _ptr(xd), None)
            x = np.empty((xd[1] - xd[0], xd[3] - xd[2]), np.float32)
            self.L.ref_batch_x_in(bh, _ptr(xd), _ptr(x))
            out["x_in"] = (xd.copy(), x)
            lab = np.empty(b, np.int32)
            self.L.ref_batch_labels(bh, _ptr(lab))
            out["labels"] = lab
            return out
        finally:
            self.L.ref_batch_free(bh)

    def train(self, h, dims, cfg: ModelConfig, b, seed, step0=0, n_steps=1, prec=0,
              optimizer=-1, lr=1e-3, eps=1e-6, want_logits=True, want_weights=False):
        mc, md = cfg.arrays()
        d = np.asarray(dims, np.int32)
        total = int(self.L.ref_param_total(_ptr(mc), _ptr(md)))
        losses = np.zeros(n_steps, np.float32)
        logits = np.zeros((b, cfg.d_out), np.float32) if want_logits else None
        grads = np.zeros(total, np.float32)
        weights = np.zeros(total, np.float32) if want_weights else None
        self._check(self.L.ref_train(h, _ptr(d), _ptr(mc), _ptr(md), b, seed, step0, n_steps, prec,
                                     optimizer, lr, eps, _ptr(losses), _ptr(logits), _ptr(grads),
                                     _ptr(weights)))
        return losses, logits, unflatten(cfg, grads), (unflatten(cfg, weights) if want_weights else None)

    def train_eval(self, h, n, dims, cfg: ModelConfig, b, seed, n_steps=1, prec=0, optimizer=1, lr=1e-3,
                   eps=1e-6, want_logits=True):
        """n_steps of train_run's step loop, then evaluate_full_graph (model.hpp:493-537).
        Returns (counts[6] = correct train/val/test + totals, eval logits n x d_out or None)."""
        mc, md = cfg.arrays()
        d = np.asarray(dims, np.int32)
        counts = np.zeros(6, np.uint64)
        logits = np.zeros((n, cfg.d_out), np.float32) if want_logits else None
        self._check(self.L.ref_train_eval(h, _ptr(d), _ptr(mc), _ptr(md), b, seed, n_steps, prec, optimizer, lr,
                                          eps, _ptr(counts), _ptr(logits)))
        return counts, logits

    def comm_stats(self, h, dims, cfg: ModelConfig, b, seed, n_steps, prec=0, evaluate=False):
        """The reference's CommStats snapshot after n_steps of the train_run
        loop (+ one evaluate_full_graph), in the layout of Ctx.comm_stats."""
        mc, md = cfg.arrays()
        d = np.asarray(dims, np.int32)
        out = np.zeros(28, np.uint64)
        self._check(self.L.ref_comm_stats(h, _ptr(d), _ptr(mc), _ptr(md), b, seed, n_steps, prec,
                                          int(evaluate), _ptr(out)))
        axes, phases = ("D", "X", "Y", "Z"), ("sampling", "forward", "backward", "dp_sync", "other")
        return {
            "bytes": {a: {p: int(out[i * 5 + j]) for j, p in enumerate(phases)} for i, a in enumerate(axes)},
            "allreduce_calls": {a: int(out[20 + i]) for i, a in enumerate(axes)},
            "allgather_calls": {a: int(out[24 + i]) for i, a in enumerate(axes)},
        }

    # layer operators on the one-rank grid (ref_shim.cpp, pmm.hpp:76-401)
    def contract(self, a: np.ndarray, b: np.ndarray, prec: int = 0) -> np.ndarray:
        a, b = np.ascontiguousarray(a, np.float32), np.ascontiguousarray(b, np.float32)
        c = np.empty((a.shape[0], b.shape[1]), np.float32)
        self._check(self.L.ref_contract(a.shape[0], a.shape[1], b.shape[1], _ptr(a), _ptr(b), prec, _ptr(c)))
        return c

    def spmm(self, a: Csr, f: np.ndarray, prec: int = 0) -> np.ndarray:
        f = np.ascontiguousarray(f, np.float32)
        h = np.empty((a.n_rows, f.shape[1]), np.float32)
        rp, ci = np.ascontiguousarray(a.row_ptr, np.int64), np.ascontiguousarray(a.col_idx, np.int64)
        va = np.ascontiguousarray(a.values, np.float64)
        self._check(self.L.ref_spmm(a.n_rows, a.n_cols, _ptr(rp), _ptr(ci), _ptr(va), _ptr(f), f.shape[1], prec,
                                    _ptr(h)))
        return h

    def rmsnorm(self, x, gamma, eps, dy=None):
        x, gamma = np.ascontiguousarray(x, np.float32), np.ascontiguousarray(gamma, np.float32)
        m, n = x.shape
        y, rms = np.empty_like(x), np.empty(m, np.float32)
        dx, dg = (np.empty_like(x), np.empty(n, np.float32)) if dy is not None else (None, None)
        dy = np.ascontiguousarray(dy, np.float32) if dy is not None else None
        self._check(self.L.ref_rmsnorm(m, n, _ptr(x), _ptr(gamma), eps, _ptr(dy), _ptr(y), _ptr(rms), _ptr(dx),
                                       _ptr(dg)))
        return y, rms, dx, dg

    def fused(self, x, h_prev, rate, key, training, dy=None):
        x = np.ascontiguousarray(x, np.float32)
        h = np.ascontiguousarray(h_prev, np.float32) if h_prev is not None else None
        out, scale = np.empty_like(x), np.empty_like(x)
        dx = np.empty_like(x) if dy is not None else None
        dy = np.ascontiguousarray(dy, np.float32) if dy is not None else None
        self._check(self.L.ref_fused(x.shape[0], x.shape[1], _ptr(x), _ptr(h), rate, key, int(training), _ptr(dy),
                                     _ptr(out), _ptr(scale), _ptr(dx)))
        return out, scale, dx

    def cross_entropy(self, logits, labels):
        logits = np.ascontiguousarray(logits, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        loss = np.zeros(1, np.float32)
        grad = np.empty_like(logits)
        self._check(self.L.ref_cross_entropy(logits.shape[0], logits.shape[1], _ptr(logits), _ptr(labels),
                                             _ptr(loss), _ptr(grad)))
        return float(loss[0]), grad

    def init_weights(self, cfg: ModelConfig, seed: int):
        mc, md = cfg.arrays()
        out = np.zeros(int(self.L.ref_param_total(_ptr(mc), _ptr(md))), np.float32)
        self._check(self.L.ref_init_weights(_ptr(mc), _ptr(md), seed, _ptr(out)))
        return unflatten(cfg, out)

    def bench(self, h, dims, cfg: ModelConfig, b, seed, warmup, steps, prec=0):
        mc, md = cfg.arrays()
        d = np.asarray(dims, np.int32)
        step_ms = np.zeros(steps)
        phase = np.zeros(5)
        self._check(self.L.ref_bench(h, _ptr(d), _ptr(mc), _ptr(md), b, seed, warmup, steps, prec,
                                     _ptr(step_ms), _ptr(phase)))
        return step_ms, phase


def unflatten(cfg: ModelConfig, flat: np.ndarray) -> list[np.ndarray]:
    out, off = [], 0
    for _, shp in cfg.param_shapes():
        k = int(np.prod(shp))
        out.append(flat[off:off + k].reshape(shp).copy())
        off += k
    return out
