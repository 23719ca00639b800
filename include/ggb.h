/* ggb.h — C ABI of libggb.so, the B200-native (sm_100a) mini-batch GCN
 * training step of ScaleGNN (arxiv 2604.02651).
 *
 * The reference boundary is the C++ API of /root/reference/proj (namespace
 * gridgnn; there is no FFI). Each entry point below replaces the reference
 * function cited beside it; the header-only C++ drop-in
 * paper_2604_02651_b200/cpp/gridgnn/ggb.hpp restores the reference's own
 * names, by-value results and exception types on top of it, and the Python
 * mirror paper_2604_02651_b200/gridgnn.py binds it through ctypes.
 *
 * Conventions: plain pointers and sizes only; every call returns a status
 * code and never throws; host arrays are caller-owned; device memory is owned
 * by the handles and freed by the matching *_destroy. A handle is used by one
 * host thread at a time (the prefetch producer owns its batches until it hands
 * them over, as the reference PrefetchQueue does, model.hpp:556-581).
 */
#ifndef GGB_H_
#define GGB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum ggb_status {
  GGB_OK = 0,
  GGB_EINVAL = 1,    /* -> std::invalid_argument (e.g. sampling.cpp:12-13) */
  GGB_ECONTRACT = 2, /* -> CommContract (comm.hpp:44-46, pmm.hpp:67-69)    */
  GGB_ETIMEOUT = 3,  /* -> CommTimeout (comm.hpp:41-43)                      */
  GGB_ECUDA = 4,     /* -> std::runtime_error                                */
  GGB_ENCCL = 5,     /* -> std::runtime_error                                */
  GGB_EINTERNAL = 9
};

/* comm.hpp:22 Precision: GGB_FP32 = kFp32; GGB_BF16_WIRE = kBf16Roundtrip
 * reproduced exactly (each contribution rounded to bf16, fp32 sum in axis
 * order: an all-gather of bf16); GGB_BF16_SUM = bf16 payloads summed by NCCL
 * (half the bytes of kFp32 with one ring all-reduce; rounding differs from
 * kBf16Roundtrip within the bf16-communication tolerance). */
enum ggb_precision { GGB_FP32 = 0, GGB_BF16_WIRE = 1, GGB_BF16_SUM = 2 };
enum ggb_optimizer { GGB_SGD = 0, GGB_ADAM = 1 };       /* model.hpp:45 Optimizer */

typedef struct ggb_ctx_s* ggb_ctx_t;     /* one per (process, GPU): grid coords, streams, comms, sampler */
typedef struct ggb_graph_s* ggb_graph_t;
typedef struct ggb_dataset_s* ggb_dataset_t; /* host Dataset (dataset.hpp:16-29) + its raw edge list */ /* Dataset + RankContext plane shards resident in HBM */
typedef struct ggb_batch_s* ggb_batch_t; /* StepBatch resident in HBM (model.hpp:238-246) */
typedef struct ggb_state_s* ggb_state_t; /* ModelState resident in HBM (model.hpp:87-105) */

/* ModelConfig (model.hpp:26-43) */
typedef struct {
  int32_t layers;
  int64_t d_in, d_h, d_out;
  double dropout_rate;
  int32_t use_rmsnorm, use_dropout, use_residual;
} ggb_model_config;

const char* ggb_last_error(void); /* thread-local message of the last failure */
int ggb_version(void);

/* ---- context: replaces Communicator/RankComm (comm.hpp:203-408) ------------
 * dims = {g_d, g_x, g_y, g_z}; rank numbering as DeviceGrid (grid.hpp:26-28).
 * nccl_uid (128 bytes from ggb_get_unique_id on rank 0, broadcast by the
 * caller) creates the world communicator and one split per axis. With
 * nccl_uid == NULL the context is "virtual": sampling and single-rank compute
 * work; any collective over a group larger than one fails GGB_ECONTRACT.
 * stream: the CUDA stream compute is launched on (NULL = library-owned). */
int ggb_get_unique_id(uint8_t out[128]);
/* number of visible CUDA devices (0 and GGB_ECUDA without a usable driver) */
int ggb_device_count(int32_t* out);
int ggb_ctx_create(const int32_t dims[4], int32_t rank, int32_t device, const uint8_t* nccl_uid,
                   void* stream, ggb_ctx_t* out);
int ggb_ctx_destroy(ggb_ctx_t ctx);
int ggb_ctx_set_stream(ggb_ctx_t ctx, void* stream);
int ggb_ctx_synchronize(ggb_ctx_t ctx);
/* CommConfig::timeout (comm.hpp:195-198, default 60 s; also GGB_COMM_TIMEOUT_MS):
 * a host wait on the context's stream (ggb_ctx_synchronize, the loss read of
 * ggb_train_step, barriers) polls the NCCL communicators' asynchronous errors
 * and this deadline; on either it aborts the communicators (their in-flight
 * kernels return) and fails with GGB_ENCCL / GGB_ETIMEOUT (CommTimeout:
 * "collective timed out: not all group members arrived", comm.hpp:157-158).
 * Later collectives on the context fail with GGB_ETIMEOUT. */
int ggb_ctx_set_comm_timeout(ggb_ctx_t ctx, int64_t timeout_ms);
/* counters = {kernels launched on ctx since creation, host->device bytes,
 * device->host bytes} */
int ggb_ctx_counters(ggb_ctx_t ctx, uint64_t* counters);
/* CommStats (reference comm.hpp:75-117, 385-403): the reference's accounting
 * of every logical collective of the step, charged at its call sites —
 * all-reduce: count * elem_bytes * (g-1)/g (elem_bytes 2 on the bf16 wires),
 * all-gather: the whole gathered payload, nothing in a singleton group.
 * out[GGB_COMM_STATS_LEN] = bytes[axis][phase] (axis D,X,Y,Z; phase sampling,
 * forward, backward, dp_sync, other; 20 entries), then all-reduce calls per
 * axis (4), then all-gather calls per axis (4). grid_total != 0 sums over
 * every rank of the grid (Communicator::snapshot; collective: every rank
 * calls it); reset != 0 zeroes this rank's counters after reading.
 * Phases: train_step's forward + loss (forward) and backward (backward),
 * dp_sync (dp_sync), anything else (other). */
#define GGB_COMM_STATS_LEN 28
int ggb_ctx_comm_stats(ggb_ctx_t ctx, int32_t grid_total, int32_t reset, uint64_t* out);
/* Per-kernel-class timing with CUDA events on the ctx stream. Classes:
 * 0 sampling, 1 SpMM fwd, 2 SpMM bwd, 3 GEMM fwd, 4 GEMM dX, 5 GEMM dW,
 * 6 other element-wise passes, 7 optimizer, 8 collectives, 9 fused
 * RMSNorm/ReLU/dropout/residual forward, 10 its backward, 11 cross-entropy.
 * read: totals since the last reset of time (ms), algorithmic bytes, flops
 * and launch counts (arrays of 12). */
int ggb_ctx_profile(ggb_ctx_t ctx, int32_t enable);
int ggb_ctx_profile_read(ggb_ctx_t ctx, double* ms, double* bytes, double* flops, int64_t* counts,
                         int32_t reset);

/* ---- sampler: sample_vertices (sampling.cpp:11-33) ------------------------- */
int ggb_sample_vertices(ggb_ctx_t ctx, int64_t n, int64_t b, uint64_t seed, uint64_t step,
                        int64_t* host_out);

/* ---- graph: Dataset (dataset.hpp:16-29) + make_rank_context (model.hpp:217-234)
 * Host CSR of D^-1/2(A+I)D^-1/2 (int64 row_ptr/col_idx, fp64 values). Uploads
 * this rank's static plane shards (make_csr_shard, shardsample.cpp:19-45) and
 * their transposes, the feature column slice and the labels. symmetric != 0
 * asserts A == A^T (always true for normalize_adjacency outputs,
 * dataset.cpp:47-83) and skips the host transpose. */
int ggb_graph_create(ggb_ctx_t ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                     const double* values, int32_t symmetric, int64_t d_in, const float* features,
                     int64_t n_classes, const int32_t* labels, int32_t layers, ggb_graph_t* out);
/* generate_synthetic (dataset.cpp:85-131) implemented natively (bit-identical
 * to the reference generator), then uploaded as ggb_graph_create does. */
int ggb_graph_generate_synthetic(ggb_ctx_t ctx, int64_t n, double avg_degree, int64_t d_in,
                                 int64_t n_classes, uint64_t seed, int32_t layers,
                                 ggb_graph_t* out);
/* The same dataset generated on the device: edges, the
 * normalized CSR, labels and split tags are bit-identical to
 * generate_synthetic (dataset.cpp:85-150); features follow the same polar
 * sequence with CUDA's fp64 log (a value may differ by one fp32 ulp in rare
 * cases). No host pass, so papers100M-scale graphs build in seconds. */
int ggb_graph_generate_synthetic_device(ggb_ctx_t ctx, int64_t n, double avg_degree, int64_t d_in,
                                        int64_t n_classes, uint64_t seed, int32_t layers,
                                        ggb_graph_t* out);
/* Host copies of a graph's dataset (tests): the full normalized CSR (needs
 * a full-matrix shard on this rank, i.e. a 1x1x1 grid), features (full
 * device copy only), labels, split; any pointer may be NULL. col_idx is
 * int64 like the reference's CsrMatrix. */
int ggb_graph_export(ggb_graph_t g, int64_t* row_ptr, int64_t* col_idx, double* values, float* features,
                     int32_t* labels, uint8_t* split);
/* ---- host datasets and files. No GPU needed except for
 * ggb_graph_from_dataset. Formats and validation messages are the
 * reference's (dataset.cpp:152-280): text edge list ("u v" per line, '#'
 * comments), SGNF (features), SGNL (labels), SGNS (split tags).
 * load_dataset (dataset.cpp:178-239); errors -> GGB_EINVAL with the
 * reference's message (std::invalid_argument there). */
int ggb_dataset_load(const char* edges, const char* features, const char* labels, const char* split,
                     ggb_dataset_t* out);
/* generate_synthetic + synthetic_edges (dataset.cpp:85-150), host native. */
int ggb_dataset_generate_synthetic(int64_t n, double avg_degree, int64_t d_in, int64_t n_classes,
                                   uint64_t seed, ggb_dataset_t* out);
/* R-MAT input (BASELINE configs[0]; new code — the reference has only its ER
 * generator, dataset.cpp:133-150): m edge draws over 2^scale vertices with
 * Graph500 quadrant probabilities (a, b, c, 1-a-b-c), generated on the GPU
 * (counter-based, one thread per edge). ggb_rmat_edges returns the raw list
 * (host_uv = 2 x m); ggb_dataset_generate_rmat builds the dataset from it as
 * generate_synthetic does from its ER list (normalize_adjacency,
 * dataset.cpp:47-83; features, degree-quantile labels and split from seed),
 * so ggb_dataset_save + the reference's load_dataset reproduce it. */
int ggb_rmat_edges(ggb_ctx_t ctx, int32_t scale, int64_t m, double a, double b, double c, uint64_t seed,
                   int64_t* host_uv);
int ggb_dataset_generate_rmat(ggb_ctx_t ctx, int32_t scale, int64_t m, double a, double b, double c,
                              int64_t d_in, int64_t n_classes, uint64_t seed, ggb_dataset_t* out);
/* info = {n, nnz, d_in, n_classes, raw_edges} (5 entries) */
int ggb_dataset_info(ggb_dataset_t d, int64_t* info);
/* any pointer may be NULL; col_idx int64 (CsrMatrix), edges_uv = 2 x raw_edges */
int ggb_dataset_export(ggb_dataset_t d, int64_t* row_ptr, int64_t* col_idx, double* values, float* features,
                       int32_t* labels, uint8_t* split, int64_t* edges_uv);
/* save_edge_list / save_features / save_labels / save_split (dataset.cpp:241-280),
 * byte-identical to the reference's CLI `gen` output (gridgnn_main.cpp:313-324);
 * a NULL path skips that file. */
int ggb_dataset_save(ggb_dataset_t d, const char* edges, const char* features, const char* labels,
                     const char* split);
/* ggb_graph_create + ggb_graph_set_split from a host dataset (make_rank_context). */
int ggb_graph_from_dataset(ggb_ctx_t ctx, ggb_dataset_t d, int32_t layers, ggb_graph_t* out);
int ggb_dataset_destroy(ggb_dataset_t d);

/* Split tags (Dataset::split, dataset.hpp:12,23): 0 train, 1 val, 2 test,
 * 3 unused; one byte per vertex. generate_synthetic sets them itself
 * (dataset.cpp:122-129); needed only by ggb_evaluate_full_graph. */
int ggb_graph_set_split(ggb_graph_t g, const uint8_t* split);
int ggb_graph_destroy(ggb_graph_t g);
/* Keep the feature slice in host memory instead of HBM, as the reference's
 * Dataset does (build_step_batch reads ds.features rows per step,
 * model.hpp:293-303): the slice moves to mapped pinned host memory and every
 * batch build gathers its x_in rows over PCIe (zero-copy loads on the
 * sampling stream; counted in the context's h2d bytes). Not reversible. */
int ggb_graph_features_to_host(ggb_graph_t g);
/* info = {n, nnz, d_in, n_classes, distinct_plane_shards, device_bytes, features_on_host}
 * (7 entries) */
int ggb_graph_info(ggb_graph_t g, int64_t* info);

/* ---- batches: build_step_batch (model.hpp:250-309) / build_local_minibatch
 * (shardsample.cpp:124-156). Communication-free. The batch handle is reused
 * (grow-only buffers) when passed back in *inout; NULL creates one. */
int ggb_build_step_batch(ggb_ctx_t ctx, ggb_graph_t g, int64_t b, uint64_t group_seed,
                         uint64_t step, ggb_batch_t* inout);
int ggb_batch_destroy(ggb_batch_t batch);
/* Sampling/training overlap: the train_run prefetch producer and its queue
 * (model.hpp:556-581, 631-656). A native producer thread builds the batches
 * of steps first_step, first_step+1, ... on its own CUDA stream into two
 * slots; next() hands out the batch of the following step, ordering the
 * ctx stream after it with a CUDA event and releasing the previous batch once
 * the ctx stream's work on it completes. Handed-out batches are owned by the
 * prefetcher (do not destroy them); they are bit-identical to
 * ggb_build_step_batch's. With layers > 0 and dropout_rate > 0 the producer
 * also evaluates each layer's dropout keep-bits for the step ahead
 * (element_unit(dropout_key(run_seed, dp, step, l), row, col) >= rate,
 * pmm.hpp:317-322, model.hpp:164-171), taking the integer hashing off the
 * training stream; the forward uses them when its keys match. */
typedef struct ggb_prefetch_s* ggb_prefetch_t;
int ggb_prefetch_create(ggb_ctx_t ctx, ggb_graph_t g, int64_t b, uint64_t group_seed, uint64_t first_step,
                        uint64_t run_seed, int32_t layers, int64_t d_h, double dropout_rate,
                        ggb_prefetch_t* out);
int ggb_prefetch_next(ggb_prefetch_t pf, ggb_batch_t* batch_out);
int ggb_prefetch_destroy(ggb_prefetch_t pf);
/* info = {b, n, planes, x_r0, x_r1, x_c0, x_c1, nnz_extracted, nnz_kept} */
int ggb_batch_info(ggb_batch_t batch, int64_t* info);
int ggb_batch_sample(ggb_batch_t batch, int64_t* host_out);
/* batch_off for axis in {1,2,3}: dims[axis]+1 offsets */
int ggb_batch_offsets(ggb_batch_t batch, int32_t axis, int64_t* host_out);
/* dims = {n_rows, n_cols, nnz, r0, r1, c0, c1}; arrays may be NULL (query) */
int ggb_batch_plane(ggb_batch_t batch, int32_t plane, int32_t transposed, int64_t* dims,
                    int64_t* row_ptr, int64_t* col_idx, double* values);
/* x_in block (x_r1-x_r0) x (x_c1-x_c0) as exact fp32 copies of the features */
int ggb_batch_x_in(ggb_batch_t batch, float* host_out);
int ggb_batch_labels(ggb_batch_t batch, int32_t* host_out);

/* ---- model state: init_state (model.hpp:175-208) ------------------------------ */
int ggb_state_create(ggb_ctx_t ctx, const ggb_model_config* cfg, uint64_t seed, ggb_state_t* out);
int ggb_state_destroy(ggb_state_t st);
/* Forward compute precision (not in the reference, whose compute is fp32):
 * GGB_COMPUTE_ACCURATE (default) keeps forward activations fp32 (fp32 SpMM
 * gathers, split-bf16 tensor-core GEMMs) so ReLU/dropout decisions match the
 * fp32 reference; GGB_COMPUTE_FAST uses bf16 operands throughout. The
 * backward pass uses bf16 operands with fp32 accumulation in both. */
enum ggb_compute { GGB_COMPUTE_ACCURATE = 0, GGB_COMPUTE_FAST = 1 };
int ggb_state_set_compute(ggb_state_t st, int32_t mode);
/* parameter views in param_views order (model.hpp:107-133): win, [w_l, gamma_l]*L, wout */
int ggb_state_num_params(ggb_state_t st);
/* info = {global_rows, global_cols, r0, r1, c0, c1}; a gamma has rows = 1 */
int ggb_state_param_info(ggb_state_t st, int32_t idx, int64_t* info);
/* which: 0 weight, 1 grad, 2 adam m, 3 adam v; local block, row-major */
int ggb_state_param_get(ggb_state_t st, int32_t idx, int32_t which, float* host_out);
int ggb_state_param_set(ggb_state_t st, int32_t idx, int32_t which, const float* host_in);

/* ---- training: train_step / forward / dp_sync / optimizer_step (model.hpp:335-478) */
/* forward + cross-entropy + backward; grads left un-synced. loss_out (host,
 * nullable: NULL keeps the call asynchronous and the loss on the device). */
int ggb_train_step(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t batch, int32_t precision,
                   uint64_t run_seed, uint64_t global_step, double rmsnorm_eps, float* loss_out);
/* device-side loss of the last train_step (one float) */
int ggb_last_loss_device(ggb_state_t st, const float** dev_ptr);
/* Enqueues the device->host copy of the last train_step's loss into host_dst
 * (pinned host memory for a truly asynchronous copy) on the ctx stream and
 * returns without waiting: the caller reads it after a later wait (a training
 * loop that logs step t's loss while step t+1 runs). */
int ggb_loss_to_host_async(ggb_ctx_t ctx, ggb_state_t st, float* host_dst);
/* logits block of the last forward: dims = {r0, r1, c0, c1}; out may be NULL */
int ggb_state_logits(ggb_state_t st, int64_t* dims, float* host_out);
int ggb_forward(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t batch, int32_t precision,
                int32_t training, uint64_t run_seed, uint64_t global_step, double rmsnorm_eps);
/* evaluate_full_graph (model.hpp:493-537): forward over the eval batch (built
 * with b = n, seed, step 0 as train_run does, model.hpp:625) with dropout off,
 * argmax per vertex (ties to the lowest class id), per-split counts summed
 * over the grid. counts = {correct train, val, test, total train, val, test}
 * (EvalCounts, model.hpp:480-490), identical on every rank. */
int ggb_evaluate_full_graph(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t eval_batch, ggb_graph_t g,
                            int32_t precision, double rmsnorm_eps, uint64_t* counts);
int ggb_dp_sync(ggb_ctx_t ctx, ggb_state_t st);
int ggb_optimizer_step(ggb_ctx_t ctx, ggb_state_t st, int32_t optimizer, double lr);

/* ---- layer operators (include/gridgnn/pmm.hpp:76-401) --------------------------
 * A ggb_block is one rank's block of a 2D-sharded fp32 matrix: the metadata of
 * the reference's ShardedTensor (tensor.hpp:75-86) with the block in HBM.
 * Layout = (row_axis, col_axis), distinct PMM axes (1 = X, 2 = Y, 3 = Z);
 * row_off / col_off are HOST arrays of dims[row_axis] + 1 / dims[col_axis] + 1
 * partition offsets into [0, g_rows] / [0, g_cols] (explicit, as the batch
 * rows are split where the sorted sample meets the vertex partition); this
 * rank's block is rows [row_off[x_r], row_off[x_r + 1]) x cols
 * [col_off[x_c], col_off[x_c + 1]) with x_r, x_c its grid coordinates, stored
 * row-major at `data` with leading dimension `ld` (elements). Outputs are
 * caller-allocated blocks whose metadata must equal the result's (CommContract
 * otherwise). Collectives run on the context's NCCL axis communicators; every
 * member of a group calls with matching shapes, as in the reference. */
typedef struct {
  int32_t row_axis, col_axis;
  int64_t g_rows, g_cols;
  const int64_t* row_off;
  const int64_t* col_off;
  float* data;
  int64_t ld;
} ggb_block;
/* A ShardedSparse (tensor.hpp:88-96): the block as CSR in HBM with LOCAL
 * column ids (int64 row_ptr, int32 col, fp32 values = (float) of the fp64
 * reference values, pmm.hpp:160). */
typedef struct {
  int32_t row_axis, col_axis;
  int64_t g_rows, g_cols;
  const int64_t* row_off;
  const int64_t* col_off;
  const int64_t* row_ptr;
  const int32_t* col;
  const float* val;
} ggb_csr_block;
/* contract (pmm.hpp:97-130): c = a . b, all-reduce along a.col_axis with the
 * precision's wire; a (r, k), b (k, t) -> c (r, t). Split-bf16 tcgen05 GEMM
 * (fp32-accurate to ~2^-16). */
int ggb_contract(ggb_ctx_t ctx, const ggb_block* a, const ggb_block* b, const ggb_block* c, int32_t precision);
/* spmm (pmm.hpp:134-167): h = a . f, all-reduce along a.col_axis. */
int ggb_spmm(ggb_ctx_t ctx, const ggb_csr_block* a, const ggb_block* f, const ggb_block* h, int32_t precision);
/* transposed (pmm.hpp:76-92): out is the transposed shard's block (layout and offsets swapped). */
int ggb_transposed(ggb_ctx_t ctx, const ggb_block* t, const ggb_block* out);
/* gather_full (pmm.hpp:171-195): the whole g_rows x g_cols matrix (row-major,
 * leading dimension ld_full) on every rank of the DP group. */
int ggb_gather_full(ggb_ctx_t ctx, const ggb_block* t, float* full, int64_t ld_full);
/* reshard (pmm.hpp:197-204) to dst's layout / offsets, as a point-to-point
 * block permutation (the reference all-gathers the whole matrix). */
int ggb_reshard(ggb_ctx_t ctx, const ggb_block* src, const ggb_block* dst);
/* parallel_rmsnorm_fwd (pmm.hpp:214-243): y = gamma . x / rms, rms over the
 * full g_cols (fp32 all-reduce of the row sums of squares along x.col_axis);
 * gamma = this rank's column slice (device), rms = one per local row (device). */
int ggb_rmsnorm_fwd(ggb_ctx_t ctx, const ggb_block* x, const float* gamma, double eps, const ggb_block* y,
                    float* rms);
/* parallel_rmsnorm_bwd (pmm.hpp:251-287): dx and the column slice of dgamma
 * (all-reduced along x.row_axis), device pointers. */
int ggb_rmsnorm_bwd(ggb_ctx_t ctx, const ggb_block* x, const float* gamma, const float* rms, const ggb_block* dy,
                    const ggb_block* dx, float* dgamma);
/* fused_elementwise_fwd (pmm.hpp:299-328): out = x . scale + h_prev (nullable),
 * scale = (x > 0) . (training && rate > 0 ? [element_unit(key, row, col) >= rate] / (1 - rate) : 1);
 * keep_bits (device, nullable) receives scale != 0 as ggb_mask_words(cols)
 * words per row (the row kernels' layout) instead of the fp32 scale matrix. */
int ggb_fused_elementwise_fwd(ggb_ctx_t ctx, const ggb_block* x, const ggb_block* h_prev, double rate,
                              uint64_t mask_key, int32_t training, const ggb_block* out, uint32_t* keep_bits);
/* fused_elementwise_bwd (pmm.hpp:331-341): dx = dy . scale from those bits,
 * scale = keep_scale where a bit is set (keep_scale = (float)(1 / (1 - rate))
 * when the forward dropped, else 1), 0 elsewhere. */
int ggb_fused_elementwise_bwd(ggb_ctx_t ctx, const ggb_block* dy, const uint32_t* keep_bits, float keep_scale,
                              const ggb_block* dx);
/* keep-bit words per row of a block with `cols` local columns */
int64_t ggb_mask_words(int64_t cols);
/* parallel_cross_entropy (pmm.hpp:352-401): loss (device float, replicated),
 * grad = (softmax - onehot) / g_rows; labels = the global batch's labels (device int32). */
int ggb_cross_entropy(ggb_ctx_t ctx, const ggb_block* logits, const int32_t* labels, float* loss,
                      const ggb_block* grad);
/* A batch plane's CSR block as a ggb_csr_block (pointers stay valid while the batch lives). */
int ggb_batch_csr_block(ggb_batch_t batch, int32_t plane, int32_t transposed, ggb_csr_block* out);
/* train_step split at the reference's seams (model.hpp:459-478): ggb_forward
 * (above), then ggb_loss = parallel_cross_entropy on its logits (the gradient
 * stays in the state), then ggb_backward (model.hpp:378-420). */
int ggb_loss(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t batch, float* loss_out);
int ggb_backward(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t batch, int32_t precision);

/* device memory for host-side callers of the layer operators (the C++
 * drop-in headers cpp/gridgnn/tensor.hpp / pmm.hpp stage ShardedTensor blocks
 * through these; copies run on the context's stream and complete on return) */
int ggb_device_alloc(ggb_ctx_t ctx, size_t bytes, void** out);
int ggb_device_free(ggb_ctx_t ctx, void* p);
int ggb_memcpy_h2d(ggb_ctx_t ctx, void* dst, const void* src, size_t bytes);
int ggb_memcpy_d2h(ggb_ctx_t ctx, void* dst, const void* src, size_t bytes);

/* ---- kernels exposed for unit tests (device pointers, row-major) ------------- */
/* sample_vertices with an extra, test-only rejection rule (a draw x is also
 * rejected when x % reject_mod == 0): rejections of next_below (rng.hpp:38-45)
 * otherwise occur with probability < n / 2^64 per draw, too rarely to test the
 * parallel re-draw passes; the oracle applies the same rule. */
int ggb_sample_vertices_test_reject(ggb_ctx_t ctx, int64_t n, int64_t b, uint64_t seed, uint64_t step,
                                    uint64_t reject_mod, int64_t* host_out);
/* C[m x n] = A[m x k] . Bt[n x k]^T in bf16 x bf16 -> fp32 on tcgen05.
 * c (fp32) and/or c_bf16 may be NULL. Leading dimensions in elements. */
int ggb_gemm_bf16(ggb_ctx_t ctx, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda,
                  const void* bt, int64_t ldb, float* c, int64_t ldc, void* c_bf16, int64_t ldcb);
/* Split-bf16: fp32 operands as (hi, lo) bf16 pairs, C = (Ah+Al).(Bh+Bl)^T
 * minus the Al.Bl term, 3 tcgen05 MMAs per k-step, fp32 accumulate. */
int ggb_gemm_split_bf16(ggb_ctx_t ctx, int64_t m, int64_t n, int64_t k, const void* a_hi, const void* a_lo,
                        int64_t lda, const void* bt_hi, const void* bt_lo, int64_t ldb, float* c, int64_t ldc);
/* DW[kw x nw] = X[m x kw]^T . DY[m x nw] (contraction over the m rows). */
int ggb_gemm_wgrad_bf16(ggb_ctx_t ctx, int64_t m, int64_t kw, int64_t nw, const void* x,
                        int64_t ldx, const void* dy, int64_t lddy, float* dw, int64_t lddw);
/* H[rows x f] = A . F with A in CSR (int64 row_ptr, int32 col, fp32 val) and
 * F bf16; out fp32 (out) and/or bf16 (out_bf16); accumulate != 0 adds into out. */
int ggb_spmm_csr(ggb_ctx_t ctx, int64_t rows, const int64_t* row_ptr, const int32_t* col,
                 const float* val, const void* f, int64_t ldf, int64_t fcols, float* out,
                 int64_t ldo, void* out_bf16, int64_t ldob, int32_t accumulate);
/* Same with fp32 F (the accurate forward's gathers; pmm.hpp:160 casts the fp64
 * value to Real and accumulates in Real): out fp32 and/or the bf16 (hi, lo)
 * split pair of the fp32 result (out_hi, out_lo may be NULL). */
int ggb_spmm_csr_f32(ggb_ctx_t ctx, int64_t rows, const int64_t* row_ptr, const int32_t* col,
                     const float* val, const float* f, int64_t ldf, int64_t fcols, float* out,
                     int64_t ldo, void* out_hi, void* out_lo, int64_t ldob, int32_t accumulate);

#ifdef __cplusplus
}
#endif
#endif /* GGB_H_ */
