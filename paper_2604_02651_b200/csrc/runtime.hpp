// Host-side runtime objects behind the opaque ggb_* handles.
#pragma once

#include <array>
#include <cstddef>
#include <memory>
#include <vector>

#include "common.hpp"

namespace ggb {

struct Comm;  // comm.cu (NCCL per-axis communicators)
struct Prof;  // prof.hpp (per-kernel-class event timing)

/// CommStats accounting (comm.hpp:24-25, 75-117, 385-403): every logical
/// collective of the reference's step is charged to (axis, phase) with the
/// reference's model: an all-reduce charges count * elem_bytes * (g-1)/g, an
/// all-gather the whole gathered payload, nothing in a singleton group; call
/// counters always advance. Charged at the reference's call sites whether or
/// not this implementation moves those bytes (it fuses, skips or replaces some
/// of them), so the byte columns of the metrics match the reference's.
enum Phase : int { kPhaseSampling = 0, kPhaseForward = 1, kPhaseBackward = 2, kPhaseDpSync = 3, kPhaseOther = 4 };
constexpr int kNumPhases = 5;
struct CommStats {
  uint64_t bytes[4][kNumPhases] = {};
  uint64_t allreduce_calls[4] = {};
  uint64_t allgather_calls[4] = {};
};

/// Sampler scratch, reused across steps (one build at a time per context).
struct SamplerWork {
  DevBuf head;      // uint64 [n]: step-tagged (tag<<32 | step index) list heads
  int64_t head_n = 0;
  uint32_t tag = 0;
  DevBuf j, next;   // int32 [b]
  DevBuf flag;      // int32 rejection flag
  DevBuf bitmap;    // uint32 [n/32 + 2]
  DevBuf wcount;    // int32 [words]
  DevBuf wpfx;      // int32 [words + 1]: sampled ids below each word
  DevBuf scan_tmp;  // scan partials
  DevBuf cnt;       // int32 per-row kept counts
  DevBuf dev_misc;  // small device scalars (offsets, totals, counters)
  PinnedBuf host_misc;
  // second stream of the build: the PCIe gather of host-resident features
  // runs on it beside the shard extraction (created on first use, same
  // priority as the build's stream)
  struct Aux {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    Aux() = default;
    Aux(const Aux&) = delete;
    Aux& operator=(const Aux&) = delete;
    ~Aux() {
      if (s) cudaStreamDestroy(s);
      if (fork) cudaEventDestroy(fork);
      if (join) cudaEventDestroy(join);
    }
  } aux;
};

struct Ctx {
  Grid grid;
  int rank = 0;
  int coord[4] = {0, 0, 0, 0};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::unique_ptr<Comm> comm;
  SamplerWork sw;
  uint64_t launches = 0;              // kernels this library launched
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic of the step path
  int num_sms = 148;
  // side-stream context (the prefetcher): launch short non-persistent grids,
  // so compute-stream persistent kernels (one CTA per SM) are not held back
  bool side_stream = false;
  // SMs left free by the persistent kernels (SpMM pipe, GEMM) while a
  // collective runs beside them on the communication stream
  int sm_reserve = 0;
  int persistent_sms() const { return num_sms - sm_reserve > 0 ? num_sms - sm_reserve : 1; }
  std::unique_ptr<Prof> prof;
  DevBuf spmm_carry;  // per-warp partial rows of the pipelined SpMM's shared rows
  // the next SpMMs' CSR has power-law rows (the pipelined kernel then shares
  // long rows across warps); set per call site from BatchCsr::long_rows
  bool spmm_long_rows = false;
  // push-mode peer reductions: the SpMM producers also store every output
  // element at (its address + out_mirror) — the same slot area in the
  // peer's buffer (peer.cu); 0 = no mirror. Set per call site (MirrorScope).
  ptrdiff_t out_mirror = 0;
  CommStats stats;
  int phase = kPhaseOther;
  ~Ctx();
};

/// Marks the SpMMs of a scope as running over a power-law CSR block.
struct LongRowsScope {
  Ctx& ctx;
  bool prev;
  LongRowsScope(Ctx& c, bool v) : ctx(c), prev(c.spmm_long_rows) { ctx.spmm_long_rows = v; }
  ~LongRowsScope() { ctx.spmm_long_rows = prev; }
  LongRowsScope(const LongRowsScope&) = delete;
  LongRowsScope& operator=(const LongRowsScope&) = delete;
};

struct MirrorScope {
  Ctx& ctx;
  ptrdiff_t prev;
  MirrorScope(Ctx& c, ptrdiff_t d) : ctx(c), prev(c.out_mirror) { ctx.out_mirror = d; }
  ~MirrorScope() { ctx.out_mirror = prev; }
  MirrorScope(const MirrorScope&) = delete;
  MirrorScope& operator=(const MirrorScope&) = delete;
};

/// PhaseScope (comm.hpp:411-421).
struct PhaseScope {
  Ctx& ctx;
  int prev;
  PhaseScope(Ctx& c, int p) : ctx(c), prev(c.phase) { ctx.phase = p; }
  ~PhaseScope() { ctx.phase = prev; }
  PhaseScope(const PhaseScope&) = delete;
  PhaseScope& operator=(const PhaseScope&) = delete;
};

inline void charge_all_reduce(Ctx& ctx, int axis, int64_t count, int ebytes) {
  const uint64_t g = static_cast<uint64_t>(ctx.grid.dims[axis]);
  if (g > 1) ctx.stats.bytes[axis][ctx.phase] += static_cast<uint64_t>(count) * static_cast<uint64_t>(ebytes) * (g - 1) / g;
  ctx.stats.allreduce_calls[axis] += 1;
}
inline void charge_all_gather(Ctx& ctx, int axis, uint64_t payload_bytes) {
  if (ctx.grid.dims[axis] > 1) ctx.stats.bytes[axis][ctx.phase] += payload_bytes;
  ctx.stats.allgather_calls[axis] += 1;
}

/// One static plane shard (shardsample.hpp:18-25): rows [r0,r1) with local
/// row ids, global column ids restricted to [c0,c1).
struct PlaneShard {
  int64_t r0 = 0, r1 = 0, c0 = 0, c1 = 0, nnz = 0;
  DevBuf row_ptr;  // int64 [r1-r0+1]
  DevBuf col;      // int32 [nnz]
  DevBuf val;      // double [nnz]
  // rows per degree (host, built with the graph): the n largest row degrees
  // bound the entries a batch block of n sampled rows can extract
  std::vector<int64_t> rows_of_degree;
  bool power_law() const {
    const int64_t rows = r1 - r0, dmax = static_cast<int64_t>(rows_of_degree.size()) - 1;
    return rows > 0 && dmax > 8 * (nnz / rows + 1);
  }
  int64_t top_rows_nnz(int64_t rows) const {
    int64_t sum = 0;
    for (int64_t d = static_cast<int64_t>(rows_of_degree.size()) - 1; d > 0 && rows > 0; --d) {
      const int64_t k = std::min(rows, rows_of_degree[static_cast<size_t>(d)]);
      sum += k * d;
      rows -= k;
    }
    return sum;
  }
};

struct Graph {
  Ctx* ctx = nullptr;
  int64_t n = 0, nnz = 0, d_in = 0, n_classes = 0;
  int layers = 0;
  int planes = 0;  // min(layers, 3)
  // plane p -> index into shards for the static shard and its transpose
  std::vector<int> fwd_of, tr_of;
  std::vector<PlaneShard> shards;
  int64_t feat_c0 = 0, feat_c1 = 0;  // Z-slice of the feature columns held here
  DevBuf features;                   // fp32 [n][feat_c1-feat_c0] in HBM, or empty when host-resident
  PinnedBuf features_host;           // the same slice in mapped pinned host memory (ggb_graph_features_to_host)
  const float* feat_ptr = nullptr;   // device-accessible feature rows (HBM or the host mapping)
  bool features_on_host() const { return features_host.p != nullptr; }
  DevBuf labels;                     // int32 [n]
  DevBuf split;                      // uint8 [n] SplitTag (dataset.hpp:12), for evaluation
  // value-free shards (no fp64 value arrays): values recomputed from the
  // full-graph row degrees, 1 / sqrt(deg_u deg_v) in IEEE fp64 (dataset.cpp:78-79)
  bool value_free = false;
  DevBuf degree;                     // int32 [n] when value_free
  size_t device_bytes = 0;
};

/// One rank's CSR block of a rescaled batch adjacency (ShardedSparse,
/// tensor.hpp:88-96) with device arrays for the kernels.
struct BatchCsr {
  int64_t n_rows = 0, n_cols = 0;
  bool long_rows = false;  // cut from a power-law shard (max degree > 8x mean)
  mutable int64_t nnz = 0;  // host copy, valid once the batch's totals are settled
  int64_t r0 = 0, r1 = 0, c0 = 0, c1 = 0;  // global batch coordinates
  DevBuf row_ptr;  // int64 [n_rows+1]
  DevBuf col;      // int32
  DevBuf val;      // float (SpMM operand, = (float)val64 as pmm.hpp:160)
  DevBuf val64;    // double (exact reference values, for export)
};

/// Precomputed dropout keep-bits of one layer's output block (row-kernel
/// layout, ops.hpp kRowChunk): element_unit(key, r0+i, c0+j) >= rate.
struct DropMask {
  uint64_t key = 0, thresh = 0;
  int64_t r0 = 0, c0 = 0, rows = -1, cols = -1, ldm = 0;
  DevBuf bits;  // uint32 [rows][ldm]
};

struct Batch {
  Ctx* ctx = nullptr;
  std::vector<DropMask> masks;  // per layer, filled by the prefetcher
  int64_t b = 0, n = 0;
  int planes = 0;
  DevBuf sample;  // int64 [b], strictly increasing
  std::array<std::vector<int64_t>, 4> batch_off;
  std::vector<int> csr_of;   // plane -> index in csrs (forward block)
  std::vector<int> csrt_of;  // plane -> index in csrs (transposed block)
  std::vector<BatchCsr> csrs;
  int nblocks = 0;  // csrs in use (csrs only grows)
  int64_t x_r0 = 0, x_r1 = 0, x_c0 = 0, x_c1 = 0, x_ld = 0;
  DevBuf x_in;    // bf16 [x_r1-x_r0][x_ld], zero padded (hi of the split pair)
  DevBuf x_in_lo; // bf16 lo residual: x == hi + lo to ~2^-16
  DevBuf labels;  // int32 [b]
  // first-layer pre-aggregation P = A_0 . x_in (sampler.cu preaggregate): fp32
  // x_in rows, P as split bf16 [A_0 rows][x_ld]; a cache of the batch, hence mutable
  mutable DevBuf x_f, p_in, p_in_lo;
  mutable bool p_ready = false, x_f_ready = false;
  // host view of the build's device totals (per block nnz, per block
  // extracted count): copied to pinned memory as the build is enqueued and
  // settled (settle_totals) on first host use, so the build never waits
  mutable uint64_t nnz_extracted = 0, nnz_kept = 0;
  PinnedBuf totals;
  EventHandle totals_ready;
  mutable bool totals_pending = false;
  uint64_t h2d_bytes = 0;  // feature bytes this build read over PCIe (host-resident features)
  const Graph* graph = nullptr;
};

// sampler.cu
// reject_mod: test-only extra rejection rule (0 = the reference's sampler)
void sample_set(Ctx& ctx, int64_t n, int64_t b, uint64_t seed, uint64_t step, int64_t* d_sample,
                uint64_t reject_mod = 0);
// want_xf: also keep the fp32 x_in rows for preaggregate() (same gather)
void build_step_batch(Ctx& ctx, const Graph& g, int64_t b, uint64_t group_seed, uint64_t step,
                      Batch& out, bool want_xf = false);
void gather_x_in_fp32(Ctx& ctx, const Batch& bt, float* d_out);
/// Fill the host nnz / extraction counters of a batch (waits for its build).
void settle_totals(const Batch& bt);
/// Degree histogram of a static shard (one download of its row pointers).
void shard_degree_profile(Ctx& ctx, PlaneShard& sh);
bool preagg_eligible(const Ctx& ctx, const Batch& bt);
void preaggregate(Ctx& ctx, const Batch& bt);

// scan.cu: out[0..n] = exclusive prefix sums of in[0..n), out[n] = total.
void exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, DevBuf& tmp,
                               cudaStream_t s);
void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, DevBuf& tmp, cudaStream_t s);

}  // namespace ggb
