// Full-graph evaluation (evaluate_full_graph, model.hpp:493-537): one forward
// of the trained model over the eval batch (b = N: every vertex, p = 1, so
// the plane blocks are the graph's own shards) with dropout off, then argmax
// accuracy per split tag.
//
//   argmax  : warp per logits row, strict '>' from the lowest float so ties
//             resolve to the lowest class id and NaN never wins (model.hpp:502-508)
//   classes : when the class axis is split, the (best value, class id) pairs of
//             the axis members are gathered and combined in axis order with the
//             same strict '>' (model.hpp:509-521)
//   counts  : per-split correct / total, summed over the logits row axis
//             (model.hpp:522-536)
#include <cfloat>

#include "comm.hpp"
#include "trainer.hpp"

namespace ggb {
namespace {

constexpr int kT = 256;

__global__ void __launch_bounds__(kT) k_row_argmax(const float* __restrict__ lg, int64_t rows, int64_t cols,
                                                   int64_t ld, int64_t c0, int64_t g_cols, float2* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (kT / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  float bv = -FLT_MAX;
  int64_t bi = g_cols;
  for (int64_t j = lane; j < cols; j += 32) {
    const float v = lg[r * ld + j];
    if (v > bv) {  // lane-local scan is in ascending column order
      bv = v;
      bi = c0 + j;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    // the serial scan keeps the first strict maximum: larger value wins, equal
    // values (both candidates, not NaN) go to the lower class id
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) out[r] = make_float2(bv, __int_as_float(static_cast<int>(bi)));
}

__global__ void __launch_bounds__(kT) k_eval_count(const float2* __restrict__ parts, int n_parts, int64_t rows,
                                                   int64_t r0, const int64_t* __restrict__ sample,
                                                   const int32_t* __restrict__ labels,
                                                   const uint8_t* __restrict__ split, int64_t g_cols,
                                                   unsigned long long* __restrict__ counts) {
  __shared__ unsigned int part[6];
  if (threadIdx.x < 6) part[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
  if (i < rows) {
    float best = -FLT_MAX;
    int64_t pred = g_cols;
    for (int p = 0; p < n_parts; ++p) {
      const float2 e = parts[static_cast<int64_t>(p) * rows + i];
      if (e.x > best) {
        best = e.x;
        pred = __float_as_int(e.y);
      }
    }
    const int64_t v = sample[r0 + i];
    const int tag = split[v];
    if (tag < 3) {
      atomicAdd(&part[3 + tag], 1u);
      if (pred == labels[v]) atomicAdd(&part[tag], 1u);
    }
  }
  __syncthreads();
  if (threadIdx.x < 6 && part[threadIdx.x]) atomicAdd(&counts[threadIdx.x], part[threadIdx.x]);
}

}  // namespace

void evaluate_full_graph(State& st, const Batch& eval, const Graph& g, int precision, double eps,
                         uint64_t counts_out[6]) {
  Ctx& ctx = *st.ctx;
  require(eval.graph == &g, "evaluate_full_graph: the eval batch was built from another graph");
  require(eval.b == g.n, "evaluate_full_graph: the eval batch must hold every vertex (b == n)");
  require(g.split.bytes >= static_cast<size_t>(g.n), "evaluate_full_graph: the graph has no split tags");
  forward(st, eval, precision, false, 0, 0, eps);
  const Block& lb = st.logits_blk;
  const int64_t rows = lb.rows();
  const int col_axis = lb.lay.col, row_axis = lb.lay.row;
  const int parts = ctx.grid.dims[col_axis];
  // the reference gathers (value, index) as two all-gathers (fp32, int64) and
  // all-reduces six u64 counters (model.hpp:508-509, 533)
  charge_all_gather(ctx, col_axis, static_cast<uint64_t>(rows) * parts * 4);
  charge_all_gather(ctx, col_axis, static_cast<uint64_t>(rows) * parts * 8);
  charge_all_reduce(ctx, row_axis, 6, 8);
  DevBuf& wk = st.tmp;
  // [best pairs: rows] [gathered: parts x rows] [counts: 6 u64]
  const size_t pair_bytes = static_cast<size_t>(rows) * sizeof(float2);
  const size_t need = pair_bytes * (1 + parts) + 64;
  uint8_t* base = static_cast<uint8_t*>(wk.reserve(need));
  float2* mine = reinterpret_cast<float2*>(base);
  float2* all = parts > 1 ? mine + rows : mine;
  auto* counts = reinterpret_cast<unsigned long long*>(base + pair_bytes * (1 + parts));
  GGB_CUDA(cudaMemsetAsync(counts, 0, 6 * sizeof(unsigned long long), ctx.stream));
  if (rows > 0) {
    k_row_argmax<<<static_cast<unsigned>((rows + kT / 32 - 1) / (kT / 32)), kT, 0, ctx.stream>>>(
        st.logits.as<float>(), rows, lb.cols(), lb.cols(), lb.c0, lb.g_cols, mine);
    ++ctx.launches;
  }
  if (parts > 1) all_gather(ctx, col_axis, reinterpret_cast<const float*>(mine), 2 * rows, reinterpret_cast<float*>(all));
  if (rows > 0) {
    k_eval_count<<<static_cast<unsigned>((rows + kT - 1) / kT), kT, 0, ctx.stream>>>(
        all, parts, rows, lb.r0, eval.sample.as<int64_t>(), g.labels.as<int32_t>(), g.split.as<uint8_t>(),
        lb.g_cols, counts);
    ++ctx.launches;
  }
  all_reduce_u64(ctx, row_axis, reinterpret_cast<uint64_t*>(counts), 6);
  GGB_CUDA(cudaMemcpyAsync(counts_out, counts, 6 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx.stream));
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
  ctx.d2h_bytes += 6 * sizeof(uint64_t);
}

}  // namespace ggb
