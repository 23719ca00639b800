// Communication-free uniform vertex sampling and induced-subgraph CSR
// construction (ScaleGNN Alg. 2) as sm_100a kernels, bit-exact with the
// reference:
//   sample_vertices      src/sampling.cpp:11-33  (partial Fisher-Yates, sorted)
//   locate_ranges        src/shardsample.cpp:47-56
//   extract_rows         src/shardsample.cpp:58-87
//   filter_and_remap     src/shardsample.cpp:89-109
//   assemble_shard       src/shardsample.cpp:111-122 (+ csr.cpp:29-94)
//   build_step_batch     include/gridgnn/model.hpp:250-309
//
// Sampling. The reference swaps perm[i] <-> perm[j_i], j_i = i +
// next_below(n-i), for i < b, then sorts the first b entries. Only the SET
// of the first b entries matters, and it is resolved in parallel:
//   val(k) = value at position k just before step k
//          = val(m) for the last m < k with j_m == k, else k;
//   out(i) = val(i) if j_i == i, else val(m) for the last m < i with
//            j_m == j_i, else j_i.
// Steps sharing a target are chained through a step-tagged head table (the
// analogue of the reference RemapTable tags, shardsample.hpp:29-55), the
// chosen ids are set in an n-bit bitmap, and a popcount prefix over the
// bitmap words both compacts the sorted sample and serves as the O(1)
// global-id -> sample-rank table that replaces every binary search of the
// reference (locate_ranges, filter_and_remap, sample_partition).
//
// Extraction. One warp per sampled row streams the row's column ids with
// coalesced loads, tests membership in the bitmap, ballots, and writes the
// kept entries in order: rows arrive in increasing global id and columns are
// sorted within a static shard row, so the output is canonical CSR
// (csr_from_triples order) without a sort. The transposed block is extracted
// the same way from the static transposed shard, which yields exactly the
// stable csr_transpose order.
#include <cmath>

#include "ops.hpp"
#include "prof.hpp"
#include "rng.cuh"
#include "trainer.hpp"
#include "runtime.hpp"

namespace ggb {
namespace {

constexpr int kThreads = 256;

// Rejection sampling of next_below (rng.hpp:38-45): a draw x >= limit is
// discarded and the stream advances, so every later step reads its counter
// one further. reject_mod > 0 adds "x % reject_mod == 0" as a rejection
// (a test-only rule that makes rejections frequent, mirrored by the oracle).
__device__ __forceinline__ bool rejected(uint64_t x, uint64_t limit, uint64_t reject_mod) {
  return x >= limit || (reject_mod && x % reject_mod == 0);
}

// Draws of steps i >= from, assuming `shift` rejections before them: step i
// reads counter i + shift. The first rejected step goes to *next_first
// (atomicMin); steps before `from` keep their draws. Pass 0 covers all steps
// with no rejections assumed; pass p > 0 re-draws only the suffix from the
// first rejection the previous pass found (a no-op when there was none).
__global__ void k_draw(int64_t n, int64_t b, uint64_t s0, const int64_t* __restrict__ first_in, int shift,
                       int64_t* __restrict__ next_first, uint64_t reject_mod, int32_t* __restrict__ j) {
  const int64_t from = first_in ? *first_in : 0;
  if (from >= b) return;
  const int64_t i = from + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= b) return;
  const uint64_t bound = static_cast<uint64_t>(n - i);
  const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
  const uint64_t x = stream_draw(s0, static_cast<uint64_t>(i + shift));
  if (rejected(x, limit, reject_mod)) atomicMin(reinterpret_cast<unsigned long long*>(next_first), i);
  j[i] = static_cast<int32_t>(i + static_cast<int64_t>(x % bound));
}

// More rejections than the passes cover (probability ~ (b n / 2^64)^3 per
// batch): exact sequential replay from the start.
__global__ void k_draw_replay(int64_t n, int64_t b, uint64_t s0, const int64_t* last_first, uint64_t reject_mod,
                              int32_t* j) {
  if (*last_first >= b) return;
  uint64_t k = 0;
  for (int64_t i = 0; i < b; ++i) {
    const uint64_t bound = static_cast<uint64_t>(n - i);
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x;
    do {
      x = stream_draw(s0, k++);
    } while (rejected(x, limit, reject_mod));
    j[i] = static_cast<int32_t>(i + static_cast<int64_t>(x % bound));
  }
}

__global__ void k_fill_i64(int64_t* p, int n, int64_t v) {
  if (threadIdx.x < n) p[threadIdx.x] = v;
}

__global__ void k_link(int64_t b, const int32_t* __restrict__ j, unsigned long long* head,
                       uint32_t tag, int32_t* __restrict__ next) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= b) return;
  const unsigned long long mine = (static_cast<unsigned long long>(tag) << 32) | static_cast<uint32_t>(i);
  const unsigned long long old = atomicExch(head + j[i], mine);
  next[i] = (static_cast<uint32_t>(old >> 32) == tag) ? static_cast<int32_t>(old & 0xffffffffu) : -1;
}

// Largest step m < limit whose target is t, or -1.
__device__ __forceinline__ int32_t last_before(const unsigned long long* head, const int32_t* next,
                                               uint32_t tag, int32_t t, int32_t limit) {
  const unsigned long long h = head[t];
  if (static_cast<uint32_t>(h >> 32) != tag) return -1;
  int32_t m = static_cast<int32_t>(h & 0xffffffffu), best = -1;
  while (m >= 0) {
    if (m < limit && m > best) best = m;
    m = next[m];
  }
  return best;
}

__global__ void k_resolve(int64_t b, const int32_t* __restrict__ j,
                          const unsigned long long* __restrict__ head,
                          const int32_t* __restrict__ next, uint32_t tag, uint32_t* bitmap) {
  const int64_t i64 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i64 >= b) return;
  const int32_t i = static_cast<int32_t>(i64);
  const int32_t ji = j[i];
  int32_t cur;
  bool chain = true;  // cur is a position whose pre-step value val(cur) is wanted
  if (ji == i) {
    cur = i;
  } else {
    cur = last_before(head, next, tag, ji, i);
    if (cur < 0) {  // position ji untouched before step i: it still holds ji
      cur = ji;
      chain = false;
    }
  }
  if (chain) {
    for (;;) {
      const int32_t p = last_before(head, next, tag, cur, cur);
      if (p < 0) break;
      cur = p;
    }
  }
  atomicOr(bitmap + (cur >> 5), 1u << (cur & 31));
}

__global__ void k_popc(int64_t words, const uint32_t* __restrict__ bitmap, int32_t* __restrict__ cnt) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w < words) cnt[w] = __popc(bitmap[w]);
}

__global__ void k_compact(int64_t words, const uint32_t* __restrict__ bitmap,
                          const int32_t* __restrict__ wpfx, int64_t* __restrict__ out) {
  const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= words) return;
  uint32_t m = bitmap[w];
  int64_t pos = wpfx[w];
  while (m) {
    const int bit = __ffs(m) - 1;
    out[pos++] = w * 32 + bit;
    m &= m - 1;
  }
}

__device__ __forceinline__ int64_t rank_of(const uint32_t* bitmap, const int32_t* wpfx, int64_t v) {
  const int64_t w = v >> 5;
  return wpfx[w] + __popc(bitmap[w] & ((1u << (v & 31)) - 1u));
}

// batch_off: ranks of the block_partition boundaries (sample_partition)
__global__ void k_ranks(int m, const int64_t* __restrict__ q, const uint32_t* __restrict__ bitmap,
                        const int32_t* __restrict__ wpfx, int64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] = rank_of(bitmap, wpfx, q[i]);
}

// Pass 1: kept entries per sampled row; block totals of the extracted count.
__global__ void k_extract_count(int64_t nr, const int64_t* __restrict__ sample, int64_t row_lo,
                                int64_t shard_r0, const int64_t* __restrict__ srp,
                                const int32_t* __restrict__ scol, const uint32_t* __restrict__ bitmap,
                                int32_t* __restrict__ cnt, unsigned long long* extracted) {
  __shared__ unsigned long long part[kThreads / 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + wib;
  unsigned long long ext = 0;
  if (w < nr) {
    const int64_t v = sample[row_lo + w];
    const int64_t e0 = srp[v - shard_r0], e1 = srp[v - shard_r0 + 1];
    int32_t c = 0;
    // 64 entries per iteration (two per lane), all loads issued before the
    // ballots: the col -> bitmap chain is paid once per 64 entries
    for (int64_t e = e0; e < e1; e += 64) {
      const int64_t k0 = e + lane, k1 = k0 + 32;
      const int32_t c0 = k0 < e1 ? scol[k0] : -1, c1 = k1 < e1 ? scol[k1] : -1;
      const uint32_t w0 = c0 >= 0 ? __ldg(bitmap + (c0 >> 5)) : 0u, w1 = c1 >= 0 ? __ldg(bitmap + (c1 >> 5)) : 0u;
      const bool keep0 = c0 >= 0 && ((w0 >> (c0 & 31)) & 1u), keep1 = c1 >= 0 && ((w1 >> (c1 & 31)) & 1u);
      c += __popc(__ballot_sync(0xffffffffu, keep0)) + __popc(__ballot_sync(0xffffffffu, keep1));
    }
    if (lane == 0) cnt[w] = c;
    ext = static_cast<unsigned long long>(e1 - e0);
  }
  if (lane == 0) part[wib] = ext;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int k = 0; k < kThreads / 32; ++k) s += part[k];
    if (s) atomicAdd(extracted, s);
  }
}

// Pass 2: write the kept entries (canonical order), fp64 rescale by 1/p of
// off-diagonal entries (global ids), compact column ids via the rank table.
__global__ void k_extract_fill(int64_t nr, const int64_t* __restrict__ sample, int64_t row_lo,
                               int64_t shard_r0, const int64_t* __restrict__ srp,
                               const int32_t* __restrict__ scol, const double* __restrict__ sval,
                               const int32_t* __restrict__ deg, const uint32_t* __restrict__ bitmap, const int32_t* __restrict__ wpfx,
                               int64_t col_lo, double p, const int64_t* __restrict__ row_ptr,
                               int32_t* __restrict__ col_out, float* __restrict__ val_out,
                               double* __restrict__ val64_out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5);
  if (w >= nr) return;
  const int64_t v = sample[row_lo + w];
  const int64_t e0 = srp[v - shard_r0], e1 = srp[v - shard_r0 + 1];
  int64_t pos = row_ptr[w];
  const uint32_t lt = (1u << lane) - 1u;
  const double dv = deg ? static_cast<double>(deg[v]) : 0.0;
  // 64 entries per iteration (two per lane, loads hoisted), in CSR order:
  // entries k0 = e + lane first, then k1 = e + 32 + lane
  auto emit = [&](int64_t k, int32_t col, uint32_t word, int64_t dst) {
    const int64_t rk = wpfx[col >> 5] + __popc(word & ((1u << (col & 31)) - 1u));
    col_out[dst] = static_cast<int32_t>(rk - col_lo);
    // value-free shards: the normalized value from the two row degrees
    // (dataset.cpp:78-79; IEEE fp64 multiply, sqrt and divide, so exact)
    double x = deg ? __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(dv, static_cast<double>(deg[col])))) : sval[k];
    if (v != static_cast<int64_t>(col)) x = x / p;
    val_out[dst] = static_cast<float>(x);
    val64_out[dst] = x;
  };
  for (int64_t e = e0; e < e1; e += 64) {
    const int64_t k0 = e + lane, k1 = k0 + 32;
    const int32_t c0 = k0 < e1 ? scol[k0] : -1, c1 = k1 < e1 ? scol[k1] : -1;
    const uint32_t w0 = c0 >= 0 ? __ldg(bitmap + (c0 >> 5)) : 0u, w1 = c1 >= 0 ? __ldg(bitmap + (c1 >> 5)) : 0u;
    const bool keep0 = c0 >= 0 && ((w0 >> (c0 & 31)) & 1u), keep1 = c1 >= 0 && ((w1 >> (c1 & 31)) & 1u);
    const uint32_t m0 = __ballot_sync(0xffffffffu, keep0), m1 = __ballot_sync(0xffffffffu, keep1);
    if (keep0) emit(k0, c0, w0, pos + __popc(m0 & lt));
    if (keep1) emit(k1, c1, w1, pos + __popc(m0) + __popc(m1 & lt));
    pos += __popc(m0) + __popc(m1);
  }
}

// x_in rows: bf16 hi (+ lo residual for the split-bf16 GEMM) and/or exact
// fp32, zero padded to the row stride. One warp per gathered row (grid-stride),
// 16-byte loads when the feature rows are 16-byte aligned.
__device__ __forceinline__ uint2 pack4_bf16(float a, float b, float c, float d) {
  __nv_bfloat162 h0 = __floats2bfloat162_rn(a, b), h1 = __floats2bfloat162_rn(c, d);
  return make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
}
__device__ __forceinline__ float lo_of(float v) { return v - __bfloat162float(__float2bfloat16_rn(v)); }

// U: rows in flight per warp (U > 1 for the PCIe-latency-bound host gather);
// Q: 16-byte quads per lane (rows of <= 128 Q floats). Q is sized to the row
// so the register footprint stays small: the host gather runs for
// milliseconds beside the step's persistent SpMM / GEMM CTAs and must fit the
// register file next to them (Q = 4 at U = 4 took 102 registers per thread,
// which kept those CTAs off the SMs holding gather blocks)
template <int U, int Q>
__global__ void k_gather_x(int64_t rows, int64_t cols, int64_t ld, const int64_t* __restrict__ sample,
                           int64_t row_lo, const float* __restrict__ feats, int64_t fld,
                           bf16* __restrict__ xb, bf16* __restrict__ xl, float* __restrict__ xf, int64_t xfld) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool vec = (cols & 3) == 0 && (fld & 3) == 0 && (ld & 3) == 0 && (!xf || (xfld & 3) == 0) && ld <= 128 * Q;
  if (vec) {
    for (int64_t rb = w0; rb < rows; rb += nw * U) {
      float4 x[U][Q];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = rb + u * nw;
        const float* src = r < rows ? feats + sample[row_lo + r] * fld : nullptr;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int64_t c = lane * 4 + q * 128;
          x[u][q] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (src && c < cols) x[u][q] = __ldg(reinterpret_cast<const float4*>(src + c));
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = rb + u * nw;
        if (r >= rows) break;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int64_t c = lane * 4 + q * 128;
          if (c >= ld) break;
          const float4 v = x[u][q];
          if (xb) *reinterpret_cast<uint2*>(xb + r * ld + c) = pack4_bf16(v.x, v.y, v.z, v.w);
          if (xl) *reinterpret_cast<uint2*>(xl + r * ld + c) = pack4_bf16(lo_of(v.x), lo_of(v.y), lo_of(v.z), lo_of(v.w));
          if (xf && c < xfld) *reinterpret_cast<float4*>(xf + r * xfld + c) = v;
        }
      }
    }
    return;
  }
  for (int64_t r = w0; r < rows; r += nw) {
    const float* src = feats + sample[row_lo + r] * fld;
    for (int64_t c = lane; c < ld; c += 32) {
      const float x = c < cols ? src[c] : 0.0f;
      const bf16 h = __float2bfloat16_rn(x);
      if (xb) xb[r * ld + c] = h;
      if (xl) xl[r * ld + c] = __float2bfloat16_rn(x - __bfloat162float(h));
      if (xf && c < xfld) xf[r * xfld + c] = x;
    }
  }
}

// Rows that do not split into 16-byte vectors (d_in % 4 != 0, e.g. 602)
// from host memory: every lane issues its K column loads of the row before
// storing any, so a warp keeps a whole row of PCIe reads in flight instead of
// one load per lane (the plain scalar loop: ~12 GB/s at C3).
template <int K>
__global__ void k_gather_x_wide(int64_t rows, int64_t cols, int64_t ld, const int64_t* __restrict__ sample,
                                int64_t row_lo, const float* __restrict__ feats, int64_t fld, bf16* __restrict__ xb,
                                bf16* __restrict__ xl, float* __restrict__ xf, int64_t xfld) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w0; r < rows; r += nw) {
    const float* src = feats + sample[row_lo + r] * fld;
    float v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t c = lane + 32 * k;
      v[k] = c < cols ? __ldg(src + c) : 0.0f;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int64_t c = lane + 32 * k;
      if (c >= ld) break;
      const bf16 h = __float2bfloat16_rn(v[k]);
      if (xb) xb[r * ld + c] = h;
      if (xl) xl[r * ld + c] = __float2bfloat16_rn(v[k] - __bfloat162float(h));
      if (xf && c < xfld) xf[r * xfld + c] = v[k];
    }
  }
}

// Host-resident features are read over PCIe by a small grid with several
// rows in flight per warp, so the gather, which runs for milliseconds on the
// sampling stream, holds only part of a few SMs while keeping enough reads
// outstanding for the link (measured at C2: 245 MB in ~5 ms, ~49 GB/s, the
// same from 32 to 296 blocks; round 2, e2e ms/step: 16 blocks 11.24-11.58,
// 24 11.51, 32 11.75-11.81 — the fewer SMs it touches, the less it slows the
// step's persistent kernels).
int host_gather_blocks() {
  static int v = [] {
    const char* e = std::getenv("GGB_HOST_GATHER_BLOCKS");
    const int b = e ? std::atoi(e) : 16;
    return b > 0 ? b : 16;
  }();
  return v;
}

void launch_gather_x(const Ctx& ctx, cudaStream_t s, bool host, int64_t rows, int64_t cols, int64_t ld,
                     const int64_t* sample, int64_t row_lo, const float* feats, int64_t fld, bf16* xb, bf16* xl,
                     float* xf, int64_t xfld) {
  if (rows <= 0) return;
  if (host) {
    // GGB_HOST_GATHER_TPB: threads per block (32 .. 256). One-warp blocks
    // (2K registers) would fit beside a persistent SpMM CTA on the same SM,
    // where a 256-thread block (16K) does not, but they measured slower
    // end to end (C2 e2e 13.9-14.4 vs 12.7-13.2 ms/step): 256 stays
    static const int tpb = [] {
      const char* e = std::getenv("GGB_HOST_GATHER_TPB");
      const int t = e ? std::atoi(e) : 256;
      return t >= 32 && t <= 256 && t % 32 == 0 ? t : 256;
    }();
    const int wpb = tpb / 32;
    const unsigned blocks = std::max(
        1u, static_cast<unsigned>(std::min<int64_t>(ceil_div(rows, 4 * wpb), 8 * host_gather_blocks() / wpb)));
    const bool vec4 = (cols & 3) == 0 && (fld & 3) == 0 && (ld & 3) == 0 && (!xf || (xfld & 3) == 0) && ld <= 512;
    if (!vec4 && ld <= 640) {
      const unsigned wblocks = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 8 * 4), 4 * host_gather_blocks())));
      k_gather_x_wide<20><<<wblocks, 256, 0, s>>>(rows, cols, ld, sample, row_lo, feats, fld, xb, xl, xf, xfld);
    } else if (ld <= 128)
      k_gather_x<4, 1><<<blocks, tpb, 0, s>>>(rows, cols, ld, sample, row_lo, feats, fld, xb, xl, xf, xfld);
    else if (ld <= 256)
      k_gather_x<4, 2><<<blocks, tpb, 0, s>>>(rows, cols, ld, sample, row_lo, feats, fld, xb, xl, xf, xfld);
    else
      k_gather_x<4, 4><<<blocks, tpb, 0, s>>>(rows, cols, ld, sample, row_lo, feats, fld, xb, xl, xf, xfld);
  } else {
    const unsigned blocks =
        static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 8), ctx.num_sms * 64)));
    if (ld <= 128)
      k_gather_x<1, 1><<<blocks, 256, 0, s>>>(rows, cols, ld, sample, row_lo, feats, fld, xb, xl, xf, xfld);
    else
      k_gather_x<1, 4><<<blocks, 256, 0, s>>>(rows, cols, ld, sample, row_lo, feats, fld, xb, xl, xf, xfld);
  }
  GGB_LAUNCH_CHECK();
}

__global__ void k_gather_labels(int64_t b, const int64_t* __restrict__ sample,
                                const int32_t* __restrict__ labels, int32_t* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < b) out[i] = labels[sample[i]];
}

inline unsigned blocks(int64_t n, int t = kThreads) { return static_cast<unsigned>(ceil_div(n, t)); }

}  // namespace

constexpr int kDrawPasses = 3;  // re-draw passes after the first (rejections they absorb: kDrawPasses - 1)

void sample_set(Ctx& ctx, int64_t n, int64_t b, uint64_t seed, uint64_t step, int64_t* d_sample,
                uint64_t reject_mod) {
  require(b >= 1 && b <= n, "sample_vertices: need 1 <= b <= n");
  require(n < (int64_t{1} << 31) - 64, "sample_vertices: n must be < 2^31");
  SamplerWork& sw = ctx.sw;
  cudaStream_t s = ctx.stream;
  if (sw.head_n < n) {
    sw.head.reserve(static_cast<size_t>(n) * 8);
    GGB_CUDA(cudaMemsetAsync(sw.head.p, 0, static_cast<size_t>(n) * 8, s));
    sw.head_n = n;
    sw.tag = 0;
  }
  if (++sw.tag == 0) {  // tag wrap: clear the table
    GGB_CUDA(cudaMemsetAsync(sw.head.p, 0, static_cast<size_t>(sw.head_n) * 8, s));
    sw.tag = 1;
  }
  const int64_t words = n / 32 + 2;
  int32_t* j = sw.j.reserve_n<int32_t>(b);
  int32_t* next = sw.next.reserve_n<int32_t>(b);
  int64_t* first = sw.flag.reserve_n<int64_t>(kDrawPasses + 1);  // first rejected step found by each pass
  uint32_t* bitmap = sw.bitmap.reserve_n<uint32_t>(words);
  int32_t* wcount = sw.wcount.reserve_n<int32_t>(words);
  int32_t* wpfx = sw.wpfx.reserve_n<int32_t>(words + 1);
  GGB_CUDA(cudaMemsetAsync(bitmap, 0, static_cast<size_t>(words) * 4, s));
  const uint64_t s0 = splitmix64(seed + step);  // sampling.cpp:16
  k_fill_i64<<<1, 32, 0, s>>>(first, kDrawPasses + 1, b);
  k_draw<<<blocks(b), kThreads, 0, s>>>(n, b, s0, nullptr, 0, first, reject_mod, j);
  for (int p = 1; p < kDrawPasses; ++p)
    k_draw<<<blocks(b), kThreads, 0, s>>>(n, b, s0, first + p - 1, p, first + p, reject_mod, j);
  k_draw_replay<<<1, 1, 0, s>>>(n, b, s0, first + kDrawPasses - 1, reject_mod, j);
  k_link<<<blocks(b), kThreads, 0, s>>>(b, j, sw.head.as<unsigned long long>(), sw.tag, next);
  k_resolve<<<blocks(b), kThreads, 0, s>>>(b, j, sw.head.as<unsigned long long>(), next, sw.tag,
                                           bitmap);
  k_popc<<<blocks(words), kThreads, 0, s>>>(words, bitmap, wcount);
  exclusive_scan_i32(wcount, wpfx, words, sw.scan_tmp, s);
  k_compact<<<blocks(words), kThreads, 0, s>>>(words, bitmap, wpfx, d_sample);
  GGB_LAUNCH_CHECK();
  ctx.launches += 8 + kDrawPasses;
}

namespace {

void extract_block(Ctx& ctx, const PlaneShard& sh, const int64_t* d_sample, int64_t row_lo,
                   int64_t row_hi, int64_t col_lo, int64_t col_hi, int64_t b, int64_t n,
                   BatchCsr& out, int32_t* d_cnt, unsigned long long* d_ext) {
  out.n_rows = row_hi - row_lo;
  out.n_cols = col_hi - col_lo;
  int64_t* rp = out.row_ptr.reserve_n<int64_t>(out.n_rows + 1);
  if (out.n_rows > 0) {
    k_extract_count<<<blocks(out.n_rows, kThreads / 32), kThreads, 0, ctx.stream>>>(
        out.n_rows, d_sample, row_lo, sh.r0, sh.row_ptr.as<int64_t>(), sh.col.as<int32_t>(),
        ctx.sw.bitmap.as<uint32_t>(), d_cnt, d_ext);
    ctx.launches += 1;
  }
  exclusive_scan_i32_to_i64(d_cnt, rp, out.n_rows, ctx.sw.scan_tmp, ctx.stream);
  ctx.launches += 3;
  (void)b;
  (void)n;
}

void fill_block(Ctx& ctx, const PlaneShard& sh, const int32_t* deg, const int64_t* d_sample, int64_t row_lo,
                int64_t col_lo, int64_t b, int64_t n, BatchCsr& out, int64_t cap) {
  out.col.reserve_n<int32_t>(cap);
  out.val.reserve_n<float>(cap);
  out.val64.reserve_n<double>(cap);
  if (out.n_rows == 0) return;
  const double p = static_cast<double>(b - 1) / static_cast<double>(n - 1);  // shardsample.cpp:116
  k_extract_fill<<<blocks(out.n_rows, kThreads / 32), kThreads, 0, ctx.stream>>>(
      out.n_rows, d_sample, row_lo, sh.r0, sh.row_ptr.as<int64_t>(), sh.col.as<int32_t>(),
      sh.val.as<double>(), deg, ctx.sw.bitmap.as<uint32_t>(), ctx.sw.wpfx.as<int32_t>(), col_lo, p,
      out.row_ptr.as<int64_t>(), out.col.as<int32_t>(), out.val.as<float>(), out.val64.as<double>());
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

}  // namespace

// GGB_AUX_GATHER=0 keeps the PCIe feature gather on the build's stream
bool aux_gather_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GGB_AUX_GATHER");
    return !(e && e[0] == '0');
  }();
  return on;
}

void build_step_batch(Ctx& ctx, const Graph& g, int64_t b, uint64_t group_seed, uint64_t step,
                      Batch& bt, bool want_xf) {
  require(b >= 2 && b <= g.n, "build_local_minibatch: need 2 <= b <= N");
  ProfScope prof(ctx, kProfSample);
  cudaStream_t s = ctx.stream;
  bt.ctx = &ctx;
  bt.graph = &g;
  bt.b = b;
  bt.n = g.n;
  bt.planes = g.planes;
  int64_t* d_sample = bt.sample.reserve_n<int64_t>(b);
  sample_set(ctx, g.n, b, group_seed, step, d_sample);

  // batch_off[a] = sample_partition(S, block_partition(N, g_a)) (model.hpp:257-259);
  // with X, Y and Z unsplit every partition is [0, N), so every offset list is
  // {0, b} and the device rank query (a host round trip) is skipped
  const bool flat = ctx.grid.dims[1] == 1 && ctx.grid.dims[2] == 1 && ctx.grid.dims[3] == 1;
  int64_t* dmisc = nullptr;
  int64_t* hmisc = nullptr;
  int m = 0;
  if (flat) {
    for (int a = 1; a < 4; ++a) bt.batch_off[a] = {0, b};
    dmisc = ctx.sw.dev_misc.reserve_n<int64_t>(64);
    hmisc = static_cast<int64_t*>(ctx.sw.host_misc.reserve(64 * 8));
  } else {
  std::vector<int64_t> q;
  for (int a = 1; a < 4; ++a) {
    auto off = block_partition(g.n, ctx.grid.dims[a]);
    q.insert(q.end(), off.begin(), off.end());
  }
  m = static_cast<int>(q.size());
  // device scratch: [0,m) queries, [m,2m) ranks, [2m, 2m+2) extracted counters
  dmisc = ctx.sw.dev_misc.reserve_n<int64_t>(2 * m + 64);
  hmisc = static_cast<int64_t*>(ctx.sw.host_misc.reserve((2 * m + 64) * 8));
  std::copy(q.begin(), q.end(), hmisc);
  GGB_CUDA(cudaMemcpyAsync(dmisc, hmisc, m * 8, cudaMemcpyHostToDevice, s));
  k_ranks<<<1, 128, 0, s>>>(m, dmisc, ctx.sw.bitmap.as<uint32_t>(), ctx.sw.wpfx.as<int32_t>(),
                            dmisc + m);
  ctx.launches += 1;
  GGB_CUDA(cudaMemcpyAsync(hmisc + m, dmisc + m, m * 8, cudaMemcpyDeviceToHost, s));
  ctx.h2d_bytes += m * 8;
  ctx.d2h_bytes += m * 8;
  GGB_CUDA(cudaStreamSynchronize(s));
  {
    int k = 0;
    for (int a = 1; a < 4; ++a) {
      bt.batch_off[a].assign(hmisc + m + k, hmisc + m + k + ctx.grid.dims[a] + 1);
      k += ctx.grid.dims[a] + 1;
    }
  }
  }

  bt.p_ready = false;
  // x_in (X,Z) = features[S rows of this X block, Z column block] (model.hpp:293-303).
  // Needs only the sample and the batch offsets: host-resident features are
  // gathered over PCIe on the second stream while the shard blocks are
  // extracted on this one (joined before the build returns).
  const bool gather_aside = g.features_on_host() && aux_gather_enabled();
  {
    const auto& xo = bt.batch_off[kInputFeatureLayout.row];
    const int cx = ctx.coord[kInputFeatureLayout.row];
    bt.x_r0 = xo[cx];
    bt.x_r1 = xo[cx + 1];
    bt.x_c0 = g.feat_c0;
    bt.x_c1 = g.feat_c1;
    const int64_t cols = bt.x_c1 - bt.x_c0;
    bt.x_ld = round_up(std::max<int64_t>(cols, 1), 8);
    const int64_t rows = bt.x_r1 - bt.x_r0;
    bf16* xb = bt.x_in.reserve_n<bf16>(std::max<int64_t>(rows, 1) * bt.x_ld);
    bf16* xl = bt.x_in_lo.reserve_n<bf16>(std::max<int64_t>(rows, 1) * bt.x_ld);
    // fp32 rows too when the first layer will be pre-aggregated (one gather)
    // (host-resident features: always, so the rows cross PCIe once)
    bt.x_f_ready = (want_xf || g.features_on_host()) && preagg_enabled() && preagg_eligible(ctx, bt);
    float* xf = bt.x_f_ready ? bt.x_f.reserve_n<float>(std::max<int64_t>(rows, 1) * bt.x_ld) : nullptr;
    cudaStream_t xs = s;
    if (gather_aside) {
      SamplerWork::Aux& ax = ctx.sw.aux;
      if (!ax.s) {
        int prio = 0;
        GGB_CUDA(cudaStreamGetPriority(s, &prio));
        GGB_CUDA(cudaStreamCreateWithPriority(&ax.s, cudaStreamNonBlocking, prio));
        GGB_CUDA(cudaEventCreateWithFlags(&ax.fork, cudaEventDisableTiming));
        GGB_CUDA(cudaEventCreateWithFlags(&ax.join, cudaEventDisableTiming));
      }
      GGB_CUDA(cudaEventRecord(ax.fork, s));
      GGB_CUDA(cudaStreamWaitEvent(ax.s, ax.fork, 0));
      xs = ax.s;
    }
    if (rows > 0) {
      launch_gather_x(ctx, xs, g.features_on_host(), rows, cols, bt.x_ld, d_sample, bt.x_r0, g.feat_ptr, cols, xb,
                      xl, xf, bt.x_ld);
      ctx.launches += 1;
    }
    bt.h2d_bytes = g.features_on_host() ? static_cast<uint64_t>(rows) * cols * 4 : 0;
    ctx.h2d_bytes += bt.h2d_bytes;
  }

  // Plane blocks. Identical static shards (e.g. every plane on 1x1x1 grids)
  // share one extracted block.
  struct Key {
    int shard;
    int64_t rl, rh, cl, ch;
  };
  std::vector<Key> keys;
  bt.csr_of.assign(g.planes, -1);
  bt.csrt_of.assign(g.planes, -1);
  auto find_or_add = [&](int shard, int64_t rl, int64_t rh, int64_t cl, int64_t ch) {
    for (size_t k = 0; k < keys.size(); ++k)
      if (keys[k].shard == shard && keys[k].rl == rl && keys[k].rh == rh && keys[k].cl == cl &&
          keys[k].ch == ch)
        return static_cast<int>(k);
    keys.push_back({shard, rl, rh, cl, ch});
    return static_cast<int>(keys.size() - 1);
  };
  for (int p = 0; p < g.planes; ++p) {
    const Layout lay = adjacency_layout(p + 1);
    const auto& ro = bt.batch_off[lay.row];
    const auto& co = bt.batch_off[lay.col];
    const int cr = ctx.coord[lay.row], cc = ctx.coord[lay.col];
    const int64_t rl = ro[cr], rh = ro[cr + 1], cl = co[cc], ch = co[cc + 1];
    bt.csr_of[p] = find_or_add(g.fwd_of[p], rl, rh, cl, ch);
    bt.csrt_of[p] = find_or_add(g.tr_of[p], cl, ch, rl, rh);
  }
  if (bt.csrs.size() < keys.size()) bt.csrs.resize(keys.size());

  int64_t max_rows = 0;
  for (auto& k : keys) max_rows = std::max(max_rows, k.rh - k.rl);
  // per block: counts region, one extracted counter
  int32_t* d_cnt = ctx.sw.cnt.reserve_n<int32_t>((max_rows + 1) * keys.size() + 1);
  unsigned long long* d_ext = reinterpret_cast<unsigned long long*>(dmisc + 2 * m);
  GGB_CUDA(cudaMemsetAsync(d_ext, 0, 8 * keys.size(), s));
  for (size_t k = 0; k < keys.size(); ++k) {
    const Key& kk = keys[k];
    BatchCsr& out = bt.csrs[k];
    out.long_rows = g.shards[kk.shard].power_law();
    out.r0 = kk.rl;
    out.r1 = kk.rh;
    out.c0 = kk.cl;
    out.c1 = kk.ch;
    extract_block(ctx, g.shards[kk.shard], d_sample, kk.rl, kk.rh, kk.cl, kk.ch, b, g.n, out,
                  d_cnt + k * (max_rows + 1), d_ext + k);
  }
  // totals: row_ptr[n_rows] of every block, plus the extracted counters, to
  // the batch's pinned buffer; the host reads them only when it needs them
  const size_t nk = keys.size();
  bt.nblocks = static_cast<int>(nk);
  int64_t* tot = static_cast<int64_t*>(bt.totals.reserve(16 * nk + 16));
  for (size_t k = 0; k < nk; ++k)
    GGB_CUDA(cudaMemcpyAsync(tot + k, bt.csrs[k].row_ptr.as<int64_t>() + bt.csrs[k].n_rows, 8,
                             cudaMemcpyDeviceToHost, s));
  GGB_CUDA(cudaMemcpyAsync(tot + nk, d_ext, 8 * nk, cudaMemcpyDeviceToHost, s));
  GGB_CUDA(cudaEventRecord(bt.totals_ready.get(), s));
  bt.totals_pending = true;
  ctx.d2h_bytes += 16 * nk;
  // Output capacity of every block without a host round trip: its kept
  // entries are at most its extracted ones, at most the n_rows largest row
  // degrees of its static shard. Past a memory budget (papers100M-scale
  // blocks), or when profiling needs the byte counts, wait for the exact
  // totals instead.
  std::vector<int64_t> cap(nk);
  size_t need = 0;
  bool bounded = true;
  for (size_t k = 0; k < nk; ++k) {
    const PlaneShard& sh = g.shards[keys[k].shard];
    bounded = bounded && !sh.rows_of_degree.empty();
    cap[k] = sh.top_rows_nnz(bt.csrs[k].n_rows) + 1;
    need += static_cast<size_t>(cap[k]) * (4 + 4 + 8);
  }
  if (!bounded || need > (size_t{2} << 30) || prof_of(ctx).on) {
    settle_totals(bt);
    for (size_t k = 0; k < nk; ++k) cap[k] = bt.csrs[k].nnz + bt.csrs[k].nnz / 16 + 1024;  // headroom for later steps
  }
  for (size_t k = 0; k < nk; ++k)
    fill_block(ctx, g.shards[keys[k].shard], g.value_free ? g.degree.as<int32_t>() : nullptr, d_sample, keys[k].rl,
               keys[k].cl, b, g.n, bt.csrs[k], cap[k]);

  if (gather_aside) {  // join the PCIe gather
    GGB_CUDA(cudaEventRecord(ctx.sw.aux.join, ctx.sw.aux.s));
    GGB_CUDA(cudaStreamWaitEvent(s, ctx.sw.aux.join, 0));
  }
  int32_t* lab = bt.labels.reserve_n<int32_t>(b);
  k_gather_labels<<<blocks(b), kThreads, 0, s>>>(b, d_sample, g.labels.as<int32_t>(), lab);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
  // algorithmic bytes: draws/links/bitmap over b, the bitmap and
  // its prefix over n/32 words, per block the sampled row pointers, the
  // extracted column ids, the kept entries (fp64 value read; int32 col, fp32
  // and fp64 value writes), the feature gather and the labels.
  if (!bt.totals_pending) {  // settled above (profiling)
    double bytes = 8.0 * b * 4 + (g.n / 32.0) * 12;
    for (size_t k = 0; k < nk; ++k) {
      const BatchCsr& c = bt.csrs[k];
      // per kept entry: the value read (fp64, or a 4-byte degree when value-free), int32 col + fp32 + fp64 writes
      bytes += c.n_rows * 16.0 * 2 + static_cast<double>(tot[nk + k]) * 4.0 * 2 +
               c.nnz * ((g.value_free ? 4.0 : 8.0) + 4 + 4 + 8);
    }
    bytes += static_cast<double>(bt.x_r1 - bt.x_r0) * (bt.x_c1 - bt.x_c0) * (4 + 2 + 2) + b * 12.0;
    prof.bytes = bytes;
  }
}

void settle_totals(const Batch& bt) {
  if (!bt.totals_pending) return;
  GGB_CUDA(cudaEventSynchronize(bt.totals_ready.e));
  const int64_t* tot = static_cast<const int64_t*>(bt.totals.p);
  const size_t nk = static_cast<size_t>(bt.nblocks);
  for (size_t k = 0; k < nk; ++k) bt.csrs[k].nnz = tot[k];
  // counters as build_step_batch accumulates them (model.hpp:265-268): one
  // build_local_minibatch per plane, counting its forward block
  bt.nnz_extracted = 0;
  bt.nnz_kept = 0;
  for (int p = 0; p < bt.planes; ++p) {
    bt.nnz_extracted += static_cast<uint64_t>(tot[nk + bt.csr_of[p]]);
    bt.nnz_kept += static_cast<uint64_t>(bt.csrs[bt.csr_of[p]].nnz);
  }
  bt.totals_pending = false;
}

void shard_degree_profile(Ctx& ctx, PlaneShard& sh) {
  const int64_t rows = sh.r1 - sh.r0;
  sh.rows_of_degree.clear();
  if (rows <= 0) return;
  std::vector<int64_t> rp(static_cast<size_t>(rows) + 1);
  GGB_CUDA(cudaMemcpyAsync(rp.data(), sh.row_ptr.p, rp.size() * 8, cudaMemcpyDeviceToHost, ctx.stream));
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
  int64_t dmax = 0;
  for (int64_t r = 0; r < rows; ++r) dmax = std::max(dmax, rp[r + 1] - rp[r]);
  sh.rows_of_degree.assign(static_cast<size_t>(dmax) + 1, 0);
  for (int64_t r = 0; r < rows; ++r) ++sh.rows_of_degree[static_cast<size_t>(rp[r + 1] - rp[r])];
}

void gather_x_in_fp32(Ctx& ctx, const Batch& bt, float* d_out) {
  const int64_t rows = bt.x_r1 - bt.x_r0, cols = bt.x_c1 - bt.x_c0;
  if (rows <= 0 || cols <= 0) return;
  launch_gather_x(ctx, ctx.stream, bt.graph->features_on_host(), rows, cols, cols, bt.sample.as<int64_t>(), bt.x_r0,
                  bt.graph->feat_ptr, cols, nullptr, nullptr, d_out, cols);
  ctx.launches += 1;
}

// Pre-aggregated input features of the first layer, P = A_0 . x_in.
// The reference's first layer computes A_0 . (x_in . W_in) (model.hpp:346-351);
// with d_in < H the association (A_0 . x_in) . W_in gathers d_in-wide rows
// instead of H-wide ones, and P depends on the batch only (no weights), so it
// is built with the batch, on the sampling stream when prefetched. Valid when
// plane 0's column axis (X) and x_in's column axis (Z) are unsplit, i.e. the
// X- and Z-partial sums of the two contractions need no all-reduce.
bool preagg_eligible(const Ctx& ctx, const Batch& bt) {
  return bt.planes >= 1 && ctx.grid.dims[kX] == 1 && ctx.grid.dims[kZ] == 1 && bt.x_c1 > bt.x_c0;
}

void preaggregate(Ctx& ctx, const Batch& bt) {
  require(preagg_eligible(ctx, bt), "preaggregate: grid splits the first layer's contractions");
  const BatchCsr& A = bt.csrs[bt.csr_of[0]];
  const int64_t xrows = bt.x_r1 - bt.x_r0, cols = bt.x_c1 - bt.x_c0;
  contract(A.c0 == bt.x_r0 && A.c1 == bt.x_r1, "preaggregate: A_0 columns differ from the x_in rows");
  float* xf = bt.x_f.reserve_n<float>(std::max<int64_t>(xrows, 1) * bt.x_ld);
  const bool gather = !bt.x_f_ready;
  bf16* ph = bt.p_in.reserve_n<bf16>(std::max<int64_t>(A.n_rows, 1) * bt.x_ld);
  bf16* pl = bt.p_in_lo.reserve_n<bf16>(std::max<int64_t>(A.n_rows, 1) * bt.x_ld);
  if (xrows > 0 && gather) {
    launch_gather_x(ctx, ctx.stream, bt.graph->features_on_host(), xrows, cols, bt.x_ld, bt.sample.as<int64_t>(),
                    bt.x_r0, bt.graph->feat_ptr, cols, nullptr, nullptr, xf, bt.x_ld);
    ctx.launches += 1;
  }
  if (A.n_rows > 0) {
    // padding columns of P stay zero (the GEMM reads K up to x_ld)
    GGB_CUDA(cudaMemsetAsync(ph, 0, static_cast<size_t>(A.n_rows) * bt.x_ld * 2, ctx.stream));
    GGB_CUDA(cudaMemsetAsync(pl, 0, static_cast<size_t>(A.n_rows) * bt.x_ld * 2, ctx.stream));
    LongRowsScope lrs(ctx, A.long_rows);
    spmm_csr_f32(ctx, A.n_rows, A.row_ptr.as<int64_t>(), A.col.as<int32_t>(), A.val.as<float>(), xf, bt.x_ld, cols,
                 nullptr, 0, ph, pl, bt.x_ld, 0);
  }
  bt.x_f_ready = true;
  bt.p_ready = true;
}

}  // namespace ggb
