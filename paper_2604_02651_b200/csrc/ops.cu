// Row-wise and element-wise kernels of the GCN layer, each citing the
// reference operator it replaces:
//   parallel_rmsnorm_fwd/bwd     pmm.hpp:206-287
//   fused_elementwise_fwd/bwd    pmm.hpp:289-341 (ReLU . dropout + residual)
//   parallel_cross_entropy       pmm.hpp:343-401
//   optimizer_step (SGD / Adam)  model.hpp:435-456
//   fill_weight_shard            model.hpp:139-149
// The dropout mask is the reference's counter hash
// element_unit(key, global_row, global_col) >= rate (pmm.hpp:317-322),
// evaluated in the forward pass and kept as one bit per element for the
// backward pass instead of the reference's fp32 `scale` matrix.
#include <algorithm>
#include <cmath>

#include "ops.hpp"
#include "rng.cuh"

namespace ggb {
namespace {

constexpr int kT = 256;
inline unsigned nb(int64_t n, int t = kT) { return static_cast<unsigned>(ceil_div(n, t)); }
// warp-per-row kernels: enough 256-thread blocks for every row, capped at 8 waves of 8 blocks per SM
inline unsigned row_blocks(const Ctx& ctx, int64_t rows) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, kT / 32), ctx.num_sms * 64)));
}

__global__ void k_init_weight(float* __restrict__ w, int64_t rows, int64_t cols, int64_t r0, int64_t c0,
                              uint64_t key, double lim) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols, c = i % cols;
  // (2u - 1) * lim in round-to-nearest fp64, never contracted (model.hpp:144-148)
  const double u = element_unit(key, static_cast<uint64_t>(r0 + r), static_cast<uint64_t>(c0 + c));
  w[i] = static_cast<float>(__dmul_rn(__dadd_rn(__dmul_rn(2.0, u), -1.0), lim));
}

__global__ void k_fill(float* __restrict__ x, int64_t n, float v) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

__global__ void k_weight_bf16(const float* __restrict__ w, int64_t rows, int64_t cols, bf16* __restrict__ wb,
                              int64_t ldb, bf16* __restrict__ wt, bf16* __restrict__ wtl, int64_t ldt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows * cols) return;
  const int64_t r = i / cols, c = i % cols;
  const bf16 v = __float2bfloat16_rn(w[i]);
  if (wb) wb[r * ldb + c] = v;
  if (wt) wt[c * ldt + r] = v;
  if (wtl) wtl[c * ldt + r] = __float2bfloat16_rn(w[i] - __bfloat162float(v));
}

// Row-blocked element-wise kernels over padded row-major matrices: one warp
// per row (grid-stride over rows), lanes over 4-column quads, 16-byte loads
// where the rows allow it. No index division.
__device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__device__ __forceinline__ uint2 pack4_bf16(float a, float b, float c, float d) {
  __nv_bfloat162 h0 = __floats2bfloat162_rn(a, b), h1 = __floats2bfloat162_rn(c, d);
  return make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
}

__device__ __forceinline__ float lo_of(float v) { return v - __bfloat162float(__float2bfloat16_rn(v)); }

template <bool Split>
__global__ void k_cast_rows(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                            bf16* __restrict__ hi, bf16* __restrict__ lo, int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool vec = (cols & 3) == 0 && (ldx & 3) == 0 && (ldy & 3) == 0 && al16(x) && ((reinterpret_cast<uintptr_t>(hi) & 7) == 0) &&
                   (!Split || (reinterpret_cast<uintptr_t>(lo) & 7) == 0);
  for (int64_t r = w0; r < rows; r += nw) {
    const float* xr = x + r * ldx;
    if (vec) {
      for (int64_t c = lane * 4; c < cols; c += 128) {
        const float4 v = *reinterpret_cast<const float4*>(xr + c);
        *reinterpret_cast<uint2*>(hi + r * ldy + c) = pack4_bf16(v.x, v.y, v.z, v.w);
        if (Split) *reinterpret_cast<uint2*>(lo + r * ldy + c) = pack4_bf16(lo_of(v.x), lo_of(v.y), lo_of(v.z), lo_of(v.w));
      }
    } else {
      for (int64_t c = lane; c < cols; c += 32) {
        const float v = xr[c];
        hi[r * ldy + c] = __float2bfloat16_rn(v);
        if (Split) lo[r * ldy + c] = __float2bfloat16_rn(lo_of(v));
      }
    }
  }
}

__global__ void k_add_rows(float* __restrict__ a, int64_t lda, const float* __restrict__ b, int64_t ldb,
                           int64_t rows, int64_t cols) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool vec = (cols & 3) == 0 && (lda & 3) == 0 && (ldb & 3) == 0 && al16(a) && al16(b);
  for (int64_t r = w0; r < rows; r += nw) {
    if (vec) {
      for (int64_t c = lane * 4; c < cols; c += 128) {
        float4 u = *reinterpret_cast<float4*>(a + r * lda + c);
        const float4 v = *reinterpret_cast<const float4*>(b + r * ldb + c);
        u.x += v.x;
        u.y += v.y;
        u.z += v.z;
        u.w += v.w;
        *reinterpret_cast<float4*>(a + r * lda + c) = u;
      }
    } else {
      for (int64_t c = lane; c < cols; c += 32) a[r * lda + c] += b[r * ldb + c];
    }
  }
}


// warp per row: ss[r] = sum_j x[r][j]^2 (pmm.hpp:220-228)
__global__ void k_rowsumsq(const float* __restrict__ x, int64_t ldx, int64_t rows, int64_t cols,
                           float* __restrict__ ss) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float s = 0.f;
  for (int64_t j = lane; j < cols; j += 32) {
    const float v = x[r * ldx + j];
    s = fmaf(v, v, s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) ss[r] = s;
}

// out[c] = sum_k part[k][c]; a block owns 32 columns, its 8 warps split the
// parts, then a fixed-order combine (deterministic).
// column sums of `parts` partial rows: 32 warps per 32 columns, each warp
// summing every 32nd partial, then the warps' sums in order
__global__ void __launch_bounds__(1024) k_reduce_rows(const float* __restrict__ part, int parts, int64_t cols,
                                                     float* __restrict__ out) {
  __shared__ float sh[32][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  float s = 0.f;
  if (c < cols)
    for (int k = w; k < parts; k += 32) s += part[k * cols + c];
  sh[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < cols) {
    float t = 0.f;
#pragma unroll 8
    for (int k = 0; k < 32; ++k) t += sh[k][lane];
    out[c] = t;
  }
}

// ---- cross-entropy, warp per row ---------------------------------------------------
__global__ void k_ce_rowmax(CeArgs p) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= p.rows) return;
  float m = -3.402823466e38f;  // numeric_limits<float>::lowest()
  for (int64_t j = lane; j < p.cols; j += 32) m = fmaxf(m, p.logits[r * p.ld + j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) p.mx[r] = m;
}

__global__ void k_ce_rowsum(CeArgs p) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= p.rows) return;
  const float m = p.mx[r];
  float z = 0.f;
  for (int64_t j = lane; j < p.cols; j += 32) z += expf(p.logits[r * p.ld + j] - m);
#pragma unroll
  for (int o = 16; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  if (lane == 0) {
    const int64_t y = p.labels[p.row_g0 + r];
    p.zt[2 * r] = z;
    p.zt[2 * r + 1] = (y >= p.c0 && y < p.c0 + p.cols) ? p.logits[r * p.ld + (y - p.c0)] : 0.f;
  }
}

__global__ void k_ce_grad(CeArgs p) {
  __shared__ float part[kT / 32];
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  float contrib = 0.f;
  if (r < p.rows) {
    const float m = p.mx[r], z = p.zt[2 * r];
    const int64_t y = p.labels[p.row_g0 + r];
    for (int64_t j = lane; j < p.cols; j += 32) {
      float g = expf(p.logits[r * p.ld + j] - m) / z;
      if (p.c0 + j == y) g -= 1.f;
      const float d = g * p.invb;
      if (p.dlog) p.dlog[r * p.lddlog + j] = d;
      if (p.dlogb) p.dlogb[r * p.lddlogb + j] = __float2bfloat16_rn(d);
    }
    if (lane == 0) contrib = (m + logf(z)) - p.zt[2 * r + 1];
  }
  if (lane == 0) part[threadIdx.x >> 5] = contrib;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int k = 0; k < kT / 32; ++k) s += part[k];
    p.loss_part[blockIdx.x] = s;
  }
}

__global__ void k_sum_parts(const float* __restrict__ part, int64_t n, float* __restrict__ out) {
  __shared__ float sh[kT];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += kT) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = kT / 2; o; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

__global__ void k_scale_scalar(const float* __restrict__ in, float s, float* __restrict__ out) {
  out[0] = in[0] * s;
}

// ---- optimizer -----------------------------------------------------------------------
__global__ void k_adam(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, int64_t n, double lr, double bc1, double bc2) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  // fp64 math in the reference's evaluation order, no FMA contraction
  const double gg = static_cast<double>(g[i]);
  const double mm = __dadd_rn(__dmul_rn(b1, static_cast<double>(m[i])), __dmul_rn(1.0 - b1, gg));
  const double vv = __dadd_rn(__dmul_rn(b2, static_cast<double>(v[i])), __dmul_rn(__dmul_rn(1.0 - b2, gg), gg));
  m[i] = static_cast<float>(mm);
  v[i] = static_cast<float>(vv);
  const double step = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mm, bc1)), __dadd_rn(__dsqrt_rn(__ddiv_rn(vv, bc2)), eps));
  w[i] = __fsub_rn(w[i], static_cast<float>(step));
}

__global__ void k_sgd(float* __restrict__ w, const float* __restrict__ g, int64_t n, float lr) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) w[i] = __fsub_rn(w[i], __fmul_rn(lr, g[i]));
}

__global__ void k_scale(float* __restrict__ x, int64_t n, float s) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] *= s;
}

}  // namespace

void init_weight(Ctx& ctx, float* w, int64_t rows, int64_t cols, int64_t g_rows, int64_t g_cols,
                 int64_t r0, int64_t c0, uint64_t key) {
  if (rows * cols <= 0) return;
  const double lim = std::sqrt(6.0 / static_cast<double>(g_rows + g_cols));
  k_init_weight<<<nb(rows * cols), kT, 0, ctx.stream>>>(w, rows, cols, r0, c0, key, lim);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void fill(Ctx& ctx, float* x, int64_t n, float v) {
  if (n <= 0) return;
  k_fill<<<nb(n), kT, 0, ctx.stream>>>(x, n, v);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void weight_bf16(Ctx& ctx, const float* w, int64_t rows, int64_t cols, bf16* wb, int64_t ldb, bf16* wt,
                 bf16* wt_lo, int64_t ldt) {
  if (rows * cols <= 0) return;
  k_weight_bf16<<<nb(rows * cols), kT, 0, ctx.stream>>>(w, rows, cols, wb, ldb, wt, wt_lo, ldt);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void cast_bf16(Ctx& ctx, const float* x, int64_t rows, int64_t cols, int64_t ldx, bf16* y, int64_t ldy) {
  if (rows * cols <= 0) return;
  k_cast_rows<false><<<row_blocks(ctx, rows), kT, 0, ctx.stream>>>(x, rows, cols, ldx, y, nullptr, ldy);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void cast_split(Ctx& ctx, const float* x, int64_t rows, int64_t cols, int64_t ldx, bf16* hi, bf16* lo, int64_t ldy) {
  if (rows * cols <= 0) return;
  k_cast_rows<true><<<row_blocks(ctx, rows), kT, 0, ctx.stream>>>(x, rows, cols, ldx, hi, lo, ldy);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void add_inplace(Ctx& ctx, float* a, int64_t lda, const float* b, int64_t ldb, int64_t rows, int64_t cols) {
  if (rows * cols <= 0) return;
  k_add_rows<<<row_blocks(ctx, rows), kT, 0, ctx.stream>>>(a, lda, b, ldb, rows, cols);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void rowsumsq(Ctx& ctx, const float* x, int64_t ldx, int64_t rows, int64_t cols, float* ss) {
  if (rows <= 0) return;
  k_rowsumsq<<<nb(rows * 32), kT, 0, ctx.stream>>>(x, ldx, rows, cols, ss);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void reduce_rows(Ctx& ctx, const float* part, int parts, int64_t cols, float* out) {
  if (cols <= 0) return;
  k_reduce_rows<<<static_cast<unsigned>(ceil_div(cols, 32)), 1024, 0, ctx.stream>>>(part, parts, cols, out);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void ce_rowmax(Ctx& ctx, const CeArgs& p) {
  if (p.rows <= 0) return;
  k_ce_rowmax<<<nb(p.rows * 32), kT, 0, ctx.stream>>>(p);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}
void ce_rowsum(Ctx& ctx, const CeArgs& p) {
  if (p.rows <= 0) return;
  k_ce_rowsum<<<nb(p.rows * 32), kT, 0, ctx.stream>>>(p);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}
int ce_grad_blocks(int64_t rows) { return static_cast<int>(std::max<int64_t>(1, ceil_div(rows * 32, kT))); }
void ce_grad(Ctx& ctx, const CeArgs& p) {
  const int blocks = ce_grad_blocks(p.rows);
  if (p.rows > 0) {
    k_ce_grad<<<blocks, kT, 0, ctx.stream>>>(p);
    ctx.launches += 1;
  } else {
    GGB_CUDA(cudaMemsetAsync(p.loss_part, 0, sizeof(float), ctx.stream));
  }
  k_sum_parts<<<1, kT, 0, ctx.stream>>>(p.loss_part, p.rows > 0 ? blocks : 1, p.loss_acc);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}
void scale_scalar(Ctx& ctx, const float* in, float s, float* out) {
  k_scale_scalar<<<1, 1, 0, ctx.stream>>>(in, s, out);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void adam(Ctx& ctx, float* w, const float* g, float* m, float* v, int64_t n, double lr, double bc1,
          double bc2) {
  if (n <= 0) return;
  k_adam<<<nb(n), kT, 0, ctx.stream>>>(w, g, m, v, n, lr, bc1, bc2);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}
void sgd(Ctx& ctx, float* w, const float* g, int64_t n, float lr) {
  if (n <= 0) return;
  k_sgd<<<nb(n), kT, 0, ctx.stream>>>(w, g, n, lr);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}
void scale(Ctx& ctx, float* x, int64_t n, float s) {
  if (n <= 0) return;
  k_scale<<<nb(n), kT, 0, ctx.stream>>>(x, n, s);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

}  // namespace ggb
