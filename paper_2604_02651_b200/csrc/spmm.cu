// Sparse aggregation H = A . F of the 3D-PMM layer (spmm, pmm.hpp:134-167)
// and its backward with the transposed block. Row-split CSR SpMM, HBM-bound:
// a group of LPR lanes owns one output row and each lane owns 32 bytes of
// every gathered feature row (16 bf16 or 8 fp32 columns, two 16-byte
// vector loads), so one warp-wide load instruction moves 1 KB of useful
// data. Column ids and values are fetched once per group with a coalesced
// load and broadcast by shuffles; several gathers are kept in flight per
// lane. fp32 accumulation in CSR order.
#include <cstdlib>

#include "runtime.hpp"

namespace ggb {
namespace {

constexpr int kThreads = 256;
constexpr int kInFlight = 4;  // gathered rows in flight per lane

// N consecutive feature values of one row = 32 bytes (2 x 16-byte loads)
template <class T>
struct Vec32B;
template <>
struct Vec32B<bf16> {
  static constexpr int N = 16;
  uint4 a, b;
  __device__ __forceinline__ void load(const bf16* p) {
    a = __ldg(reinterpret_cast<const uint4*>(p));
    b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
  }
  __device__ __forceinline__ void load_half(const bf16* p) {  // only the first 8 columns exist
    a = __ldg(reinterpret_cast<const uint4*>(p));
    b = make_uint4(0, 0, 0, 0);
  }
  __device__ __forceinline__ void zero() { a = b = make_uint4(0, 0, 0, 0); }
  __device__ __forceinline__ void fma(float* acc, float v) const {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* g = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      acc[2 * i] = fmaf(v, f.x, acc[2 * i]);
      acc[2 * i + 1] = fmaf(v, f.y, acc[2 * i + 1]);
      const float2 e = __bfloat1622float2(g[i]);
      acc[8 + 2 * i] = fmaf(v, e.x, acc[8 + 2 * i]);
      acc[8 + 2 * i + 1] = fmaf(v, e.y, acc[8 + 2 * i + 1]);
    }
  }
};
template <>
struct Vec32B<float> {
  static constexpr int N = 8;
  float4 a, b;
  __device__ __forceinline__ void load(const float* p) {
    a = __ldg(reinterpret_cast<const float4*>(p));
    b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  }
  __device__ __forceinline__ void load_half(const float* p) {  // only the first 4 columns exist
    a = __ldg(reinterpret_cast<const float4*>(p));
    b = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ __forceinline__ void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ __forceinline__ void fma(float* acc, float v) const {
    acc[0] = fmaf(v, a.x, acc[0]); acc[1] = fmaf(v, a.y, acc[1]);
    acc[2] = fmaf(v, a.z, acc[2]); acc[3] = fmaf(v, a.w, acc[3]);
    acc[4] = fmaf(v, b.x, acc[4]); acc[5] = fmaf(v, b.y, acc[5]);
    acc[6] = fmaf(v, b.z, acc[6]); acc[7] = fmaf(v, b.w, acc[7]);
  }
};

template <int N>
__device__ __forceinline__ void store_bf16(bf16* dst, const float* v, int n) {
  if (n >= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < N / 8; ++q) {
      uint32_t pk[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * q + 2 * i], v[8 * q + 2 * i + 1]);
        pk[i] = *reinterpret_cast<uint32_t*>(&h2);
      }
      reinterpret_cast<uint4*>(dst)[q] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  } else {
    for (int i = 0; i < N && i < n; ++i) dst[i] = __float2bfloat16_rn(v[i]);
  }
}

template <int LPR, class TIn>
__global__ void __launch_bounds__(kThreads, 3)
    k_spmm(int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
           const float* __restrict__ val, const TIn* __restrict__ F, int64_t ldf, int fcols,
           float* __restrict__ out, int64_t ldo, bf16* __restrict__ outb, bf16* __restrict__ outlo,
           int64_t ldob, int accumulate) {
  using V = Vec32B<TIn>;
  constexpr int N = V::N;
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int g = lane / LPR, gl = lane % LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t r = warp * RPW + g;
  if (r >= rows) return;  // whole groups leave together
  const int c0 = blockIdx.y * (LPR * N) + gl * N;
  const int ncol = fcols - c0;  // valid columns of this lane (may be <= 0 or < N)
  // storage is padded to 8 elements: a lane whose tail holds < N/2 valid
  // columns only reads its first half
  const bool full = ncol > N / 2;
  const bool any = ncol > 0;
  const int64_t e0 = rp[r], e1 = rp[r + 1];
  float acc[N];
#pragma unroll
  for (int i = 0; i < N; ++i) acc[i] = 0.f;
  const TIn* Fc = F + c0;
  for (int64_t e = e0; e < e1; e += LPR) {
    const int64_t k = e + gl;
    int32_t mc = 0;
    float mv = 0.f;
    if (k < e1) {
      mc = __ldg(col + k);
      mv = __ldg(val + k);
    }
    const int cnt = static_cast<int>(e1 - e < LPR ? e1 - e : LPR);
    for (int kk = 0; kk < cnt; kk += kInFlight) {
      V fv[kInFlight];
      float vv[kInFlight];
#pragma unroll
      for (int u = 0; u < kInFlight; ++u) {
        const int src = (kk + u) & (LPR - 1);
        const int ci = __shfl_sync(gmask, mc, src, LPR);
        const float v = __shfl_sync(gmask, mv, src, LPR);
        const bool ok = (kk + u) < cnt;
        vv[u] = ok ? v : 0.f;
        const TIn* p = Fc + static_cast<int64_t>(ci) * ldf;
        if (ok && full)
          fv[u].load(p);
        else if (ok && any)
          fv[u].load_half(p);
        else
          fv[u].zero();
      }
#pragma unroll
      for (int u = 0; u < kInFlight; ++u) fv[u].fma(acc, vv[u]);
    }
  }
  if (!any) return;
  if (out) {
    float* dst = out + r * ldo + c0;
    if (ncol >= N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int q = 0; q < N / 4; ++q) {
        if (accumulate) {
          const float4 a = d4[q];
          acc[4 * q] += a.x;
          acc[4 * q + 1] += a.y;
          acc[4 * q + 2] += a.z;
          acc[4 * q + 3] += a.w;
        }
        d4[q] = make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
      }
    } else {
      for (int i = 0; i < N && i < ncol; ++i) {
        if (accumulate) acc[i] += dst[i];
        dst[i] = acc[i];
      }
    }
  }
  if (outb) store_bf16<N>(outb + r * ldob + c0, acc, ncol);
  if (outlo) {  // residual of the bf16 rounding: acc == hi + lo to ~2^-16
    float lo[N];
#pragma unroll
    for (int i = 0; i < N; ++i) lo[i] = acc[i] - __bfloat162float(__float2bfloat16_rn(acc[i]));
    store_bf16<N>(outlo + r * ldob + c0, lo, ncol);
  }
}

template <int LPR, class TIn>
void launch(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
            const TIn* f, int64_t ldf, int fcols, float* out, int64_t ldo, bf16* outb, bf16* outlo,
            int64_t ldob, int accumulate) {
  constexpr int N = Vec32B<TIn>::N;
  constexpr int RPB = (kThreads / 32) * (32 / LPR);
  dim3 grid(static_cast<unsigned>(ceil_div(rows, RPB)), static_cast<unsigned>(ceil_div(fcols, LPR * N)));
  k_spmm<LPR, TIn><<<grid, kThreads, 0, ctx.stream>>>(rows, rp, col, val, f, ldf, fcols, out, ldo, outb,
                                                      outlo, ldob, accumulate);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

template <class TIn>
void dispatch(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val, const TIn* f,
              int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* outb, bf16* outlo, int64_t ldob,
              int accumulate) {
  if (rows <= 0 || fcols <= 0) return;
  require(ldf % 8 == 0 && (reinterpret_cast<uintptr_t>(f) & 15) == 0,
          "spmm: feature operand needs 16-byte aligned rows of 8-element multiples");
  require(!(accumulate && !out), "spmm: accumulate needs an fp32 output");
  constexpr int N = Vec32B<TIn>::N;
  const int fc = static_cast<int>(fcols);
  const int64_t lanes = ceil_div(fcols, N);  // lanes needed for the row
  if (lanes > 16)
    launch<32>(ctx, rows, rp, col, val, f, ldf, fc, out, ldo, outb, outlo, ldob, accumulate);
  else if (lanes > 8)
    launch<16>(ctx, rows, rp, col, val, f, ldf, fc, out, ldo, outb, outlo, ldob, accumulate);
  else if (lanes > 4)
    launch<8>(ctx, rows, rp, col, val, f, ldf, fc, out, ldo, outb, outlo, ldob, accumulate);
  else
    launch<4>(ctx, rows, rp, col, val, f, ldf, fc, out, ldo, outb, outlo, ldob, accumulate);
}

}  // namespace

bool spmm_pipe(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val, const void* f,
               int esize, int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* outb, bf16* outlo, int64_t ldob,
               int accumulate);

int spmm_kernel_choice() {  // GGB_SPMM=rowsplit forces the register-pipelined kernel
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("GGB_SPMM");
    v = (e && std::string(e) == "rowsplit") ? 1 : 0;
  }
  return v;
}

// the non-pipelined kernels do not mirror their stores (push mode): copy the
// finished block to the mirror instead
void mirror_copy(Ctx& ctx, int64_t rows, int64_t fcols, float* out, int64_t ldo, bf16* outb, int64_t ldob) {
  if (!ctx.out_mirror) return;
  if (out)
    GGB_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(out) + ctx.out_mirror, ldo * 4, out, ldo * 4, fcols * 4, rows,
                               cudaMemcpyDeviceToDevice, ctx.stream));
  if (outb)
    GGB_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(outb) + ctx.out_mirror, ldob * 2, outb, ldob * 2, fcols * 2,
                               rows, cudaMemcpyDeviceToDevice, ctx.stream));
}

void spmm_csr(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
              const bf16* f, int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* outb,
              int64_t ldob, int accumulate) {
  if (rows <= 0 || fcols <= 0) return;
  require(!(accumulate && !out), "spmm: accumulate needs an fp32 output");
  require(ldf % 8 == 0 && (reinterpret_cast<uintptr_t>(f) & 15) == 0,
          "spmm: feature operand needs 16-byte aligned rows of 8-element multiples");
  if (spmm_kernel_choice() == 0 && !ctx.side_stream &&
      spmm_pipe(ctx, rows, rp, col, val, f, 2, ldf, fcols, out, ldo, outb, nullptr, ldob, accumulate))
    return;
  dispatch<bf16>(ctx, rows, rp, col, val, f, ldf, fcols, out, ldo, outb, nullptr, ldob, accumulate);
  mirror_copy(ctx, rows, fcols, out, ldo, outb, ldob);
}

void spmm_csr_f32(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
                  const float* f, int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* out_hi,
                  bf16* out_lo, int64_t ldob, int accumulate) {
  if (rows <= 0 || fcols <= 0) return;
  require(!(accumulate && !out), "spmm: accumulate needs an fp32 output");
  require(ldf % 8 == 0 && (reinterpret_cast<uintptr_t>(f) & 15) == 0,
          "spmm: feature operand needs 16-byte aligned rows of 8-element multiples");
  if (spmm_kernel_choice() == 0 && !ctx.side_stream &&
      spmm_pipe(ctx, rows, rp, col, val, f, 4, ldf, fcols, out, ldo, out_hi, out_lo, ldob, accumulate))
    return;
  dispatch<float>(ctx, rows, rp, col, val, f, ldf, fcols, out, ldo, out_hi, out_lo, ldob, accumulate);
  mirror_copy(ctx, rows, fcols, out, ldo, out_hi, ldob);
}

}  // namespace ggb
