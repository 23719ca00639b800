// Sparse aggregation H = A . F of the 3D-PMM layer (spmm, pmm.hpp:134-167)
// and its backward with the transposed block. Row-split CSR SpMM, HBM-bound:
// a group of LPR lanes owns one output row; each lane owns 8 consecutive
// feature columns (one 16-byte bf16 vector per nonzero), so a nonzero costs
// one fully used 16*LPR-byte gather. Column ids and values are fetched once
// per group with a coalesced load and broadcast by shuffles; eight gathers
// are kept in flight per lane. fp32 accumulation in CSR order.
#include "runtime.hpp"

namespace ggb {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 8;

// 8 consecutive feature values of one row: 16 B of bf16 or 32 B of fp32
template <class T>
struct Vec8;
template <>
struct Vec8<bf16> {
  uint4 u;
  __device__ __forceinline__ void load(const bf16* p) { u = __ldg(reinterpret_cast<const uint4*>(p)); }
  __device__ __forceinline__ void zero() { u = make_uint4(0, 0, 0, 0); }
  __device__ __forceinline__ void fma(float* acc, float v) const {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      acc[2 * i] = fmaf(v, f.x, acc[2 * i]);
      acc[2 * i + 1] = fmaf(v, f.y, acc[2 * i + 1]);
    }
  }
};
template <>
struct Vec8<float> {
  float4 a, b;
  __device__ __forceinline__ void load(const float* p) {
    a = __ldg(reinterpret_cast<const float4*>(p));
    b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  }
  __device__ __forceinline__ void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
  __device__ __forceinline__ void fma(float* acc, float v) const {
    acc[0] = fmaf(v, a.x, acc[0]); acc[1] = fmaf(v, a.y, acc[1]);
    acc[2] = fmaf(v, a.z, acc[2]); acc[3] = fmaf(v, a.w, acc[3]);
    acc[4] = fmaf(v, b.x, acc[4]); acc[5] = fmaf(v, b.y, acc[5]);
    acc[6] = fmaf(v, b.z, acc[6]); acc[7] = fmaf(v, b.w, acc[7]);
  }
};

__device__ __forceinline__ void store_bf16x8(bf16* dst, const float* v, bool full, int n) {
  if (full && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    uint32_t pk[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h2 = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      pk[i] = *reinterpret_cast<uint32_t*>(&h2);
    }
    *reinterpret_cast<uint4*>(dst) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  } else {
    for (int i = 0; i < 8 && i < n; ++i) dst[i] = __float2bfloat16_rn(v[i]);
  }
}

template <int LPR, class TIn>
__global__ void __launch_bounds__(kThreads, 3)
    k_spmm(int64_t rows, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
           const float* __restrict__ val, const TIn* __restrict__ F, int64_t ldf, int fcols,
           float* __restrict__ out, int64_t ldo, bf16* __restrict__ outb, bf16* __restrict__ outlo,
           int64_t ldob, int accumulate) {
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int g = lane / LPR, gl = lane % LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (g * LPR));
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t r = warp * RPW + g;
  if (r >= rows) return;  // whole groups leave together
  const int c0 = blockIdx.y * (LPR * 8) + gl * 8;
  const bool col_ok = c0 < fcols;
  const int64_t e0 = rp[r], e1 = rp[r + 1];
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
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
    // gathers in flight per lane: 8 x 16 B (bf16) or 4 x 32 B (fp32)
    constexpr int U = sizeof(TIn) == 2 ? kUnroll : kUnroll / 2;
    for (int kk = 0; kk < cnt; kk += U) {
      Vec8<TIn> fv[U];
      float vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int src = (kk + u) & (LPR - 1);
        const int ci = __shfl_sync(gmask, mc, src, LPR);
        const float v = __shfl_sync(gmask, mv, src, LPR);
        const bool ok = (kk + u) < cnt;
        vv[u] = ok ? v : 0.f;
        if (ok && col_ok)
          fv[u].load(Fc + static_cast<int64_t>(ci) * ldf);
        else
          fv[u].zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) fv[u].fma(acc, vv[u]);
    }
  }
  if (!col_ok) return;
  const bool full8 = c0 + 8 <= fcols;
  if (out) {
    float* dst = out + r * ldo + c0;
    if (full8 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
      float4* d4 = reinterpret_cast<float4*>(dst);
      if (accumulate) {
        const float4 a = d4[0], b = d4[1];
        acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
        acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
      }
      d4[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      d4[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    } else {
      for (int i = 0; i < 8 && c0 + i < fcols; ++i) {
        if (accumulate) acc[i] += dst[i];
        dst[i] = acc[i];
      }
    }
  }
  if (outb) store_bf16x8(outb + r * ldob + c0, acc, full8, fcols - c0);
  if (outlo) {  // residual of the bf16 rounding: acc == hi + lo to ~2^-16
    float lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) lo[i] = acc[i] - __bfloat162float(__float2bfloat16_rn(acc[i]));
    store_bf16x8(outlo + r * ldob + c0, lo, full8, fcols - c0);
  }
}

template <int LPR, class TIn>
void launch(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
            const TIn* f, int64_t ldf, int fcols, float* out, int64_t ldo, bf16* outb, bf16* outlo,
            int64_t ldob, int accumulate) {
  constexpr int RPB = (kThreads / 32) * (32 / LPR);
  dim3 grid(static_cast<unsigned>(ceil_div(rows, RPB)), static_cast<unsigned>(ceil_div(fcols, LPR * 8)));
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
  const int fc = static_cast<int>(fcols);
  if (fcols > 128)
    launch<32>(ctx, rows, rp, col, val, f, ldf, fc, out, ldo, outb, outlo, ldob, accumulate);
  else if (fcols > 64)
    launch<16>(ctx, rows, rp, col, val, f, ldf, fc, out, ldo, outb, outlo, ldob, accumulate);
  else if (fcols > 32)
    launch<8>(ctx, rows, rp, col, val, f, ldf, fc, out, ldo, outb, outlo, ldob, accumulate);
  else
    launch<4>(ctx, rows, rp, col, val, f, ldf, fc, out, ldo, outb, outlo, ldob, accumulate);
}

}  // namespace

void spmm_csr(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
              const bf16* f, int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* outb,
              int64_t ldob, int accumulate) {
  dispatch<bf16>(ctx, rows, rp, col, val, f, ldf, fcols, out, ldo, outb, nullptr, ldob, accumulate);
}

void spmm_csr_f32(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
                  const float* f, int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* out_hi,
                  bf16* out_lo, int64_t ldob, int accumulate) {
  dispatch<float>(ctx, rows, rp, col, val, f, ldf, fcols, out, ldo, out_hi, out_lo, ldob, accumulate);
}

}  // namespace ggb
