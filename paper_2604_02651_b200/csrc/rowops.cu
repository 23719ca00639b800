// Warp-per-row kernels of the layer's normalization / activation path, fully
// vectorized (one float4 per lane per 128-column chunk) and fused across the
// reference's separate passes when the whole row is local to the rank:
//   forward  : row sum of squares + RMSNorm apply + ReLU + dropout + residual
//              (parallel_rmsnorm_fwd pmm.hpp:214-243 + fused_elementwise_fwd
//              pmm.hpp:299-328) in one read of xw and the residual;
//   backward : fused_elementwise_bwd (pmm.hpp:331-341) + parallel_rmsnorm_bwd
//              (pmm.hpp:251-287) with the row dot product, dx and the dgamma
//              column partials in one read of dy and xw;
//   loss     : parallel_cross_entropy (pmm.hpp:352-401) max / sum-exp /
//              gradient in one pass over the logits row.
// When the row is split over the grid's column axis the same kernels run in
// two phases around the fp32 all-reduce of the row statistic.
#include <algorithm>
#include <cstdlib>

#include "ops.hpp"
#include "rng.cuh"

namespace ggb {
namespace {

constexpr int kT = 256;
constexpr int kRowsPerBlock = kT / 32;
constexpr int kMaxJ = 4;  // rows up to 512 local columns

__device__ __forceinline__ float warp_sum(float s) {
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}
__device__ __forceinline__ float warp_max(float s) {
#pragma unroll
  for (int o = 16; o; o >>= 1) s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
  return s;
}

// 4 consecutive floats at column c of a row with n valid columns (c % 4 == 0)
__device__ __forceinline__ float4 ld4(const float* row, int64_t c, int64_t n) {
  if (c + 4 <= n) return *reinterpret_cast<const float4*>(row + c);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < n) v.x = row[c];
  if (c + 1 < n) v.y = row[c + 1];
  if (c + 2 < n) v.z = row[c + 2];
  if (c + 3 < n) v.w = row[c + 3];
  return v;
}
__device__ __forceinline__ void st4(float* row, int64_t c, int64_t n, const float* v) {
  if (c + 4 <= n) {
    *reinterpret_cast<float4*>(row + c) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    for (int i = 0; i < 4 && c + i < n; ++i) row[c + i] = v[i];
  }
}
__device__ __forceinline__ void st4_bf16(bf16* row, int64_t c, int64_t n, const float* v) {
  if (c + 4 <= n) {
    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(row + c) = u;
  } else {
    for (int i = 0; i < 4 && c + i < n; ++i) row[c + i] = __float2bfloat16_rn(v[i]);
  }
}
// fp32 -> 24 bits (round to nearest even at bit 8): the P24 gather format
__device__ __forceinline__ uint32_t round24(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b + 0x7fu + ((b >> 8) & 1u)) & 0xffffff00u;
}
__device__ __forceinline__ void st4_p24(uint8_t* row, int64_t hoff, int64_t c, int64_t n, const float* v) {
  uint32_t r[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) r[i] = round24(v[i]);
  if (c + 4 <= n) {
    *reinterpret_cast<uint2*>(row + 2 * c) = make_uint2(__byte_perm(r[0], r[1], 0x7632), __byte_perm(r[2], r[3], 0x7632));
    *reinterpret_cast<uint32_t*>(row + hoff + c) =
        __byte_perm(__byte_perm(r[0], r[1], 0x0051), __byte_perm(r[2], r[3], 0x0051), 0x5410);
  } else {
    for (int i = 0; i < 4 && c + i < n; ++i) {
      reinterpret_cast<uint16_t*>(row)[c + i] = static_cast<uint16_t>(r[i] >> 16);
      row[hoff + c + i] = static_cast<uint8_t>(r[i] >> 8);
    }
  }
}
// 4 consecutive values at column c of a 24-bit row (st4_p24's layout)
__device__ __forceinline__ float4 ld4_p24(const uint8_t* row, int64_t hoff, int64_t c, int64_t n) {
  if (c + 4 <= n) {
    const uint2 h = *reinterpret_cast<const uint2*>(row + 2 * c);
    const uint32_t l = *reinterpret_cast<const uint32_t*>(row + hoff + c);
    return make_float4(__uint_as_float((h.x << 16) | ((l & 0xffu) << 8)),
                       __uint_as_float((h.x & 0xffff0000u) | (l & 0xff00u)),
                       __uint_as_float((h.y << 16) | ((l >> 8) & 0xff00u)),
                       __uint_as_float((h.y & 0xffff0000u) | ((l >> 16) & 0xff00u)));
  }
  float v[4] = {0.f, 0.f, 0.f, 0.f};
  for (int i = 0; i < 4 && c + i < n; ++i)
    v[i] = __uint_as_float((static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(row)[c + i]) << 16) |
                           (static_cast<uint32_t>(row[hoff + c + i]) << 8));
  return make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void f4(const float4& a, float* v) {
  v[0] = a.x;
  v[1] = a.y;
  v[2] = a.z;
  v[3] = a.w;
}

// chunks of 128 columns held per row; Full: cols == 128 J; kLayer: the layer
// API's instance (RMSNorm without ReLU, optional mask output)
// kPipe: a capped grid whose warps stride over the rows with the next row's
// loads issued before the current row is processed (the prologue — gamma,
// the column-term table — is paid once per warp instead of once per row)
// TPB: threads per block (rows per block = TPB / 32; the per-block column
// term table and barrier are shared by more rows at 512)
template <int J, bool Full, bool kLayer, bool kPipe = false, int TPB = kT>
__global__ void __launch_bounds__(TPB) k_fwd_row(FwdApply p) {
  constexpr int kRowsPerBlock = TPB / 32;
  // Warp per row (grid-stride, so a capped grid also works), gamma and the
  // per-lane constants held across rows.
  const int64_t ncols = Full ? static_cast<int64_t>(J) * kRowChunk : p.cols;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nj = Full ? J : static_cast<int>((p.cols + kRowChunk - 1) / kRowChunk);
  const int64_t w0 = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + wib;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kRowsPerBlock;
  float g[J][4];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    if (j >= nj) break;
    if (p.gamma)
      f4(ld4(p.gamma, j * kRowChunk + 4 * lane, ncols), g[j]);
    else
      g[j][0] = g[j][1] = g[j][2] = g[j][3] = 1.f;
  }
  const uint32_t lt = (1u << lane) - 1u;
  const float sc_on = p.drop ? p.keep_scale : 1.f;
  const bool hash = p.drop && !p.keep;
  // row's ReLU-active columns (compacted), and one keep byte per column
  __shared__ uint16_t s_list[kRowsPerBlock][32 * 4 * J];
  __shared__ __align__(16) uint8_t s_kb[kRowsPerBlock][kRowChunk * J];
  __shared__ uint64_t s_cj[kRowChunk * J];  // column_term of every local column
  if (hash) {
    for (int c = threadIdx.x; c < kRowChunk * J; c += TPB) s_cj[c] = column_term(static_cast<uint64_t>(p.col_g0 + c));
    __syncthreads();
  }
  const uint64_t T = p.thresh << 11;

  // every load of a row is issued up front: one memory round trip per row
  auto load_row = [&](int64_t r, float (&x)[J][4], float (&res)[J][4]) {
    const float* xr = p.x + r * p.ldx;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (j >= nj) break;
      const int64_t c = j * kRowChunk + 4 * lane;
      f4(ld4(xr, c, ncols), x[j]);
      if (p.res)
        f4(ld4(p.res + r * p.ldres, c, ncols), res[j]);
      else if (p.resp)
        f4(ld4_p24(p.resp + r * p.ldresp, p.reshoff, c, ncols), res[j]);
      else
        res[j][0] = res[j][1] = res[j][2] = res[j][3] = 0.f;
    }
  };
  float xn[J][4], rn[J][4];
  if (kPipe && w0 < p.rows) load_row(w0, xn, rn);

#pragma unroll 1
  for (int64_t r = w0; r < p.rows; r += nw) {
    float x[J][4], res[J][4];
    if constexpr (kPipe) {
#pragma unroll
      for (int j = 0; j < J; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) x[j][i] = xn[j][i], res[j][i] = rn[j][i];
      if (r + nw < p.rows) load_row(r + nw, xn, rn);
    } else {
      load_row(r, x, res);
    }
    float inv = 1.f;
    if (p.gamma) {  // RMSNorm on
      float ss;
      if (p.fuse_ss) {
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < J; ++j)
          if (j < nj)
#pragma unroll
            for (int i = 0; i < 4; ++i) s = fmaf(x[j][i], x[j][i], s);
        ss = warp_sum(s);
      } else {
        ss = p.ss[r];
      }
      const float rms = sqrtf(ss / p.d + p.eps);
      inv = 1.f / rms;
      if (lane == 0 && p.rms) p.rms[r] = rms;
    }
    // y = gamma * x / rms; bit 4j+i of posm: y > 0 and the column exists
    float y[J][4];
    uint32_t posm = 0;
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (j >= nj) break;
      const int64_t c = j * kRowChunk + 4 * lane;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        y[j][i] = p.gamma ? g[j][i] * x[j][i] * inv : x[j][i];
        if (((kLayer && p.no_relu) || y[j][i] > 0.f) && (Full || c + i < ncols)) posm |= 1u << (4 * j + i);
      }
    }
    uint32_t keepm = posm;
    if (p.drop && p.keep) {  // precomputed keep-bits (prefetcher)
      uint32_t kb = 0;
#pragma unroll
      for (int j = 0; j < J; ++j)
        if (j < nj)
#pragma unroll
          for (int i = 0; i < 4; ++i) kb |= ((p.keep[r * p.ldm + 4 * j + i] >> lane) & 1u) << (4 * j + i);
      keepm = posm & kb;
    } else if (hash) {
      // only ReLU-active elements need the dropout hash: the warp lists them
      // (per-slot ballots give each its list index) and every lane hashes an
      // equal share; the hashing lane writes the element's keep byte
      int total = 0;
#pragma unroll
      for (int sl = 0; sl < 4 * J; ++sl) {
        const bool on = (posm >> sl) & 1u;
        const uint32_t bl = __ballot_sync(0xffffffffu, on);
        if (on) s_list[wib][total + __popc(bl & lt)] = static_cast<uint16_t>((sl >> 2) * kRowChunk + 4 * lane + (sl & 3));
        total += __popc(bl);
      }
      __syncwarp();
      const uint64_t row_key = hash_combine(p.mask_key, static_cast<uint64_t>(p.row_g0 + r));
      for (int k = lane; k < total; k += 32) {
        const int col = s_list[wib][k];
        s_kb[wib][col] = element_keep_cj(row_key, s_cj[col], T) ? 1 : 0;
      }
      __syncwarp();
      // the lane's 4 keep bytes per chunk in one load (bytes of inactive
      // columns are stale and masked by posm)
      uint32_t kb = 0;
#pragma unroll
      for (int j = 0; j < J; ++j)
        if (j < nj) {
          const uint32_t w4 = *reinterpret_cast<const uint32_t*>(&s_kb[wib][j * kRowChunk + 4 * lane]);
          kb |= ((w4 & 1u) | ((w4 >> 7) & 2u) | ((w4 >> 14) & 4u) | ((w4 >> 21) & 8u)) << (4 * j);
        }
      keepm = posm & kb;
      __syncwarp();  // s_list / s_kb are rewritten by the next row
    }
    uint32_t myword = 0;  // lane s < 4 nj stores keep word s of the row
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (j >= nj) break;
      const int64_t c = j * kRowChunk + 4 * lane;
      float o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool on = (keepm >> (4 * j + i)) & 1u;
        const uint32_t bits = __ballot_sync(0xffffffffu, on);
        if (lane == 4 * j + i) myword = bits;
        o[i] = y[j][i] * (on ? sc_on : 0.f) + res[j][i];
      }
      if (p.out) st4(p.out + r * p.ldo, c, ncols, o);
      if (p.outp) st4_p24(p.outp + r * p.ldp, p.hoff, c, ncols, o);
      if (p.outb) {
        st4_bf16(p.outb + r * p.ldob, c, ncols, o);
        if (p.outlo) {
          float lo[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) lo[i] = o[i] - __bfloat162float(__float2bfloat16_rn(o[i]));
          st4_bf16(p.outlo + r * p.ldob, c, ncols, lo);
        }
      }
    }
    if ((!kLayer || p.mask) && lane < 4 * nj) p.mask[r * p.ldm + lane] = myword;
  }
}

// Dropout keep-bits element_unit(key, row, col) >= rate (pmm.hpp:317-322) of
// a block, in the row-kernel layout: one thread per (row, word), word 4j+i
// holding bit l for column 128j + 4l + i. Pure integer work, independent of
// the activations, so the prefetcher runs it ahead on its own stream.
__global__ void __launch_bounds__(128) k_dropout_keep(uint64_t key, int64_t rows, int64_t cols, int64_t row_g0,
                                                      int64_t col_g0, uint64_t thresh, uint32_t* __restrict__ out,
                                                      int64_t ldm) {
  // grid-stride over a small persistent grid: the kernel runs beside the
  // training stream and must leave room for its CTAs
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < rows * ldm;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
  const int64_t r = t / ldm, w = t % ldm;
  const int64_t j = w / 4, i = w % 4;
  const uint64_t row_key = hash_combine(key, static_cast<uint64_t>(row_g0 + r));
  uint32_t bits = 0;
#pragma unroll 4
  for (int l = 0; l < 32; ++l) {
    const int64_t c = j * kRowChunk + 4 * l + i;
    if (c < cols && element_keep_cj(row_key, column_term(static_cast<uint64_t>(col_g0 + c)), thresh << 11))
      bits |= 1u << l;
  }
  out[t] = bits;
  }
}

// Row dot product s_r = sum_j dxn * gamma * x (the all-reduced input of the
// split-row backward).
__global__ void __launch_bounds__(kT) k_bwd_row_stats(BwdApply p) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + (threadIdx.x >> 5);
  if (r >= p.rows) return;
  const int nj = static_cast<int>((p.cols + kRowChunk - 1) / kRowChunk);
  float s = 0.f;
  for (int j = 0; j < nj; ++j) {
    const int64_t c = j * kRowChunk + 4 * lane;
    float dy[4], x[4], g[4];
    f4(ld4(p.dy + r * p.lddy, c, p.cols), dy);
    f4(ld4(p.x + r * p.ldx, c, p.cols), x);
    f4(ld4(p.gamma, c, p.cols), g);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool keep = !p.mask || ((p.mask[r * p.ldm + 4 * j + i] >> lane) & 1u);
      const float dxn = keep ? dy[i] * p.keep_scale : 0.f;
      s += dxn * g[i] * x[i];
    }
  }
  s = warp_sum(s);
  if (lane == 0) p.s[r] = s;
}

// dx = gamma*dxn/r - x*s/(d r^3) (bf16 out); dgamma_j += dxn*x/r accumulated
// per lane over the block's rows (grid-stride), then reduced across the
// block's warps into dgamma_part[block][cols].
// kLayer: the layer API's parallel_rmsnorm_bwd / element-wise backward
// (fp32 dx, optional mask); the training step's instance (bf16 dx, mask
// always present) keeps its own code generation.
template <int J, bool kLayer>
__global__ void __launch_bounds__(kT, J <= 2 ? 4 : 2) k_bwd_row(BwdApply p) {
  constexpr int kMaxJ = J;
  __shared__ float sh[kRowsPerBlock][kMaxJ * kRowChunk];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nj = static_cast<int>((p.cols + kRowChunk - 1) / kRowChunk);
  float dg[kMaxJ][4];
#pragma unroll
  for (int j = 0; j < kMaxJ; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) dg[j][i] = 0.f;
  // narrow rows: two rows per iteration (both rows' loads issued before either
  // row's reductions) to double the warp's memory-level parallelism; wider
  // rows already hold enough loads in flight and need the registers for
  // occupancy
  constexpr int R = J == 1 ? 2 : 1;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kRowsPerBlock;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + wib; r0 < p.rows; r0 += R * stride) {
    float dxr[R][kMaxJ][4], xr[R][kMaxJ][4];
#pragma unroll
    for (int h = 0; h < R; ++h) {
      const int64_t r = r0 + h * stride;
      if (r >= p.rows) break;
      const uint32_t* mrow = (!kLayer || p.mask) ? p.mask + r * p.ldm : nullptr;
#pragma unroll
      for (int j = 0; j < kMaxJ; ++j) {
        if (j >= nj) break;
        const int64_t c = j * kRowChunk + 4 * lane;
        float dy[4];
        f4(ld4(p.dy + r * p.lddy, c, p.cols), dy);
        f4(ld4(p.x + r * p.ldx, c, p.cols), xr[h][j]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          dxr[h][j][i] = ((kLayer && !mrow) || ((mrow[4 * j + i] >> lane) & 1u)) ? dy[i] * p.keep_scale : 0.f;
      }
    }
#pragma unroll
    for (int h = 0; h < R; ++h) {
    const int64_t r = r0 + h * stride;
    if (r >= p.rows) break;
    float(&dxn)[kMaxJ][4] = dxr[h];
    float(&x)[kMaxJ][4] = xr[h];
    float inv = 1.f, coef = 0.f;
    if (p.rms) {
      float s;
      if (p.fuse_s) {
        float a = 0.f;
#pragma unroll
        for (int j = 0; j < kMaxJ; ++j) {
          if (j >= nj) break;
          float g[4];
          f4(ld4(p.gamma, j * kRowChunk + 4 * lane, p.cols), g);
#pragma unroll
          for (int i = 0; i < 4; ++i) a += dxn[j][i] * g[i] * x[j][i];
        }
        s = warp_sum(a);
      } else {
        s = p.s[r];
      }
      const float rr = p.rms[r];
      inv = 1.f / rr;
      coef = s / (p.d * rr * rr * rr);
    }
#pragma unroll
    for (int j = 0; j < kMaxJ; ++j) {
      if (j >= nj) break;
      const int64_t c = j * kRowChunk + 4 * lane;
      float dx[4];
      if (p.rms) {
        float g[4];
        f4(ld4(p.gamma, c, p.cols), g);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          dx[i] = g[i] * dxn[j][i] * inv - x[j][i] * coef;
          dg[j][i] += dxn[j][i] * x[j][i] * inv;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) dx[i] = dxn[j][i];
      }
      if constexpr (kLayer)
        st4(p.dxf + r * p.lddxf, c, p.cols, dx);
      else
        st4_bf16(p.dxb + r * p.lddxb, c, p.cols, dx);
    }
    }
  }
  if (!p.dgamma_part) return;
#pragma unroll
  for (int j = 0; j < kMaxJ; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) sh[wib][j * kRowChunk + 4 * lane + i] = dg[j][i];
  __syncthreads();
  for (int64_t c = threadIdx.x; c < p.cols; c += kT) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < kRowsPerBlock; ++k) s += sh[k][c];
    p.dgamma_part[static_cast<int64_t>(blockIdx.x) * p.cols + c] = s;
  }
}

// Cross-entropy in one pass per row (class block fully local): row max,
// sum of exp, label logit, per-row loss, gradient (softmax - onehot) / B.
__global__ void __launch_bounds__(kT) k_ce_row(CeArgs p) {
  __shared__ float part[kRowsPerBlock];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + wib;
  float contrib = 0.f;
  if (r < p.rows) {
    const float* lr = p.logits + r * p.ld;
    float m = -3.402823466e38f;
    for (int64_t j = lane; j < p.cols; j += 32) m = fmaxf(m, lr[j]);
    m = warp_max(m);
    float z = 0.f;
    for (int64_t j = lane; j < p.cols; j += 32) z += expf(lr[j] - m);
    z = warp_sum(z);
    const int64_t y = p.labels[p.row_g0 + r];
    for (int64_t j = lane; j < p.cols; j += 32) {
      float g = expf(lr[j] - m) / z;
      if (p.c0 + j == y) g -= 1.f;
      const float d = g * p.invb;
      if (p.dlog) p.dlog[r * p.lddlog + j] = d;
      if (p.dlogb) p.dlogb[r * p.lddlogb + j] = __float2bfloat16_rn(d);
    }
    const float zy = (y >= p.c0 && y < p.c0 + p.cols) ? lr[y - p.c0] : 0.f;
    contrib = (m + logf(z)) - zy;
  }
  if (lane == 0) part[wib] = contrib;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int k = 0; k < kRowsPerBlock; ++k) s += part[k];
    p.loss_part[blockIdx.x] = s;
  }
}

// Register-resident variant for narrow class blocks: LPR lanes per row (32/LPR
// rows per warp), VPL logits per lane, one global read of the row.
template <int LPR, int VPL>
__global__ void __launch_bounds__(kT) k_ce_row_reg(CeArgs p) {
  constexpr int RPW = 32 / LPR;
  __shared__ float part[kRowsPerBlock];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, gl = lane % LPR;
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * kRowsPerBlock + wib) * RPW + lane / LPR;
  const bool ok = r < p.rows;
  float v[VPL];
  float m = -3.402823466e38f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int64_t j = gl + static_cast<int64_t>(LPR) * k;
    v[k] = (ok && j < p.cols) ? p.logits[r * p.ld + j] : -3.402823466e38f;
    m = fmaxf(m, v[k]);
  }
#pragma unroll
  for (int o = LPR / 2; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float z = 0.f;
#pragma unroll
  for (int k = 0; k < VPL; ++k) {
    const int64_t j = gl + static_cast<int64_t>(LPR) * k;
    v[k] = (ok && j < p.cols) ? expf(v[k] - m) : 0.f;
    z += v[k];
  }
#pragma unroll
  for (int o = LPR / 2; o; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  float contrib = 0.f;
  if (ok) {
    const int64_t y = p.labels[p.row_g0 + r];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      const int64_t j = gl + static_cast<int64_t>(LPR) * k;
      if (j >= p.cols) continue;
      float g = v[k] / z;
      if (p.c0 + j == y) g -= 1.f;
      const float d = g * p.invb;
      if (p.dlog) p.dlog[r * p.lddlog + j] = d;
      if (p.dlogb) p.dlogb[r * p.lddlogb + j] = __float2bfloat16_rn(d);
    }
    if (gl == 0) {
      const float zy = (y >= p.c0 && y < p.c0 + p.cols) ? p.logits[r * p.ld + (y - p.c0)] : 0.f;
      contrib = (m + logf(z)) - zy;
    }
  }
  // warp total of the row contributions (lanes gl == 0 hold them)
#pragma unroll
  for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
  if (lane == 0) part[wib] = contrib;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int k = 0; k < kRowsPerBlock; ++k) s += part[k];
    p.loss_part[blockIdx.x] = s;
  }
}

__global__ void k_sum_parts_row(const float* __restrict__ part, int64_t n, float* __restrict__ out) {
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

inline unsigned row_blocks(int64_t rows) { return static_cast<unsigned>(ceil_div(rows, kRowsPerBlock)); }

}  // namespace

template <int J, bool Full, bool kLayer>
void launch_fwd_row_k(Ctx& ctx, const FwdApply& p) {
  // a warp per row: the row's load latency is hidden by the other resident
  // warps rather than by a software pipeline. GGB_FWD_ROW_BPS=b caps the grid
  // at b blocks per SM striding over the rows (measured slower: 4 -> 1.76
  // ms/step, 8 -> 1.66, one warp per row 1.58)
  static const int bps = [] {
    const char* e = std::getenv("GGB_FWD_ROW_BPS");
    return e ? std::atoi(e) : 0;
  }();
  // GGB_FWD_ROW_PIPE=b: b blocks per SM, warps stride with the next row's
  // loads in flight (software pipeline)
  static const int pipe = [] {
    const char* e = std::getenv("GGB_FWD_ROW_PIPE");
    return e ? std::atoi(e) : 0;
  }();
  int64_t g = ceil_div(p.rows, kRowsPerBlock);
  if (pipe > 0 && !kLayer) {
    g = std::min<int64_t>(g, static_cast<int64_t>(pipe) * ctx.num_sms);
    k_fwd_row<J, Full, kLayer, true><<<static_cast<unsigned>(std::max<int64_t>(1, g)), kT, 0, ctx.stream>>>(p);
    return;
  }
  // GGB_FWD_ROW_TPB=512: 16 rows per block
  static const int tpb = [] {
    const char* e = std::getenv("GGB_FWD_ROW_TPB");
    return e && std::atoi(e) == 512 ? 512 : 256;
  }();
  if (tpb == 512 && !kLayer && bps == 0) {
    k_fwd_row<J, Full, kLayer, false, 512>
        <<<static_cast<unsigned>(std::max<int64_t>(1, ceil_div(p.rows, 16))), 512, 0, ctx.stream>>>(p);
    return;
  }
  if (bps > 0) g = std::min<int64_t>(g, static_cast<int64_t>(bps) * ctx.num_sms);
  k_fwd_row<J, Full, kLayer><<<static_cast<unsigned>(std::max<int64_t>(1, g)), kT, 0, ctx.stream>>>(p);
}

template <int J, bool Full>
void launch_fwd_row(Ctx& ctx, const FwdApply& p) {
  if (p.no_relu || !p.mask) {
    launch_fwd_row_k<J, Full, true>(ctx, p);
    return;
  }
  launch_fwd_row_k<J, Full, false>(ctx, p);
}

void fwd_apply(Ctx& ctx, const FwdApply& p) {
  if (p.rows <= 0) return;
  require(p.cols <= kMaxJ * kRowChunk, "row kernels: at most 512 local feature columns");
  require(p.ldx % 4 == 0 && (!p.res || p.ldres % 4 == 0) && (!p.out || p.ldo % 4 == 0),
          "row kernels: fp32 rows must be 16-byte aligned");
  if (p.cols <= kRowChunk) {
    if (p.cols == kRowChunk)
      launch_fwd_row<1, true>(ctx, p);
    else
      launch_fwd_row<1, false>(ctx, p);
  } else if (p.cols <= 2 * kRowChunk) {
    if (p.cols == 2 * kRowChunk)
      launch_fwd_row<2, true>(ctx, p);
    else
      launch_fwd_row<2, false>(ctx, p);
  } else {
    if (p.cols == kMaxJ * kRowChunk)
      launch_fwd_row<kMaxJ, true>(ctx, p);
    else
      launch_fwd_row<kMaxJ, false>(ctx, p);
  }
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void bwd_stats(Ctx& ctx, const BwdApply& p) {
  if (p.rows <= 0) return;
  k_bwd_row_stats<<<row_blocks(p.rows), kT, 0, ctx.stream>>>(p);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

int bwd_apply_blocks(Ctx& ctx, int64_t rows, int64_t cols) {
  // one resident wave (4 blocks x 8 warps per SM up to 256 columns, 2 above),
  // grid-stride: few enough blocks that the dgamma partials reduce in
  // microseconds, enough warps in flight to saturate HBM
  const int per_sm = cols <= 2 * kRowChunk ? 4 : 2;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(row_blocks(rows), per_sm * ctx.num_sms)));
}

void bwd_apply(Ctx& ctx, const BwdApply& p, int blocks) {
  if (p.rows <= 0) return;
  require(p.cols <= kMaxJ * kRowChunk, "row kernels: at most 512 local feature columns");
  require(p.lddy % 4 == 0 && p.ldx % 4 == 0, "row kernels: fp32 rows must be 16-byte aligned");
  if (p.dxf) {
    require(!p.dxb, "row kernels: one dx format per call");
    if (p.cols <= kRowChunk)
      k_bwd_row<1, true><<<blocks, kT, 0, ctx.stream>>>(p);
    else if (p.cols <= 2 * kRowChunk)
      k_bwd_row<2, true><<<blocks, kT, 0, ctx.stream>>>(p);
    else
      k_bwd_row<kMaxJ, true><<<blocks, kT, 0, ctx.stream>>>(p);
  } else if (p.cols <= kRowChunk)
    k_bwd_row<1, false><<<blocks, kT, 0, ctx.stream>>>(p);
  else if (p.cols <= 2 * kRowChunk)  // (two rows per iteration here measured 2.1x slower: spills at 3 blocks/SM)
    k_bwd_row<2, false><<<blocks, kT, 0, ctx.stream>>>(p);
  else
    k_bwd_row<kMaxJ, false><<<blocks, kT, 0, ctx.stream>>>(p);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void dropout_keep(Ctx& ctx, uint64_t key, int64_t rows, int64_t cols, int64_t row_g0, int64_t col_g0,
                  uint64_t thresh, uint32_t* out, int64_t ldm) {
  if (rows <= 0) return;
  const int64_t blocks = std::min<int64_t>(ceil_div(rows * ldm, 128), 2 * ctx.num_sms);
  k_dropout_keep<<<static_cast<unsigned>(blocks), 128, 0, ctx.stream>>>(
      key, rows, cols, row_g0, col_g0, thresh, out, ldm);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

void ce_fused(Ctx& ctx, const CeArgs& p) {
  // rows per block: 8 warps x (32 / lanes-per-row)
  const int rpw = p.cols <= 64 ? 2 : 1;
  const unsigned blocks = std::max<unsigned>(1u, static_cast<unsigned>(ceil_div(p.rows, kRowsPerBlock * rpw)));
  require(static_cast<int64_t>(blocks) <= ce_grad_blocks(p.rows) + 1, "ce: partial buffer too small");
  if (p.rows > 0) {
    if (p.cols <= 64)
      k_ce_row_reg<16, 4><<<blocks, kT, 0, ctx.stream>>>(p);
    else if (p.cols <= 128)
      k_ce_row_reg<32, 4><<<blocks, kT, 0, ctx.stream>>>(p);
    else if (p.cols <= 256)
      k_ce_row_reg<32, 8><<<blocks, kT, 0, ctx.stream>>>(p);
    else
      k_ce_row<<<blocks, kT, 0, ctx.stream>>>(p);
    ctx.launches += 1;
  } else {
    GGB_CUDA(cudaMemsetAsync(p.loss_part, 0, sizeof(float), ctx.stream));
  }
  k_sum_parts_row<<<1, kT, 0, ctx.stream>>>(p.loss_part, p.rows > 0 ? blocks : 1, p.loss_acc);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

}  // namespace ggb
