// Pipelined row-split SpMM (the production path of spmm, pmm.hpp:134-167).
//
// Each warp of a persistent grid (one CTA per SM) owns a contiguous range of
// output rows and streams the nonzeros of that range in CSR order through a
// private STAGES-deep ring in shared memory: for every nonzero the gathered
// feature row (RB bytes: 256, 512 or 1024) is copied with cp.async (LDGSTS,
// 16 B per lane), so rows in flight cost shared memory, not registers, and
// the row_ptr -> col/val -> feature-row dependency chain is hidden behind
// STAGES-1 stages of look-ahead. A stage is 4 KB = S = 4096/RB nonzeros; its
// copies are issued by one unrolled loop of 8 warp-wide LDGSTS (every lane
// copies one 16-byte chunk per iteration), so the issue side costs a few
// instructions per nonzero. Column ids / values are loaded one stage ahead.
// The consumer accumulates in fp32 registers (lane l owns 16-byte chunks l and
// l+32 of the row) and flushes a row when the stream crosses its row_ptr
// boundary; empty rows flush zeros.
#include <cstdlib>
#include <string>
#include <type_traits>

#include "runtime.hpp"

namespace ggb {
namespace {

// 24-bit rows (the forward's layer activations, written by the fused row
// kernel): each value's fp32 bits rounded to the nearest multiple of 2^8,
// stored as a 16-bit high plane [C16 x u16] then an 8-bit low plane
// [C16 x u8] (C16 = cols rounded up to 8); decoded as (hi << 16) | (lo << 8).
struct P24 {};

constexpr int kWarps = 16;
constexpr int kStages = 3;
constexpr int kStageBytes = 4096;  // per warp per stage

struct PipeArgs {
  int64_t rows;
  const int64_t* rp;
  const int32_t* col;
  const float* val;
  const uint8_t* F;  // feature rows
  uint32_t ldf_bytes;
  int vcpr;  // valid 16-byte chunks of a row (the rest of RB is not read)
  int fcols;
  float* out;
  int64_t ldo;
  bf16* outb;
  bf16* outlo;
  int64_t ldob;
  int accumulate;
  int ocpr;  // output chunks of EPC columns (the flush's unit)
  int hoff;  // P24: byte offset of the low plane in a row
  int balanced;  // work-balanced row ranges (else an even row split)
  // rows longer than split_len nonzeros are split across warps along the
  // merge path (rows, nonzeros); partial sums go to per-warp carry rows and
  // k_spmm_carry_fixup adds them in warp order (deterministic)
  int64_t split_mult;  // rows of more than max(64, split_mult * work per warp) nonzeros are split
  float* lead;        // [warps][carry_ld]: partial of the warp's first row (owned by it, begun earlier)
  float* tail;        // [warps][carry_ld]: partial of the row the warp leaves unfinished
  int64_t* lead_row;  // [warps] row id or -1
  int64_t* tail_row;  // [warps] row id or -1
  int carry_ld;
  ptrdiff_t mirror;   // push mode (peer.cu): every output store is repeated at address + mirror
};

template <class T>
__device__ __forceinline__ T* mirror_of(T* p, ptrdiff_t d) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(p) + d);
}

// Warp work split: 2 = merge path with long rows shared (default), 1 =
// work-balanced whole rows (GGB_SPMM_SPLIT=balanced), 0 = even row split, the
// round-1 scheme (GGB_SPMM_SPLIT=rows)
int split_mode() {
  static const int v = [] {
    const char* e = std::getenv("GGB_SPMM_SPLIT");
    if (e && std::string(e) == "rows") return 0;
    if (e && std::string(e) == "balanced") return 1;
    return 2;
  }();
  return v;
}

__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

// Work-balanced row ranges: warp w of W owns rows [first(w), first(w+1)),
// first(w) = the smallest row r with cost(r) >= w * cost(rows) / W, where
// cost(r) = (rp[r] - rp[0]) + r counts nonzeros (one gathered feature row
// each) plus one flush per row. Power-law graphs (R-MAT) put thousands of
// nonzeros in a few rows: an even row split leaves their warps running long
// after the rest. Warp-cooperative 32-ary search: ~4 dependent loads.
__device__ __forceinline__ int64_t balanced_first_row(const int64_t* rp, int64_t rows, int64_t w, int64_t W,
                                                      int lane) {
  if (w <= 0) return 0;
  if (w >= W) return rows;
  const int64_t base = rp[0];
  const int64_t total = (rp[rows] - base) + rows;
  // target = ceil(w * total / W) without overflowing 64 bits
  const int64_t target = (total / W) * w + ((total % W) * w + W - 1) / W;
  int64_t lo = 0, hi = rows;  // cost(hi) >= target; answer in (lo, hi] unless cost(lo) >= target
  if (target <= 0) return 0;
  while (hi - lo > 1) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t probe = imin(hi, lo + (lane + 1) * step);
    const bool ge = (__ldg(rp + probe) - base) + probe >= target;
    const uint32_t m = __ballot_sync(0xffffffffu, ge);
    const int first = m ? __ffs(m) - 1 : 31;
    const int64_t nhi = imin(hi, lo + (first + 1) * step);
    lo = lo + first * step;
    hi = nhi;
  }
  return hi;
}

// Point (row, nonzero) of warp w's start on the merge path of (row flushes,
// nonzeros): diagonal d = ceil(w * total / W), total = nonzeros + rows. A
// point inside a row of at most split_len nonzeros snaps back to that row's
// start (the row stays whole); one at a row's end moves to the next row's
// start. So only long rows are shared between warps.
__device__ __forceinline__ void path_point(const int64_t* rp, int64_t rows, int64_t w, int64_t W, int64_t split_mult,
                                           int lane, int64_t& r, int64_t& e) {
  const int64_t base = rp[0];
  const int64_t total = (rp[rows] - base) + rows;
  const int64_t split_len = split_mult * (total / W) > 64 ? split_mult * (total / W) : 64;
  if (w <= 0) {
    r = 0;
    e = base;
    return;
  }
  const int64_t d = w >= W ? total : (total / W) * w + ((total % W) * w + W - 1) / W;
  if (d >= total) {
    r = rows;
    e = rp[rows];
    return;
  }
  // smallest r' with cost(r') >= d + 1, minus one (cost(r') = rp[r'] - base + r')
  r = balanced_first_row(rp, rows, d + 1, total, lane) - 1;
  e = base + (d - r);
  const int64_t s = rp[r], t = rp[r + 1];
  if (e > s && t - s <= split_len) {
    e = s;
  } else if (e == t && e > s) {
    r += 1;
  }
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// TIn: element type of F; RB: smem bytes per gathered row; kMerge: merge-path
// ranges with long rows shared across warps (power-law inputs) — a separate
// instance, so the whole-row kernel keeps its code generation; kMirror: the
// push-mode instance (peer.cu) that repeats every output store into the
// peer's slot (separate, so the plain kernels keep their code too: the
// runtime-offset stores may alias for the compiler and serialized the
// backward's accumulate loads, 2.2 -> 3.3 ms/step).
template <class TIn, int RB, bool kMerge, bool kMirror = false>
__global__ void __launch_bounds__(kWarps * 32, 1) k_spmm_pipe(const PipeArgs a) {
  constexpr bool kP24 = std::is_same_v<TIn, P24>;
  constexpr int EPC = kP24 ? 8 : 16 / static_cast<int>(sizeof(TIn));  // elements per lane chunk
  constexpr int CPR = RB / 16;                                         // 16-byte chunks per row slot
  constexpr int S = kStageBytes / RB;                                  // nonzeros per stage
  constexpr int CPL = kP24 ? 1 : (CPR > 32 ? 2 : 1);                   // chunks per lane (consumer)
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* ring = smem + static_cast<size_t>(wib) * kStages * kStageBytes;
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
  float* meta_val = reinterpret_cast<float*>(smem + kWarps * kStages * kStageBytes) + wib * kStages * 32;

  const int64_t total_warps = static_cast<int64_t>(gridDim.x) * kWarps;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kWarps + wib;
  int64_t r_begin, r_end, e_begin, e_end;
  bool lead = false;  // the first row began in earlier warps: its flush goes to the carry
  if constexpr (kMerge) {
    path_point(a.rp, a.rows, gw, total_warps, a.split_mult, lane, r_begin, e_begin);
    path_point(a.rp, a.rows, gw + 1, total_warps, a.split_mult, lane, r_end, e_end);
    lead = r_begin < a.rows && e_begin > a.rp[r_begin];
    if (lane == 0) {
      a.lead_row[gw] = -1;
      a.tail_row[gw] = -1;
    }
  } else if (a.balanced) {
    r_begin = balanced_first_row(a.rp, a.rows, gw, total_warps, lane);
    r_end = balanced_first_row(a.rp, a.rows, gw + 1, total_warps, lane);
    e_begin = a.rp[r_begin];
    e_end = a.rp[r_end];
  } else {
    const int64_t per = (a.rows + total_warps - 1) / total_warps;
    r_begin = imin(a.rows, gw * per);
    r_end = imin(a.rows, r_begin + per);
    e_begin = a.rp[r_begin];
    e_end = a.rp[r_end];
  }
  if (kMerge ? (r_begin >= r_end && e_begin >= e_end) : r_begin >= r_end) return;
  const int64_t n_stages = (e_end - e_begin + S - 1) / S;

  int32_t nx_col = 0;  // lane k < S: column id / value of entry k of the next stage to issue
  float nx_val = 0.f;
  auto load_meta = [&](int64_t t) {
    const int64_t e = e_begin + t * S + lane;
    nx_col = 0;
    nx_val = 0.f;
    if (lane < S && t < n_stages && e < e_end) {
      nx_col = __ldg(a.col + e);
      nx_val = __ldg(a.val + e);
    }
  };
  auto issue = [&](int64_t t) {
    if (t < n_stages) {
      const int slot = static_cast<int>(t % kStages);
      const int valid = static_cast<int>(imin(S, e_end - (e_begin + t * S)));
      if (lane < S) meta_val[slot * 32 + lane] = nx_val;
      const uint32_t dst0 = ring_s + slot * kStageBytes;
#pragma unroll
      for (int it = 0; it < kStageBytes / 512; ++it) {
        const int idx = it * 32 + lane;  // chunk of the stage: entry k, chunk ch
        const int k = idx / CPR, ch = idx % CPR;
        const int32_t c = __shfl_sync(0xffffffffu, nx_col, k);
        if (k < valid && ch < a.vcpr)
          cp_async16(dst0 + idx * 16, a.F + static_cast<uint64_t>(static_cast<uint32_t>(c)) * a.ldf_bytes + ch * 16);
      }
    }
    cp_commit();
    load_meta(t + 1);
  };

  load_meta(0);
#pragma unroll 1
  for (int t = 0; t < kStages - 1; ++t) issue(t);

  float acc[CPL][EPC];
#pragma unroll
  for (int q = 0; q < CPL; ++q)
#pragma unroll
    for (int i = 0; i < EPC; ++i) acc[q][i] = 0.f;
  int64_t row = r_begin;
  int64_t row_end_e = a.rp[row + 1];

  // the partial sums of a shared row, in column order, to a carry row
  auto to_carry = [&](float* dst) {
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int ch = lane + 32 * q;
      if (ch < a.ocpr) {
#pragma unroll
        for (int i = 0; i < EPC; ++i) dst[ch * EPC + i] = acc[q][i];
      }
#pragma unroll
      for (int i = 0; i < EPC; ++i) acc[q][i] = 0.f;
    }
  };

  auto flush = [&]() {
    if constexpr (kMerge) {
      if (lead && row == r_begin) {
        to_carry(a.lead + gw * a.carry_ld);
        if (lane == 0) a.lead_row[gw] = row;
        return;
      }
    }
#pragma unroll
    for (int q = 0; q < CPL; ++q) {
      const int ch = lane + 32 * q;
      const int64_t cc = static_cast<int64_t>(ch) * EPC;
      if (ch < a.ocpr) {
        const bool whole = cc + EPC <= a.fcols;
        if (a.out) {
          float* dst = a.out + row * a.ldo + cc;
          if (whole && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int v = 0; v < EPC; v += 4) {
              float4 o = make_float4(acc[q][v], acc[q][v + 1], acc[q][v + 2], acc[q][v + 3]);
              if (a.accumulate) {
                const float4 p = *reinterpret_cast<const float4*>(dst + v);
                o.x += p.x;
                o.y += p.y;
                o.z += p.z;
                o.w += p.w;
                acc[q][v] = o.x;
                acc[q][v + 1] = o.y;
                acc[q][v + 2] = o.z;
                acc[q][v + 3] = o.w;
              }
              *reinterpret_cast<float4*>(dst + v) = o;
              if constexpr (kMirror) *reinterpret_cast<float4*>(mirror_of(dst + v, a.mirror)) = o;
            }
          } else {
            for (int i = 0; i < EPC && cc + i < a.fcols; ++i) {
              if (a.accumulate) acc[q][i] += dst[i];
              dst[i] = acc[q][i];
              if constexpr (kMirror) *mirror_of(dst + i, a.mirror) = acc[q][i];
            }
          }
        }
        if (a.outb) {
          bf16* db = a.outb + row * a.ldob + cc;
          bf16* dl = a.outlo ? a.outlo + row * a.ldob + cc : nullptr;
          if (whole && (reinterpret_cast<uintptr_t>(db) & (EPC * 2 - 1)) == 0) {
            uint32_t hi[EPC / 2], lo[EPC / 2];
#pragma unroll
            for (int v = 0; v < EPC; v += 2) {
              hi[v / 2] = pack_bf16(acc[q][v], acc[q][v + 1]);
              const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&hi[v / 2]);
              const float2 hf = __bfloat1622float2(h);
              lo[v / 2] = pack_bf16(acc[q][v] - hf.x, acc[q][v + 1] - hf.y);
            }
            if constexpr (EPC == 8) {
              *reinterpret_cast<uint4*>(db) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
              if constexpr (kMirror) *reinterpret_cast<uint4*>(mirror_of(db, a.mirror)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
              if (dl) *reinterpret_cast<uint4*>(dl) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            } else {
              *reinterpret_cast<uint2*>(db) = make_uint2(hi[0], hi[1]);
              if constexpr (kMirror) *reinterpret_cast<uint2*>(mirror_of(db, a.mirror)) = make_uint2(hi[0], hi[1]);
              if (dl) *reinterpret_cast<uint2*>(dl) = make_uint2(lo[0], lo[1]);
            }
          } else {
            for (int i = 0; i < EPC && cc + i < a.fcols; ++i) {
              const bf16 h = __float2bfloat16_rn(acc[q][i]);
              db[i] = h;
              if constexpr (kMirror) *mirror_of(db + i, a.mirror) = h;
              if (dl) dl[i] = __float2bfloat16_rn(acc[q][i] - __bfloat162float(h));
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < EPC; ++i) acc[q][i] = 0.f;
    }
  };

#pragma unroll 1
  for (int64_t t = 0; t < n_stages; ++t) {
    issue(t + kStages - 1);
    cp_wait<kStages - 1>();
    __syncwarp();
    const int slot = static_cast<int>(t % kStages);
    const int64_t e0 = e_begin + t * S;
    const int valid = static_cast<int>(imin(S, e_end - e0));
    const uint8_t* base = ring + slot * kStageBytes;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      if (k < valid) {
        while (e0 + k >= row_end_e) {  // crossed into the next row(s): flush; empty rows give zeros
          flush();
          ++row;
          row_end_e = a.rp[row + 1];
        }
        const float v = meta_val[slot * 32 + k];
        if constexpr (kP24) {
          if (lane < a.ocpr) {  // lane owns columns 8 lane .. 8 lane + 7
            const uint4 h = *reinterpret_cast<const uint4*>(base + k * RB + lane * 16);
            const uint2 w = *reinterpret_cast<const uint2*>(base + k * RB + a.hoff + lane * 8);
            const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[2] = {w.x, w.y};
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const uint32_t hi = (i & 1) ? (hw[i >> 1] & 0xffff0000u) : (hw[i >> 1] << 16);
              const uint32_t lo = __byte_perm(lw[i >> 2], 0u, 0x4404u | ((i & 3) << 4));  // byte (i&3) -> byte 1
              acc[0][i] = fmaf(v, __uint_as_float(hi | lo), acc[0][i]);
            }
          }
          continue;
        }
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const int ch = lane + 32 * q;
          if (ch < a.vcpr) {
            const uint4 u = *reinterpret_cast<const uint4*>(base + k * RB + ch * 16);
            if constexpr (sizeof(TIn) == 2) {
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 f = __bfloat1622float2(h[i]);
                acc[q][2 * i] = fmaf(v, f.x, acc[q][2 * i]);
                acc[q][2 * i + 1] = fmaf(v, f.y, acc[q][2 * i + 1]);
              }
            } else {
              acc[q][0] = fmaf(v, __uint_as_float(u.x), acc[q][0]);
              acc[q][1] = fmaf(v, __uint_as_float(u.y), acc[q][1]);
              acc[q][2] = fmaf(v, __uint_as_float(u.z), acc[q][2]);
              acc[q][3] = fmaf(v, __uint_as_float(u.w), acc[q][3]);
            }
          }
        }
      }
    }
    __syncwarp();  // the slot is refilled by a later issue
  }
  cp_wait<0>();
  while (row < r_end) {  // the last row and any trailing empty rows of the range
    flush();
    ++row;
  }
  if constexpr (kMerge) {
    if (r_end < a.rows && e_end > a.rp[r_end]) {  // row r_end continues in later warps
      to_carry(a.tail + gw * a.carry_ld);
      if (lane == 0) a.tail_row[gw] = r_end;
    }
  }
}

// Rows shared by several warps: (tails of the earlier warps in warp order) +
// the owner's lead partial, then the flush epilogue (accumulate into the fp32
// output; bf16 hi / lo split). One warp per owner.
__global__ void k_spmm_carry_fixup(const PipeArgs a, int64_t warps) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= warps) return;
  const int64_t row = a.lead_row[w];
  if (row < 0) return;
  int64_t w0 = w;
  while (w0 > 0 && a.tail_row[w0 - 1] == row) --w0;
  for (int64_t c = lane; c < a.fcols; c += 32) {
    float s = 0.f;
    for (int64_t k = w0; k < w; ++k) s += a.tail[k * a.carry_ld + c];
    s += a.lead[w * a.carry_ld + c];
    if (a.out) {
      float* dst = a.out + row * a.ldo + c;
      if (a.accumulate) s += *dst;
      *dst = s;
      if (a.mirror) *mirror_of(dst, a.mirror) = s;
    }
    if (a.outb) {
      const bf16 h = __float2bfloat16_rn(s);
      a.outb[row * a.ldob + c] = h;
      if (a.mirror) *mirror_of(a.outb + row * a.ldob + c, a.mirror) = h;
      if (a.outlo) a.outlo[row * a.ldob + c] = __float2bfloat16_rn(s - __bfloat162float(h));
    }
  }
}

template <class TIn, int RB, bool kMerge, bool kMirror>
void set_smem_attr() {
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    GGB_CUDA(cudaFuncSetAttribute(k_spmm_pipe<TIn, RB, kMerge, kMirror>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kWarps * kStages * kStageBytes + kWarps * kStages * 32 * 4));
  }
}

template <class TIn, int RB>
void launch_pipe(Ctx& ctx, PipeArgs a) {
  const int smem = kWarps * kStages * kStageBytes + kWarps * kStages * 32 * 4;
  const int grid = ctx.persistent_sms();
  const int64_t warps = static_cast<int64_t>(grid) * kWarps;
  // merge path when the caller flags long rows (ctx.spmm_long_rows: a power-law
  // shard) unless GGB_SPMM_SPLIT forces a whole-row split
  const int mode = split_mode() == 2 ? (ctx.spmm_long_rows ? 2 : 1) : split_mode();
  a.balanced = mode >= 1;
  if (mode == 2) {
    a.carry_ld = static_cast<int>(round_up(a.fcols, 8));
    a.split_mult = 4;
    float* base = ctx.spmm_carry.reserve_n<float>(static_cast<size_t>(warps) * (2 * a.carry_ld + 4));
    a.lead = base;
    a.tail = base + warps * a.carry_ld;
    a.lead_row = reinterpret_cast<int64_t*>(base + 2 * warps * a.carry_ld);
    a.tail_row = a.lead_row + warps;
  }
  const bool mirror = a.mirror != 0;
  if constexpr (std::is_same_v<TIn, P24>) require(!mirror, "spmm: no mirrored 24-bit instance");
  if (mode == 2 && mirror) {
    if constexpr (!std::is_same_v<TIn, P24>) {
      set_smem_attr<TIn, RB, true, true>();
      k_spmm_pipe<TIn, RB, true, true><<<grid, kWarps * 32, smem, ctx.stream>>>(a);
    }
  } else if (mode == 2) {
    set_smem_attr<TIn, RB, true, false>();
    k_spmm_pipe<TIn, RB, true, false><<<grid, kWarps * 32, smem, ctx.stream>>>(a);
  } else if (mirror) {
    if constexpr (!std::is_same_v<TIn, P24>) {
      set_smem_attr<TIn, RB, false, true>();
      k_spmm_pipe<TIn, RB, false, true><<<grid, kWarps * 32, smem, ctx.stream>>>(a);
    }
  } else {
    set_smem_attr<TIn, RB, false, false>();
    k_spmm_pipe<TIn, RB, false, false><<<grid, kWarps * 32, smem, ctx.stream>>>(a);
  }
  if (mode == 2) {
    k_spmm_carry_fixup<<<static_cast<unsigned>(ceil_div(warps, 8)), 256, 0, ctx.stream>>>(a, warps);
    ctx.launches += 1;
  }
}

}  // namespace

// Row-split SpMM through the pipelined kernel when a gathered row fits a
// 1 KB slot; returns false otherwise (the caller falls back).
bool spmm_pipe(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val, const void* f,
               int esize, int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* outb, bf16* outlo, int64_t ldob,
               int accumulate) {
  const int64_t row_bytes = round_up(fcols * esize, 16);
  if (row_bytes > 1024 || rows <= 0 || fcols <= 0) return false;
  if (ldf * esize >= (int64_t{1} << 32)) return false;
  PipeArgs a{};
  a.rows = rows;
  a.rp = rp;
  a.col = col;
  a.val = val;
  a.F = static_cast<const uint8_t*>(f);
  a.ldf_bytes = static_cast<uint32_t>(ldf * esize);
  a.vcpr = static_cast<int>(row_bytes / 16);
  a.fcols = static_cast<int>(fcols);
  a.out = out;
  a.ldo = ldo;
  a.outb = outb;
  a.outlo = outlo;
  a.ldob = ldob;
  a.accumulate = accumulate;
  a.ocpr = a.vcpr;
  a.mirror = ctx.out_mirror;
  require(!(a.mirror && (outlo || accumulate)), "spmm: a mirrored output is a plain partial (no lo half, no accumulate)");
  if (esize == 2) {
    if (row_bytes <= 256)
      launch_pipe<bf16, 256>(ctx, a);
    else if (row_bytes <= 512)
      launch_pipe<bf16, 512>(ctx, a);
    else
      launch_pipe<bf16, 1024>(ctx, a);
  } else {
    if (row_bytes <= 256)
      launch_pipe<float, 256>(ctx, a);
    else if (row_bytes <= 512)
      launch_pipe<float, 512>(ctx, a);
    else
      launch_pipe<float, 1024>(ctx, a);
  }
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
  return true;
}

// Forward SpMM gathering 24-bit rows (see P24): fcols <= 256, row stride
// ld_bytes (a multiple of 16, >= 3 * round_up(fcols, 8)).
bool spmm_pipe_p24(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
                   const uint8_t* f, int64_t ld_bytes, int64_t fcols, bf16* out_hi, bf16* out_lo, int64_t ldob) {
  const int64_t c16 = round_up(fcols, 8);
  const int64_t row_bytes = round_up(3 * c16, 16);
  if (rows <= 0 || fcols <= 0 || fcols > 256 || ctx.side_stream) return false;
  require(ld_bytes % 16 == 0 && ld_bytes >= row_bytes && (reinterpret_cast<uintptr_t>(f) & 15) == 0,
          "spmm: 24-bit rows need 16-byte aligned rows");
  if (ld_bytes >= (int64_t{1} << 32)) return false;
  PipeArgs a{};
  a.rows = rows;
  a.rp = rp;
  a.col = col;
  a.val = val;
  a.F = f;
  a.ldf_bytes = static_cast<uint32_t>(ld_bytes);
  a.vcpr = static_cast<int>(row_bytes / 16);
  a.fcols = static_cast<int>(fcols);
  a.outb = out_hi;
  a.outlo = out_lo;
  a.ldob = ldob;
  a.ocpr = static_cast<int>(c16 / 8);
  a.hoff = static_cast<int>(2 * c16);
  if (row_bytes <= 384)
    launch_pipe<P24, 384>(ctx, a);
  else
    launch_pipe<P24, 768>(ctx, a);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
  return true;
}

}  // namespace ggb
