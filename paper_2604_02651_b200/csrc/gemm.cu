// Dense GEMMs of the 3D-PMM GCN layer (the `contract` of pmm.hpp:97-130) on
// the 5th-generation tensor cores: bf16 operands staged by TMA into 128B-
// swizzled shared memory, tcgen05.mma issued by one thread, fp32 accumulators
// in TMEM, tcgen05.ld epilogue. No materialized transposes (pmm.hpp:76-92 is
// eliminated): the forward / dX products read both operands K-major, the
// weight-gradient product reads both operands MN-major straight from the
// row-major activations.
//
//   k_gemm_kmajor : C[M x N] = A[M x K] . Bt[N x K]^T
//                   persistent over 128-row tiles; warp 0 = TMA producer,
//                   warp 1 = MMA issuer, warps 2-5 = epilogue; 2 TMEM
//                   accumulators so the epilogue of tile t overlaps the
//                   loads/MMAs of tile t+1.
//   k_gemm_wgrad  : DW[KW x NW] = X[M x KW]^T . DY[M x NW]
//                   split over the contraction (M) rows; fp32 partial tiles,
//                   reduced deterministically by k_reduce_partials.
#include <cuda.h>

#include <mutex>
#include <unordered_map>

#include "runtime.hpp"

namespace ggb {
namespace {

constexpr int kBM = 128;  // UMMA M (cta_group::1)
constexpr int kBK = 64;   // one 128-byte swizzle atom of bf16 along K
constexpr int kEpiWarps = 8;  // 2 per TMEM lane quarter, each on half of the tile's columns
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kWgradThreads = 192;
constexpr int kSmemBudget = 227 * 1024;  // dynamic smem per CTA (the sm_100 maximum)
// epilogue staging, one 4 KB buffer per epilogue warp (32 rows x 16 columns:
// fp32 2 KB, bf16 1 KB, bf16 lo 1 KB), then the barriers
constexpr int kEpiBuf = 4096;
constexpr int kEpiSmem = kEpiWarps * kEpiBuf + 256;

// ---- PTX wrappers --------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// TMA store of a shared-memory box; bulk-group completion
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t pack2_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t pack2_lo(float a, float b) {
  return pack2_bf16(a - __bfloat162float(__float2bfloat16_rn(a)), b - __bfloat162float(__float2bfloat16_rn(b)));
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 lanes x 16 consecutive fp32 columns of the accumulator
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%"
      "15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bit.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (Blackwell)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: bf16 x bf16 -> fp32, M = 128.
__host__ __device__ constexpr uint32_t idesc_bf16(int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(kBM >> 4) << 24);
}

struct GemmArgs {
  int M, N, K;
  int split;    // 1: operands given as bf16 hi + lo pairs, D += Ah.Bh + Ah.Bl + Al.Bh
  int BN;       // MMA N of one tile (multiple of 16, <= 256)
  int n_tiles;  // ceil(N / BN)
  int b_res;    // 1: B loaded once per CTA and kept in shared memory (n_tiles == 1)
  int tma_out;  // 1: outputs leave through TMA stores (16-byte aligned rows)
  int stages;
  uint32_t tmem_cols;
  float* c;
  int64_t ldc;
  bf16* cb;
  bf16* cl;  // optional lo residual of the bf16 output: c == cb + cl to ~2^-16
  int64_t ldcb;
  // push-mode peer reductions (peer.cu): tmCl is a map of the peer's copy of
  // the output and every TMA store of c (1) or cb (2) is repeated into it
  int mirror;
};

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_kmajor(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmAl, const __grid_constant__ CUtensorMap tmBl,
                  const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmCb,
                  const __grid_constant__ CUtensorMap tmCl, const GemmArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned by pointer arithmetic on the shared array, so every
  // derived pointer stays in the shared window (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = args.stages, BN = args.BN;
  const int parts = args.split ? 2 : 1;
  const int k_chunks = (args.K + kBK - 1) / kBK;
  const uint32_t bytes_a = kBM * kBK * 2, bytes_b = static_cast<uint32_t>(BN) * kBK * 2;
  // streamed stage: [A hi][A lo]?[B hi][B lo]? -- or, with B resident (one
  // n-tile: the whole B is loaded once per CTA), [A hi][A lo]? only
  const uint32_t stage_bytes = parts * (bytes_a + (args.b_res ? 0u : bytes_b));
  uint8_t* bres = smem + S * stage_bytes;  // [k chunk][hi, lo?] when b_res
  const uint32_t bres_bytes = args.b_res ? static_cast<uint32_t>(k_chunks) * parts * bytes_b : 0u;
  uint8_t* epi = bres + bres_bytes;  // kEpiWarps x kEpiBuf, 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(epi + kEpiWarps * kEpiBuf);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;  // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint64_t* bfull = tempty + 2;  // B resident loaded
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(bfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (args.M + kBM - 1) / kBM;
  const int num_tiles = m_tiles * args.n_tiles;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (args.split) {
      prefetch_tmap(&tmAl);
      prefetch_tmap(&tmBl);
    }
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, kEpiWarps);
    }
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_base_smem, args.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      if (args.b_res) {  // the whole B (single n-tile), once
        mbar_expect_tx(bfull, bres_bytes);
        for (int kc = 0; kc < k_chunks; ++kc) {
          uint8_t* sb = bres + kc * parts * bytes_b;
          tma_load_2d(sb, &tmB, bfull, kc * kBK, 0);
          if (args.split) tma_load_2d(sb + bytes_b, &tmBl, bfull, kc * kBK, 0);
        }
      }
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int mt = t / args.n_tiles, nt = t % args.n_tiles;
        for (int kc = 0; kc < k_chunks; ++kc) {
          mbar_wait(empty + stage, phase ^ 1);
          uint8_t* sa = smem + stage * stage_bytes;
          uint8_t* sb = sa + parts * bytes_a;
          mbar_expect_tx(full + stage, stage_bytes);
          tma_load_2d(sa, &tmA, full + stage, kc * kBK, mt * kBM);
          if (!args.b_res) tma_load_2d(sb, &tmB, full + stage, kc * kBK, nt * BN);
          if (args.split) {
            tma_load_2d(sa + bytes_a, &tmAl, full + stage, kc * kBK, mt * kBM);
            if (!args.b_res) tma_load_2d(sb + bytes_b, &tmBl, full + stage, kc * kBK, nt * BN);
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      const uint32_t idesc = idesc_bf16(BN, false, false);
      int stage = 0;
      uint32_t phase = 0;
      int lt = 0;
      if (args.b_res) mbar_wait(bfull, 0);
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
        const int acc = lt & 1;
        const uint32_t acc_phase = (lt >> 1) & 1;
        mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kc = 0; kc < k_chunks; ++kc) {
          mbar_wait(full + stage, phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * stage_bytes);
          const uint32_t sb = args.b_res ? smem_u32(bres + kc * parts * bytes_b) : sa + parts * bytes_a;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ah = sdesc(sa + k * 32, 16, 1024), bh = sdesc(sb + k * 32, 16, 1024);
            umma_bf16(d, ah, bh, idesc, (kc | k) != 0);
            if (args.split) {  // the two cross terms of (Ah + Al)(Bh + Bl); Al.Bl is below fp32 rounding
              umma_bf16(d, ah, sdesc(sb + bytes_b + k * 32, 16, 1024), idesc, 1);
              umma_bf16(d, sdesc(sa + bytes_a + k * 32, 16, 1024), bh, idesc, 1);
            }
          }
          umma_commit(empty + stage);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull + acc);
      }
    }
    __syncwarp();
  } else {  // ---- epilogue: warps 2..9, TMEM lane quarter = warp % 4, column half = (warp - 2) / 4
    // Each 32-row x 16-column accumulator block goes TMEM -> registers (row
    // per lane) -> padded smem tile -> registers (4 consecutive columns per
    // lane), so the global stores are row-contiguous: 4 lanes cover 64 bytes
    // of one row (fp32) and one store instruction writes 8 full row segments.
    const int q = warp & 3;
    const int half = (warp - 2) / 4;
    uint8_t* ebuf = epi + (warp - 2) * kEpiBuf;
    float* stile = reinterpret_cast<float*>(ebuf);  // 32 x 17 padded transpose tile (store fallback)
    int lt = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++lt) {
      const int mt = t / args.n_tiles, nt = t % args.n_tiles;
      const int acc = lt & 1;
      const uint32_t acc_phase = (lt >> 1) & 1;
      mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const int64_t row_base = static_cast<int64_t>(mt) * kBM + q * 32;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
      const int cspan = ((BN / 16 + 1) / 2) * 16;  // columns of this warp's half (multiple of 16)
      const int cbeg = half * cspan, cend = min(BN, cbeg + cspan);
      for (int c16 = cbeg; c16 < cend; c16 += 16) {
        float v[16];
        tmem_ld16(taddr + c16, v);
        const int col0 = nt * BN + c16;
        if (col0 >= args.N) continue;  // warp-uniform
        if (args.tma_out) {
          // lane = row: its 16 columns go to the staging boxes in the TMA
          // swizzle (fp32 64 B rows: SWIZZLE_64B; bf16 32 B rows: SWIZZLE_32B,
          // conflict-free 16-byte stores), then one lane issues the stores
          if (lane == 0) bulk_wait_read0();  // the previous block's stores have read the buffer
          __syncwarp();
          if (args.c) {
            float4* rowp = reinterpret_cast<float4*>(ebuf + lane * 64);
            const int sw = (lane >> 1) & 3;
#pragma unroll
            for (int ch = 0; ch < 4; ++ch)
              rowp[ch ^ sw] = make_float4(v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
          }
          if (args.cb) {
            const int sw = (lane >> 2) & 1;
            uint4* rowb = reinterpret_cast<uint4*>(ebuf + 2048 + lane * 32);
#pragma unroll
            for (int ch = 0; ch < 2; ++ch)
              rowb[ch ^ sw] = make_uint4(pack2_bf16(v[8 * ch], v[8 * ch + 1]), pack2_bf16(v[8 * ch + 2], v[8 * ch + 3]),
                                         pack2_bf16(v[8 * ch + 4], v[8 * ch + 5]),
                                         pack2_bf16(v[8 * ch + 6], v[8 * ch + 7]));
            if (args.cl) {
              uint4* rowl = reinterpret_cast<uint4*>(ebuf + 3072 + lane * 32);
#pragma unroll
              for (int ch = 0; ch < 2; ++ch)
                rowl[ch ^ sw] = make_uint4(pack2_lo(v[8 * ch], v[8 * ch + 1]), pack2_lo(v[8 * ch + 2], v[8 * ch + 3]),
                                           pack2_lo(v[8 * ch + 4], v[8 * ch + 5]),
                                           pack2_lo(v[8 * ch + 6], v[8 * ch + 7]));
            }
          }
          fence_async_shared();
          __syncwarp();
          if (lane == 0) {
            const int r0 = mt * kBM + q * 32;
            if (args.c) tma_store_2d(&tmC, ebuf, col0, r0);
            if (args.cb) tma_store_2d(&tmCb, ebuf + 2048, col0, r0);
            if (args.cl) tma_store_2d(&tmCl, ebuf + 3072, col0, r0);
            if (args.mirror) tma_store_2d(&tmCl, args.mirror == 1 ? ebuf : ebuf + 2048, col0, r0);
            bulk_commit();
          }
          continue;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) stile[lane * 17 + i] = v[i];
        __syncwarp();
        const int cc = (lane & 3) * 4;  // column offset within the 16-column block
        const int col = col0 + cc;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int rl = it * 8 + (lane >> 2);  // local row 0..31
          const int64_t row = row_base + rl;
          float o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) o[i] = stile[rl * 17 + cc + i];
          if (row >= args.M || col >= args.N) continue;
          const bool full4 = col + 4 <= args.N;
          if (args.c) {
            float* dst = args.c + row * args.ldc + col;
            if (full4 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0)
              *reinterpret_cast<float4*>(dst) = make_float4(o[0], o[1], o[2], o[3]);
            else
              for (int i = 0; i < 4 && col + i < args.N; ++i) dst[i] = o[i];
          }
          if (args.cb) {
            bf16* dst = args.cb + row * args.ldcb + col;
            bf16* dl = args.cl ? args.cl + row * args.ldcb + col : nullptr;
            if (full4 && (reinterpret_cast<uintptr_t>(dst) & 7) == 0) {
              __nv_bfloat162 h0 = __floats2bfloat162_rn(o[0], o[1]), h1 = __floats2bfloat162_rn(o[2], o[3]);
              *reinterpret_cast<uint2*>(dst) =
                  make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
              if (dl) {
                const float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
                __nv_bfloat162 l0 = __floats2bfloat162_rn(o[0] - f0.x, o[1] - f0.y),
                               l1 = __floats2bfloat162_rn(o[2] - f1.x, o[3] - f1.y);
                *reinterpret_cast<uint2*>(dl) =
                    make_uint2(*reinterpret_cast<uint32_t*>(&l0), *reinterpret_cast<uint32_t*>(&l1));
              }
            } else {
              for (int i = 0; i < 4 && col + i < args.N; ++i) {
                const bf16 h = __float2bfloat16_rn(o[i]);
                dst[i] = h;
                if (dl) dl[i] = __float2bfloat16_rn(o[i] - __bfloat162float(h));
              }
            }
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
    }
    if (args.tma_out && lane == 0) bulk_wait0();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, args.tmem_cols);
  }
}

struct WgradArgs {
  int M, KW, NW;
  int BN;  // multiple of 64, <= 256
  int MT;  // m-tiles (128 KW rows each) per CTA: 2 when KW <= 256 (the DY chunk is loaded once for both)
  int n_tiles, m_tiles, splits, chunks_per_split;
  int stages;
  uint32_t tmem_cols;
  float* part;  // [splits][KW][NW]
};

__global__ void __launch_bounds__(kWgradThreads, 1)
    k_gemm_wgrad(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmD,
                 const WgradArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = args.stages, BN = args.BN, MT = args.MT;
  // A' tile: MT x 128 (KW) x 64 (rows): 2 MT 64-col boxes of 64 rows x 128 B
  const uint32_t bytes_a = MT * kBM * kBK * 2, bytes_b = static_cast<uint32_t>(BN) * kBK * 2;
  const uint32_t stage_bytes = bytes_a + bytes_b;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, split = blockIdx.y;
  const int mt = (tile / args.n_tiles) * MT, nt = tile % args.n_tiles;  // first m-tile of this CTA
  const int total_chunks = (args.M + kBK - 1) / kBK;
  const int c_begin = split * args.chunks_per_split;
  const int c_end = min(total_chunks, c_begin + args.chunks_per_split);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmD);
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_base_smem, args.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int c = c_begin; c < c_end; ++c) {
        mbar_wait(empty + stage, phase ^ 1);
        uint8_t* sa = smem + stage * stage_bytes;
        uint8_t* sb = sa + bytes_a;
        mbar_expect_tx(full + stage, stage_bytes);
        for (int h = 0; h < MT * kBM / 64; ++h)
          tma_load_2d(sa + h * 8192, &tmX, full + stage, mt * kBM + h * 64, c * kBK);
        for (int h = 0; h < BN / 64; ++h)
          tma_load_2d(sb + h * 8192, &tmD, full + stage, nt * BN + h * 64, c * kBK);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16(BN, true, true);
      int stage = 0;
      uint32_t phase = 0;
      for (int c = c_begin; c < c_end; ++c) {
        mbar_wait(full + stage, phase);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + stage * stage_bytes);
        const uint32_t sb = sa + bytes_a;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)  // 16 K-rows = 2 groups of 8 rows x 128 B
          for (int t = 0; t < MT; ++t)      // m-tile t: accumulator columns [t BN, (t + 1) BN)
            umma_bf16(tmem_base + static_cast<uint32_t>(t * BN), sdesc(sa + t * 16384 + k * 2048, 8192, 1024),
                      sdesc(sb + k * 2048, 8192, 1024), idesc, (c != c_begin || k != 0));
        umma_commit(empty + stage);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit(tfull);
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    const bool any = c_end > c_begin;
    if (any) {
      mbar_wait(tfull, 0);
      tc_fence_after();
    }
    float* dst_base = args.part + static_cast<int64_t>(split) * args.KW * args.NW;
    for (int t = 0; t < MT; ++t) {
      const int64_t row = static_cast<int64_t>(mt + t) * kBM + q * 32 + lane;  // KW index
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(t * BN);
      for (int c16 = 0; c16 < BN; c16 += 16) {
        float v[16];
        if (any) {
          tmem_ld16(taddr + c16, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        const int col0 = nt * BN + c16;
        if (row >= args.KW || col0 >= args.NW) continue;
        float* dst = dst_base + row * args.NW + col0;
        if (col0 + 16 <= args.NW && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
          for (int ch = 0; ch < 4; ++ch)
            reinterpret_cast<float4*>(dst)[ch] = make_float4(v[4 * ch], v[4 * ch + 1], v[4 * ch + 2], v[4 * ch + 3]);
        } else {
          for (int i = 0; i < 16 && col0 + i < args.NW; ++i) dst[i] = v[i];
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, args.tmem_cols);
  }
}

__global__ void k_reduce_partials(const float* __restrict__ part, int splits, int64_t kw, int64_t nw,
                                  float* __restrict__ out, int64_t ldo, int accumulate) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = kw * nw;
  if (i >= total) return;
  // four independent chains over the splits (short dependent-load chains),
  // combined in a fixed order: deterministic
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int k = 0;
  for (; k + 4 <= splits; k += 4) {
    s0 += part[k * total + i];
    s1 += part[(k + 1) * total + i];
    s2 += part[(k + 2) * total + i];
    s3 += part[(k + 3) * total + i];
  }
  for (; k < splits; ++k) s0 += part[k * total + i];
  const float s = (s0 + s1) + (s2 + s3);
  float* o = out + (i / nw) * ldo + (i % nw);
  *o = accumulate ? *o + s : s;
}

// ---- host: TMA descriptors through the driver entry point ---------------------------

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  if (!fn) fail(GGB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2D bf16 row-major tensor [rows][cols] with row stride ld (elements); box
// {box_inner (cols), box_outer (rows)}; 128-byte swizzle; OOB -> zeros.
// Tensor maps are a pure function of (address, shape, stride, box, kind):
// encoded once per distinct key (per host thread) instead of on every launch,
// which keeps the host ahead of the GPU for small batches.
struct TmapKey {
  const void* base;
  int64_t rows, cols, ld;
  int a, b;  // box (operand maps) or element size (output maps, a = -esize)
  bool operator==(const TmapKey& o) const {
    return base == o.base && rows == o.rows && cols == o.cols && ld == o.ld && a == o.a && b == o.b;
  }
};
struct TmapKeyHash {
  size_t operator()(const TmapKey& k) const {
    size_t h = std::hash<const void*>()(k.base);
    for (int64_t v : {k.rows, k.cols, k.ld, static_cast<int64_t>(k.a), static_cast<int64_t>(k.b)})
      h = h * 1000003u ^ std::hash<int64_t>()(v);
    return h;
  }
};
std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash>& tmap_cache() {
  thread_local std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> c;
  if (c.size() > 4096) c.clear();
  return c;
}

CUtensorMap encode_tmap(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_inner, int box_outer);
CUtensorMap make_tmap(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_inner, int box_outer) {
  const TmapKey k{base, rows, cols, ld, box_inner, box_outer};
  auto& c = tmap_cache();
  auto it = c.find(k);
  if (it != c.end()) return it->second;
  const CUtensorMap m = encode_tmap(base, rows, cols, ld, box_inner, box_outer);
  c.emplace(k, m);
  return m;
}

CUtensorMap encode_tmap(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_inner,
                        int box_outer) {
  require((reinterpret_cast<uintptr_t>(base) & 15) == 0, "gemm: operand must be 16-byte aligned");
  require((ld * 2) % 16 == 0, "gemm: leading dimension must be a multiple of 8 elements");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 2)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(GGB_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  return m;
}

// Output map for TMA stores: [rows][cols] with row stride ld elements of
// esize bytes, box {16 columns, 32 rows}, swizzle matching the 16-column row
// bytes (fp32 64 B, bf16 32 B). Out-of-bounds parts of a box are not written.
CUtensorMap encode_out_tmap(const void* base, int64_t rows, int64_t cols, int64_t ld, int esize);
CUtensorMap make_out_tmap(const void* base, int64_t rows, int64_t cols, int64_t ld, int esize) {
  const TmapKey k{base, rows, cols, ld, -esize, 0};
  auto& c = tmap_cache();
  auto it = c.find(k);
  if (it != c.end()) return it->second;
  const CUtensorMap m = encode_out_tmap(base, rows, cols, ld, esize);
  c.emplace(k, m);
  return m;
}

CUtensorMap encode_out_tmap(const void* base, int64_t rows, int64_t cols, int64_t ld, int esize) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esize)};
  cuuint32_t box[2] = {16, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           esize == 4 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(GGB_ECUDA, "cuTensorMapEncodeTiled (output) failed: " + std::to_string(r));
  return m;
}

// GGB_PEER_PUSH_TMA=0: mirrored GEMM outputs by a copy after the kernel
// instead of a second TMA store per tile
bool mirror_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("GGB_PEER_PUSH_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool tma_store_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("GGB_GEMM_TMA_STORE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

uint32_t tmem_cols_for(int n) {
  uint32_t c = 32;
  while (c < static_cast<uint32_t>(n)) c <<= 1;
  return c;
}

bool b_resident_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("GGB_GEMM_BRES");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace

// C[m x n] = A[m x k] . Bt[n x k]^T; with a_lo/bt_lo (same layouts) the
// operands are fp32 values carried as bf16 hi + lo pairs (split-bf16).
void gemm_bf16_impl(Ctx& ctx, int64_t m, int64_t n, int64_t k, const bf16* a, const bf16* a_lo, int64_t lda,
                    const bf16* bt, const bf16* bt_lo, int64_t ldb, float* c, int64_t ldc, bf16* cb, int64_t ldcb,
                    bf16* cl = nullptr) {
  if (m <= 0 || n <= 0) return;
  require(k > 0, "gemm: k must be positive");
  require(m < (int64_t{1} << 31) && n < (int64_t{1} << 31) && k < (int64_t{1} << 31), "gemm: dims");
  GemmArgs ga{};
  ga.M = static_cast<int>(m);
  ga.N = static_cast<int>(n);
  ga.K = static_cast<int>(k);
  ga.split = (a_lo != nullptr) ? 1 : 0;
  require((a_lo != nullptr) == (bt_lo != nullptr), "gemm: split mode needs both lo operands");
  ga.BN = static_cast<int>(std::min<int64_t>(256, round_up(n, 16)));
  ga.n_tiles = static_cast<int>(ceil_div(n, ga.BN));
  // B resident when it is a single n-tile and fits beside >= 2 A stages
  // (every tile then streams only A: the dX products, the out-head and the
  // K = d_in products); otherwise A and B stream together per stage
  const int parts = 1 + ga.split;
  const int64_t kch = ceil_div(k, kBK);
  const int64_t bres_bytes = kch * parts * ga.BN * kBK * 2;
  const int fixed = 1024 + kEpiSmem;
  const int a_stage = parts * kBM * kBK * 2;
  ga.b_res = (ga.n_tiles == 1 && b_resident_enabled() && fixed + bres_bytes + 2 * a_stage <= kSmemBudget) ? 1 : 0;
  const int stage_bytes = ga.b_res ? a_stage : parts * (kBM * kBK * 2 + ga.BN * kBK * 2);
  ga.stages = std::min<int64_t>(8, (kSmemBudget - fixed - (ga.b_res ? bres_bytes : 0)) / stage_bytes);
  require(ga.stages >= 2, "gemm: tile does not fit shared memory");
  ga.tmem_cols = tmem_cols_for(2 * ga.BN);
  ga.c = c;
  ga.ldc = ldc;
  ga.cb = cb;
  ga.cl = cb ? cl : nullptr;
  ga.ldcb = ldcb;
  const CUtensorMap ta = make_tmap(a, m, k, lda, kBK, kBM);
  const CUtensorMap tb = make_tmap(bt, n, k, ldb, kBK, ga.BN);
  const CUtensorMap tal = ga.split ? make_tmap(a_lo, m, k, lda, kBK, kBM) : ta;
  const CUtensorMap tbl = ga.split ? make_tmap(bt_lo, n, k, ldb, kBK, ga.BN) : tb;
  auto al16 = [](const void* p, int64_t ld, int es) {
    return p == nullptr || ((reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld * es) % 16 == 0);
  };
  ga.tma_out = tma_store_enabled() && al16(c, ldc, 4) && al16(cb, ldcb, 2) && al16(ga.cl, ldcb, 2) ? 1 : 0;
  CUtensorMap tc = ta, tcb = ta, tcl = ta;  // unused placeholders unless tma_out
  if (ga.tma_out) {
    if (c) tc = make_out_tmap(c, m, n, ldc, 4);
    if (cb) tcb = make_out_tmap(cb, m, n, ldcb, 2);
    if (ga.cl) tcl = make_out_tmap(ga.cl, m, n, ldcb, 2);
  }
  // push mode: mirror the one output (c or cb, no lo half) into the peer's slot
  bool mirror_after = false;
  if (ctx.out_mirror) {
    require(!ga.cl && ((c != nullptr) != (cb != nullptr)), "gemm: a mirrored output is exactly one of c / cb");
    if (ga.tma_out && mirror_tma_enabled()) {
      ga.mirror = c ? 1 : 2;
      tcl = c ? make_out_tmap(reinterpret_cast<char*>(c) + ctx.out_mirror, m, n, ldc, 4)
              : make_out_tmap(reinterpret_cast<char*>(cb) + ctx.out_mirror, m, n, ldcb, 2);
    } else {
      mirror_after = true;
    }
  }
  const int smem = ga.stages * stage_bytes + static_cast<int>(ga.b_res ? bres_bytes : 0) + 1024 + kEpiSmem;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    GGB_CUDA(cudaFuncSetAttribute(k_gemm_kmajor, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBudget));
  }
  const int64_t tiles = ceil_div(m, kBM) * ga.n_tiles;
  const int grid = static_cast<int>(std::min<int64_t>(tiles, std::min(sm_count(), ctx.persistent_sms())));
  k_gemm_kmajor<<<grid, kThreads, smem, ctx.stream>>>(ta, tb, tal, tbl, tc, tcb, tcl, ga);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
  if (mirror_after) {  // register epilogue: copy the finished block to the mirror
    if (c)
      GGB_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(c) + ctx.out_mirror, ldc * 4, c, ldc * 4, n * 4, m,
                                 cudaMemcpyDeviceToDevice, ctx.stream));
    else
      GGB_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(cb) + ctx.out_mirror, ldcb * 2, cb, ldcb * 2, n * 2, m,
                                 cudaMemcpyDeviceToDevice, ctx.stream));
  }
}

void gemm_bf16(Ctx& ctx, int64_t m, int64_t n, int64_t k, const bf16* a, int64_t lda, const bf16* bt, int64_t ldb,
               float* c, int64_t ldc, bf16* cb, int64_t ldcb) {
  gemm_bf16_impl(ctx, m, n, k, a, nullptr, lda, bt, nullptr, ldb, c, ldc, cb, ldcb);
}

void gemm_split(Ctx& ctx, int64_t m, int64_t n, int64_t k, const bf16* a_hi, const bf16* a_lo, int64_t lda,
                const bf16* bt_hi, const bf16* bt_lo, int64_t ldb, float* c, int64_t ldc, bf16* cb, int64_t ldcb,
                bf16* cl) {
  gemm_bf16_impl(ctx, m, n, k, a_hi, a_lo, lda, bt_hi, bt_lo, ldb, c, ldc, cb, ldcb, cl);
}

// DW[kw x nw] = X[m x kw]^T . DY[m x nw]; ws: scratch
void gemm_wgrad_bf16(Ctx& ctx, int64_t m, int64_t kw, int64_t nw, const bf16* x, int64_t ldx,
                     const bf16* dy, int64_t lddy, float* dw, int64_t lddw, DevBuf& ws, int accumulate) {
  if (kw <= 0 || nw <= 0) return;
  if (m <= 0) {
    if (accumulate) return;
    for (int64_t r = 0; r < kw; ++r)
      GGB_CUDA(cudaMemsetAsync(dw + r * lddw, 0, nw * 4, ctx.stream));
    return;
  }
  WgradArgs wa{};
  wa.M = static_cast<int>(m);
  wa.KW = static_cast<int>(kw);
  wa.NW = static_cast<int>(nw);
  wa.BN = static_cast<int>(std::min<int64_t>(256, round_up(nw, 64)));
  wa.n_tiles = static_cast<int>(ceil_div(nw, wa.BN));
  wa.m_tiles = static_cast<int>(ceil_div(kw, kBM));
  wa.MT = wa.m_tiles == 2 ? 2 : 1;  // both m-tiles in one CTA: the DY chunk is read once
  const int tiles = (wa.m_tiles / wa.MT) * wa.n_tiles;
  const int total_chunks = static_cast<int>(ceil_div(m, kBK));
  int splits = std::max(1, sm_count() / tiles);
  splits = std::min(splits, std::max(1, total_chunks / 4));
  // the fp32 partials (written, then reduced) stay within a quarter of the operand bytes
  const double operand_bytes = static_cast<double>(m) * (kw + nw) * 2;
  splits = std::min<int>(splits, std::max(1, static_cast<int>(operand_bytes / (4.0 * kw * nw * 4))));
  wa.chunks_per_split = static_cast<int>(ceil_div(total_chunks, splits));
  wa.splits = static_cast<int>(ceil_div(total_chunks, wa.chunks_per_split));
  const int stage_bytes = wa.MT * kBM * kBK * 2 + wa.BN * kBK * 2;
  wa.stages = std::min(8, (kSmemBudget - 1024 - 256) / stage_bytes);
  wa.tmem_cols = tmem_cols_for(wa.MT * wa.BN);
  wa.part = ws.reserve_n<float>(static_cast<size_t>(wa.splits) * kw * nw);
  const CUtensorMap tx = make_tmap(x, m, kw, ldx, 64, kBK);
  const CUtensorMap td = make_tmap(dy, m, nw, lddy, 64, kBK);
  const int smem = wa.stages * stage_bytes + 1024 + 256;
  static std::atomic<uint64_t> attr{0};
  if (first_on_device(attr)) {
    GGB_CUDA(cudaFuncSetAttribute(k_gemm_wgrad, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemBudget));
  }
  dim3 grid(tiles, wa.splits);
  k_gemm_wgrad<<<grid, kWgradThreads, smem, ctx.stream>>>(tx, td, wa);
  const int64_t total = kw * nw;
  k_reduce_partials<<<static_cast<unsigned>(ceil_div(total, 256)), 256, 0, ctx.stream>>>(
      wa.part, wa.splits, kw, nw, dw, lddw, accumulate);
  GGB_LAUNCH_CHECK();
  ctx.launches += 2;
}

}  // namespace ggb
