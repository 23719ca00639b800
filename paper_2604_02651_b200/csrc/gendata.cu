// Synthetic dataset built on the device: the reference's
// generate_synthetic (dataset.cpp:85-131) with synthetic_edges
// (dataset.cpp:133-150) and normalize_adjacency (dataset.cpp:47-83), so graphs
// of papers100M scale (1.6G edges, 3.3G nonzeros) need no host pass.
//
//   edges     draw k of Stream(hash_combine(seed, 0xe0e0)) is splitmix64(s + k G)
//             (rng.hpp:26-45); next_below's rejections (probability < n / 2^64
//             per draw) are found first and skipped, so the accepted sequence is
//             the reference's exactly. Each pair (u, v), u != v, gives the keys
//             u n + v and v n + u; plus one self-loop key per vertex.
//   normalize radix sort of the keys, unique, row pointers by binary search,
//             value 1 / sqrt(deg_r deg_c) in IEEE fp64 (bit-identical).
//   features  Marsaglia polar over Stream(hash_combine(seed, 0xfea7)): attempt a
//             uses draws 2a, 2a+1; accepted attempts are ranked with per-block
//             counts and a block scan; the m-th accepted attempt gives values
//             2m, 2m+1 (rng.hpp:47-63). fp64 log is CUDA's (<= 1 ulp from the
//             host's), so a value can differ by one fp32 ulp from the host
//             generator in rare cases; everything else is bit-identical.
//   labels    degree-quantile classes (stable order by (degree, id)).
//   split     60/20/20 by element_unit(hash_combine(seed, 0x5b11), v, 0).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "gendata.hpp"
#include "runtime.hpp"
#include "rng.cuh"

namespace ggb {
namespace {

constexpr int kT = 256;
constexpr uint64_t kSentinel = ~uint64_t{0};

inline unsigned grid_for(int64_t n, int per_thread = 1) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kT * int64_t{per_thread}), 1 << 20)));
}

__global__ void k_edge_rejects(uint64_t s0, uint64_t draws, uint64_t limit, unsigned long long* cnt, uint64_t* pos,
                               int cap) {
  for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < draws;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (stream_draw(s0, k) >= limit) {
      const unsigned long long i = atomicAdd(cnt, 1ull);
      if (i < static_cast<unsigned long long>(cap)) pos[i] = k;
    }
  }
}

// stream index of the i-th accepted draw (rejections sorted ascending)
__device__ __forceinline__ uint64_t accepted_index(uint64_t i, const uint64_t* rej, int nrej) {
  uint64_t k = i;
  for (int j = 0; j < nrej; ++j)
    if (rej[j] <= k) ++k;
  return k;
}

__global__ void k_edge_keys(uint64_t s0, int64_t target, uint64_t n, const uint64_t* __restrict__ rej, int nrej,
                            uint64_t* __restrict__ keys) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < target;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t u = stream_draw(s0, accepted_index(2 * static_cast<uint64_t>(e), rej, nrej)) % n;
    const uint64_t v = stream_draw(s0, accepted_index(2 * static_cast<uint64_t>(e) + 1, rej, nrej)) % n;
    const bool keep = u != v;
    keys[2 * e] = keep ? u * n + v : kSentinel;
    keys[2 * e + 1] = keep ? v * n + u : kSentinel;
  }
}

__global__ void k_self_keys(int64_t n, uint64_t* __restrict__ keys) {
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x)
    keys[v] = static_cast<uint64_t>(v) * static_cast<uint64_t>(n) + static_cast<uint64_t>(v);
}

// row_ptr[r] = first sorted unique key >= r n
__global__ void k_row_ptr(const uint64_t* __restrict__ keys, int64_t nnz, int64_t n, int64_t* __restrict__ rp) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r <= n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t t = static_cast<uint64_t>(r) * static_cast<uint64_t>(n);
    int64_t lo = 0, hi = nnz;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < t)
        lo = mid + 1;
      else
        hi = mid;
    }
    rp[r] = lo;
  }
}

// one warp per row: column ids and 1 / sqrt(deg_r deg_c) (dataset.cpp:75-80)
__global__ void k_csr_fill(const uint64_t* __restrict__ keys, const int64_t* __restrict__ rp, int64_t n,
                           int32_t* __restrict__ col, double* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t b = rp[r], e = rp[r + 1];
    const double dr = static_cast<double>(e - b);
    const uint64_t base = static_cast<uint64_t>(r) * static_cast<uint64_t>(n);
    for (int64_t k = b + lane; k < e; k += 32) {
      const int64_t c = static_cast<int64_t>(keys[k] - base);
      col[k] = static_cast<int32_t>(c);
      if (val) {
        const double dc = static_cast<double>(rp[c + 1] - rp[c]);
        val[k] = __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(dr, dc)));
      }
    }
  }
}

// ---- features: Marsaglia polar with ranked acceptances ---------------------
constexpr int kAttemptsPerThread = 16;
constexpr int64_t kAttemptsPerBlock = int64_t{kT} * kAttemptsPerThread;

__device__ __forceinline__ bool polar_attempt(uint64_t s0, int64_t a, double& u, double& v, double& q) {
  const uint64_t x0 = stream_draw(s0, 2 * static_cast<uint64_t>(a));
  const uint64_t x1 = stream_draw(s0, 2 * static_cast<uint64_t>(a) + 1);
  // 2 * next_unit() - 1 (rng.hpp:35,54-55), each step rounded as the host does
  u = __dadd_rn(__dmul_rn(2.0, static_cast<double>(x0 >> 11) * 0x1.0p-53), -1.0);
  v = __dadd_rn(__dmul_rn(2.0, static_cast<double>(x1 >> 11) * 0x1.0p-53), -1.0);
  q = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
  return q < 1.0 && q != 0.0;
}

__global__ void k_polar_count(uint64_t s0, int64_t a0, int* __restrict__ counts) {
  const int64_t base = a0 + static_cast<int64_t>(blockIdx.x) * kAttemptsPerBlock + threadIdx.x * kAttemptsPerThread;
  int c = 0;
  double u, v, q;
  for (int i = 0; i < kAttemptsPerThread; ++i) c += polar_attempt(s0, base + i, u, v, q);
  using BR = cub::BlockReduce<int, kT>;
  __shared__ typename BR::TempStorage tmp;
  const int tot = BR(tmp).Sum(c);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void k_polar_write(uint64_t s0, int64_t a0, const int64_t* __restrict__ block_off, int64_t need,
                              int64_t total, float* __restrict__ out) {
  const int64_t base = a0 + static_cast<int64_t>(blockIdx.x) * kAttemptsPerBlock + threadIdx.x * kAttemptsPerThread;
  uint32_t flags = 0;
  double u, v, q;
  for (int i = 0; i < kAttemptsPerThread; ++i) flags |= static_cast<uint32_t>(polar_attempt(s0, base + i, u, v, q)) << i;
  using BS = cub::BlockScan<int, kT>;
  __shared__ typename BS::TempStorage tmp;
  int off;
  BS(tmp).ExclusiveSum(__popc(flags), off);
  int64_t k = block_off[blockIdx.x] + off;
  for (int i = 0; i < kAttemptsPerThread && k < need; ++i) {
    if (!((flags >> i) & 1u)) continue;
    polar_attempt(s0, base + i, u, v, q);
    const double f = sqrt(__ddiv_rn(__dmul_rn(-2.0, log(q)), q));
    if (2 * k < total) out[2 * k] = static_cast<float>(__dmul_rn(u, f));
    if (2 * k + 1 < total) out[2 * k + 1] = static_cast<float>(__dmul_rn(v, f));
    ++k;
  }
}

__global__ void k_degrees(const int64_t* __restrict__ rp, int64_t n, uint32_t* __restrict__ deg,
                          int32_t* __restrict__ ids) {
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    deg[v] = static_cast<uint32_t>(rp[v + 1] - rp[v] - 1);  // minus the self-loop
    ids[v] = static_cast<int32_t>(v);
  }
}

// full-graph row degrees (self-loop included): the normalized values are
// 1 / sqrt(deg_u deg_v) (dataset.cpp:78-79), recomputed wherever needed
__global__ void k_row_degrees(const int64_t* __restrict__ rp, int64_t n, int32_t* __restrict__ deg) {
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x)
    deg[v] = static_cast<int32_t>(rp[v + 1] - rp[v]);
}

__global__ void k_labels(const int32_t* __restrict__ order, int64_t n, int64_t n_classes, int32_t* __restrict__ labels) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    labels[order[i]] = static_cast<int32_t>((i * n_classes) / n);
}

__global__ void k_split(int64_t n, uint64_t key, uint8_t* __restrict__ split) {
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v < n;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double u = element_unit(key, static_cast<uint64_t>(v), 0);
    split[v] = u < 0.6 ? 0 : (u < 0.8 ? 1 : 2);
  }
}

// make_csr_shard (shardsample.cpp:19-45) on the device: rows [r0, r1) of a
// column-sorted CSR restricted to columns [c0, c1)
__global__ void k_shard_count(const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t r0,
                              int64_t rows, int64_t c0, int64_t c1, int64_t* __restrict__ lo, int32_t* __restrict__ cnt) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    auto lb = [&](int64_t b, int64_t e, int64_t x) {
      while (b < e) {
        const int64_t m = (b + e) >> 1;
        if (col[m] < x)
          b = m + 1;
        else
          e = m;
      }
      return b;
    };
    const int64_t b = rp[r0 + r], e = rp[r0 + r + 1];
    const int64_t l = lb(b, e, c0), h = lb(l, e, c1);
    lo[r] = l;
    cnt[r] = static_cast<int32_t>(h - l);
  }
}

__global__ void k_shard_fill(const int32_t* __restrict__ col, const double* __restrict__ val, int64_t rows,
                             const int64_t* __restrict__ lo, const int64_t* __restrict__ orp, int32_t* __restrict__ ocol,
                             double* __restrict__ oval) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < rows;
       r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t o = orp[r], len = orp[r + 1] - o, l = lo[r];
    for (int64_t k = lane; k < len; k += 32) {
      ocol[o + k] = col[l + k];
      if (oval) oval[o + k] = val[l + k];
    }
  }
}

// R-MAT edge draws (Chakrabarti et al.; Graph500 parameters a, b, c, d = 1-a-b-c):
// edge e descends `scale` levels of the adjacency quadtree, level k taking
// quadrant q(u) for u = unit(splitmix64(hash_combine(hash_combine(key, e), k)))
// (u < a: top-left, < a+b: top-right, < a+b+c: bottom-left, else
// bottom-right); the row/col bits of level k have weight 2^(scale-1-k).
// Counter-based, so every edge is independent and the list is a pure function
// of (scale, m, a, b, c, seed); oracle.c restates it for the parity tests.
__global__ void k_rmat(int scale, int64_t m, double a, double ab, double abc, uint64_t key,
                       int64_t* __restrict__ uv) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= m) return;
  const uint64_t ke = hash_combine(key, static_cast<uint64_t>(e));
  int64_t u = 0, v = 0;
  for (int k = 0; k < scale; ++k) {
    const double x = static_cast<double>(splitmix64(hash_combine(ke, static_cast<uint64_t>(k))) >> 11) * 0x1.0p-53;
    const int64_t bit = int64_t{1} << (scale - 1 - k);
    if (x >= abc) {
      u |= bit;
      v |= bit;
    } else if (x >= ab) {
      u |= bit;
    } else if (x >= a) {
      v |= bit;
    }
  }
  uv[2 * e] = u;
  uv[2 * e + 1] = v;
}

}  // namespace

void rmat_edges_device(Ctx& ctx, int scale, int64_t m, double a, double b, double c, uint64_t seed, int64_t* uv_dev) {
  require(scale >= 1 && scale <= 40, "rmat: scale must be in [1, 40]");
  require(m >= 0, "rmat: edge count must be >= 0");
  require(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0, "rmat: need a, b, c >= 0 and a + b + c <= 1");
  if (m == 0) return;
  k_rmat<<<static_cast<unsigned>(ceil_div(m, 256)), 256, 0, ctx.stream>>>(scale, m, a, a + b, a + b + c,
                                                                          hash_combine(seed, 0x7a3a7), uv_dev);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

namespace {

int bits_for(uint64_t x) {  // smallest b with 2^b > x
  int b = 0;
  while (b < 64 && (x >> b) != 0) ++b;
  return b;
}

}  // namespace

void generate_synthetic_device(Ctx& ctx, int64_t n, double avg_degree, int64_t d_in, int64_t n_classes,
                               uint64_t seed, DevDataset& ds) {
  require(n >= 1 && n < (int64_t{1} << 31) - 64, "generate_synthetic: n must be in [1, 2^31)");
  require(avg_degree >= 0, "generate_synthetic: avg_degree must be >= 0");
  require(n_classes >= 2, "generate_synthetic: n_classes must be >= 2");
  require(n_classes <= n, "generate_synthetic: n_classes > n");
  require(d_in >= 1, "generate_synthetic: d_in must be >= 1");
  cudaStream_t s = ctx.stream;
  ds.n = n;
  ds.d_in = d_in;
  ds.n_classes = n_classes;
  const int64_t target = n > 1 ? static_cast<int64_t>(avg_degree * static_cast<double>(n) / 2.0) : 0;

  // ---- edges -> keys
  const uint64_t se = hash_combine(seed, 0xe0e0);
  const uint64_t un = static_cast<uint64_t>(n);
  const uint64_t limit = UINT64_MAX - UINT64_MAX % un;
  constexpr int kRejCap = 64;
  DevBuf rejb;
  unsigned long long* d_cnt = rejb.reserve_n<unsigned long long>(1 + kRejCap);
  uint64_t* d_rej = reinterpret_cast<uint64_t*>(d_cnt + 1);
  GGB_CUDA(cudaMemsetAsync(d_cnt, 0, 8, s));
  const uint64_t draws = 2 * static_cast<uint64_t>(target) + kRejCap;
  if (target > 0) k_edge_rejects<<<grid_for(static_cast<int64_t>(draws), 8), kT, 0, s>>>(se, draws, limit, d_cnt,
                                                                                        d_rej, kRejCap);
  std::vector<unsigned long long> hr(1 + kRejCap, 0);
  GGB_CUDA(cudaMemcpyAsync(hr.data(), d_cnt, 8 * (1 + kRejCap), cudaMemcpyDeviceToHost, s));
  GGB_CUDA(cudaStreamSynchronize(s));
  const int nrej = static_cast<int>(hr[0]);
  require(nrej <= kRejCap / 2, "generate_synthetic: too many rejected draws");
  std::sort(hr.begin() + 1, hr.begin() + 1 + nrej);
  GGB_CUDA(cudaMemcpyAsync(d_rej, hr.data() + 1, 8 * std::max(nrej, 1), cudaMemcpyHostToDevice, s));

  const int64_t nkeys = 2 * target + n;
  DevBuf keys_a, keys_b, tmp;
  uint64_t* ka = keys_a.reserve_n<uint64_t>(static_cast<size_t>(nkeys));
  uint64_t* kb = keys_b.reserve_n<uint64_t>(static_cast<size_t>(nkeys));
  if (target > 0) k_edge_keys<<<grid_for(target, 4), kT, 0, s>>>(se, target, un, d_rej, nrej, ka);
  k_self_keys<<<grid_for(n, 4), kT, 0, s>>>(n, ka + 2 * target);
  GGB_LAUNCH_CHECK();
  // ---- sort + unique (the sentinel's low end_bit bits are all ones: it sorts last)
  const int end_bit = std::min(64, bits_for(un * un));
  size_t tb = 0;
  GGB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, ka, kb, nkeys, 0, end_bit, s));
  GGB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.reserve(tb), tb, ka, kb, nkeys, 0, end_bit, s));
  int64_t* d_nsel = reinterpret_cast<int64_t*>(d_cnt);
  size_t tb2 = 0;
  GGB_CUDA(cub::DeviceSelect::Unique(nullptr, tb2, kb, ka, d_nsel, nkeys, s));
  GGB_CUDA(cub::DeviceSelect::Unique(tmp.reserve(tb2), tb2, kb, ka, d_nsel, nkeys, s));
  int64_t nuniq = 0;
  GGB_CUDA(cudaMemcpyAsync(&nuniq, d_nsel, 8, cudaMemcpyDeviceToHost, s));
  uint64_t last = 0;
  GGB_CUDA(cudaStreamSynchronize(s));
  if (nuniq > 0) {
    GGB_CUDA(cudaMemcpyAsync(&last, ka + nuniq - 1, 8, cudaMemcpyDeviceToHost, s));
    GGB_CUDA(cudaStreamSynchronize(s));
  }
  const int64_t nnz = nuniq - (nuniq > 0 && last == kSentinel ? 1 : 0);
  keys_b.release();
  ds.nnz = nnz;
  int64_t* rp = ds.row_ptr.reserve_n<int64_t>(static_cast<size_t>(n) + 1);
  int32_t* col = ds.col.reserve_n<int32_t>(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
  double* val = ds.value_free ? nullptr : ds.val.reserve_n<double>(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
  k_row_ptr<<<grid_for(n + 1), kT, 0, s>>>(ka, nnz, n, rp);
  k_csr_fill<<<grid_for(n * 32), kT, 0, s>>>(ka, rp, n, col, val);
  if (ds.value_free)
    k_row_degrees<<<grid_for(n), kT, 0, s>>>(rp, n, ds.degree.reserve_n<int32_t>(static_cast<size_t>(n)));
  GGB_LAUNCH_CHECK();
  GGB_CUDA(cudaStreamSynchronize(s));
  keys_a.release();

  // ---- features
  {
    const uint64_t sf = hash_combine(seed, 0xfea7);
    const int64_t total = n * d_in;
    const int64_t need = (total + 1) / 2;
    float* out = ds.features.reserve_n<float>(static_cast<size_t>(total));
    int64_t blocks = ceil_div(static_cast<int64_t>(static_cast<double>(need) / 0.78) + 4096, kAttemptsPerBlock);
    DevBuf cnt_b, off_b;
    for (;;) {
      int* cnt = cnt_b.reserve_n<int>(static_cast<size_t>(blocks));
      k_polar_count<<<static_cast<unsigned>(blocks), kT, 0, s>>>(sf, 0, cnt);
      std::vector<int> hc(static_cast<size_t>(blocks));
      GGB_CUDA(cudaMemcpyAsync(hc.data(), cnt, 4 * blocks, cudaMemcpyDeviceToHost, s));
      GGB_CUDA(cudaStreamSynchronize(s));
      std::vector<int64_t> ho(static_cast<size_t>(blocks));
      int64_t acc = 0;
      for (int64_t b = 0; b < blocks; ++b) {
        ho[b] = acc;
        acc += hc[b];
      }
      if (acc < need) {
        blocks *= 2;
        continue;
      }
      int64_t* off = off_b.reserve_n<int64_t>(static_cast<size_t>(blocks));
      GGB_CUDA(cudaMemcpyAsync(off, ho.data(), 8 * blocks, cudaMemcpyHostToDevice, s));
      k_polar_write<<<static_cast<unsigned>(blocks), kT, 0, s>>>(sf, 0, off, need, total, out);
      GGB_LAUNCH_CHECK();
      GGB_CUDA(cudaStreamSynchronize(s));
      break;
    }
  }
  // ---- labels: stable order by (degree, id), equal buckets
  {
    DevBuf deg_a, deg_b, id_a, id_b;
    uint32_t* d0 = deg_a.reserve_n<uint32_t>(n);
    uint32_t* d1 = deg_b.reserve_n<uint32_t>(n);
    int32_t* i0 = id_a.reserve_n<int32_t>(n);
    int32_t* i1 = id_b.reserve_n<int32_t>(n);
    k_degrees<<<grid_for(n), kT, 0, s>>>(rp, n, d0, i0);
    size_t t3 = 0;
    GGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t3, d0, d1, i0, i1, n, 0, 32, s));
    GGB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.reserve(t3), t3, d0, d1, i0, i1, n, 0, 32, s));
    int32_t* labels = ds.labels.reserve_n<int32_t>(n);
    k_labels<<<grid_for(n), kT, 0, s>>>(i1, n, n_classes, labels);
    k_split<<<grid_for(n), kT, 0, s>>>(n, hash_combine(seed, 0x5b11), ds.split.reserve_n<uint8_t>(n));
    GGB_LAUNCH_CHECK();
    GGB_CUDA(cudaStreamSynchronize(s));
  }
  ctx.launches += 10;
}

void build_shard_device(Ctx& ctx, int64_t n, const DevDataset& ds, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                        PlaneShard& sh) {
  (void)n;
  cudaStream_t s = ctx.stream;
  sh.r0 = r0;
  sh.r1 = r1;
  sh.c0 = c0;
  sh.c1 = c1;
  const int64_t rows = r1 - r0;
  DevBuf lo_b, cnt_b, tmp;
  int64_t* lo = lo_b.reserve_n<int64_t>(static_cast<size_t>(std::max<int64_t>(rows, 1)));
  int32_t* cnt = cnt_b.reserve_n<int32_t>(static_cast<size_t>(std::max<int64_t>(rows, 1)));
  int64_t* orp = sh.row_ptr.reserve_n<int64_t>(static_cast<size_t>(rows) + 1);
  if (rows > 0)
    k_shard_count<<<grid_for(rows), kT, 0, s>>>(ds.row_ptr.as<int64_t>(), ds.col.as<int32_t>(), r0, rows, c0, c1, lo,
                                                 cnt);
  exclusive_scan_i32_to_i64(cnt, orp, rows, tmp, s);
  int64_t nnz = 0;
  GGB_CUDA(cudaMemcpyAsync(&nnz, orp + rows, 8, cudaMemcpyDeviceToHost, s));
  GGB_CUDA(cudaStreamSynchronize(s));
  sh.nnz = nnz;
  int32_t* ocol = sh.col.reserve_n<int32_t>(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
  double* oval = ds.value_free ? nullptr : sh.val.reserve_n<double>(static_cast<size_t>(std::max<int64_t>(nnz, 1)));
  if (rows > 0)
    k_shard_fill<<<grid_for(rows * 32), kT, 0, s>>>(ds.col.as<int32_t>(), oval ? ds.val.as<double>() : nullptr, rows,
                                                     lo, orp, ocol, oval);
  GGB_LAUNCH_CHECK();
  GGB_CUDA(cudaStreamSynchronize(s));
  ctx.launches += 3;
}

}  // namespace ggb
