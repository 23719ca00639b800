// Device-wide exclusive prefix sum (reduce-then-scan, three launches).
// Used for CSR row pointers and the sampled-bitmap word prefix.
#include "runtime.hpp"

namespace ggb {
namespace {

constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // elements per block

template <class T>
__device__ T block_exclusive_scan(T v, T* warp_sums, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < (kScanThreads / 32) ? warp_sums[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < (kScanThreads / 32)) warp_sums[lane] = w;  // inclusive warp prefix
  }
  __syncthreads();
  const T before = warp ? warp_sums[warp - 1] : T(0);
  if (total) *total = warp_sums[kScanThreads / 32 - 1];
  return before + x - v;
}

template <class Tin, class Tout>
__global__ void k_tile_sums(const Tin* in, int64_t n, Tout* sums) {
  __shared__ Tout ws[kScanThreads / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  Tout s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + static_cast<int64_t>(k) * kScanThreads + threadIdx.x;
    if (i < n) s += static_cast<Tout>(in[i]);
  }
  Tout tot;
  block_exclusive_scan<Tout>(s, ws, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <class Tout>
__global__ void k_scan_sums(Tout* sums, int64_t m) {
  // one block scans all tile sums in place (exclusive), carrying across chunks
  __shared__ Tout ws[kScanThreads / 32];
  Tout carry = 0;
  for (int64_t base = 0; base < m; base += kScanThreads) {
    const int64_t i = base + threadIdx.x;
    const Tout v = i < m ? sums[i] : Tout(0);
    Tout tot;
    const Tout ex = block_exclusive_scan<Tout>(v, ws, &tot);
    __syncthreads();
    if (i < m) sums[i] = carry + ex;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[m] = carry;
}

template <class Tin, class Tout>
__global__ void k_tile_scan(const Tin* in, Tout* out, int64_t n, const Tout* sums) {
  __shared__ Tout ws[kScanThreads / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  // blocked arrangement: thread t owns items [base + t*K, base + t*K + K)
  Tout v[kScanItems];
  Tout s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + static_cast<int64_t>(threadIdx.x) * kScanItems + k;
    v[k] = i < n ? static_cast<Tout>(in[i]) : Tout(0);
    s += v[k];
  }
  Tout run = block_exclusive_scan<Tout>(s, ws, nullptr) + sums[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + static_cast<int64_t>(threadIdx.x) * kScanItems + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = sums[gridDim.x];
}

template <class Tin, class Tout>
void scan_impl(const Tin* in, Tout* out, int64_t n, DevBuf& tmp, cudaStream_t s) {
  const int64_t tiles = n > 0 ? ceil_div(n, kScanTile) : 1;
  Tout* sums = tmp.reserve_n<Tout>(static_cast<size_t>(tiles) + 1);
  k_tile_sums<Tin, Tout><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, n, sums);
  k_scan_sums<Tout><<<1, kScanThreads, 0, s>>>(sums, tiles);
  k_tile_scan<Tin, Tout><<<static_cast<unsigned>(tiles), kScanThreads, 0, s>>>(in, out, n, sums);
  GGB_LAUNCH_CHECK();
}

}  // namespace

void exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, DevBuf& tmp,
                               cudaStream_t s) {
  scan_impl<int32_t, long long>(in, reinterpret_cast<long long*>(out), n, tmp, s);
}

void exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, DevBuf& tmp, cudaStream_t s) {
  scan_impl<int32_t, int32_t>(in, out, n, tmp, s);
}

}  // namespace ggb
