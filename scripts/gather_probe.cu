// Microbenchmark (not product code): random row-gather throughput on B200 as
// a function of row bytes, rows in flight per lane and lanes per row, to find
// what bounds the SpMM gathers. nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

template <int LPR, int VPL, int INF>  // lanes per row, uint4 per lane per row, rows in flight
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ F, int64_t row_u4, const int32_t* __restrict__ idx,
                                              int64_t n_idx, int per_group, uint4* __restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane / LPR, gl = lane % LPR;
  const int64_t grp = ((int64_t)blockIdx.x * 256 + threadIdx.x) / 32 * (32 / LPR) + g;
  const int64_t base = grp * per_group;
  if (base >= n_idx) return;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int k = 0; k < per_group; k += INF) {
    uint4 v[INF][VPL];
#pragma unroll
    for (int u = 0; u < INF; ++u) {
      const int64_t row = idx[(base + k + u) % n_idx];
#pragma unroll
      for (int q = 0; q < VPL; ++q) v[u][q] = __ldg(F + row * row_u4 + gl * VPL + q);
    }
#pragma unroll
    for (int u = 0; u < INF; ++u)
#pragma unroll
      for (int q = 0; q < VPL; ++q) { acc.x ^= v[u][q].x; acc.y += v[u][q].y; acc.z ^= v[u][q].z; acc.w += v[u][q].w; }
  }
  if (acc.x == 0x12345678) out[0] = acc;
}

template <int LPR, int VPL, int INF>
void run(const char* name, const uint4* F, int64_t nrows_total, const int32_t* idx, int64_t n_idx, uint4* out) {
  const int64_t row_u4 = (int64_t)LPR * VPL;  // row stride == gathered bytes
  const int per_group = 64;
  const int64_t groups = n_idx / per_group;
  const int64_t warps = groups / (32 / LPR);
  const int blocks = (int)((warps * 32 + 255) / 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<LPR, VPL, INF><<<blocks, 256>>>(F, row_u4, idx, n_idx, per_group, out);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) gather<LPR, VPL, INF><<<blocks, 256>>>(F, row_u4, idx, n_idx, per_group, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 5;
  const double rows = (double)groups * per_group;
  const double bytes = rows * row_u4 * 16;
  printf("%-28s row=%5lld B  %7.3f ms  %6.2f Grows/s  %7.1f GB/s\n", name, (long long)(row_u4 * 16), ms,
         rows / ms / 1e6, bytes / ms / 1e6);
  (void)nrows_total;
}

int main() {
  const size_t fbytes = (size_t)2 << 30;  // 2 GiB feature table (>> L2)
  uint4* F;
  cudaMalloc(&F, fbytes);
  cudaMemset(F, 1, fbytes);
  uint4* out;
  cudaMalloc(&out, 64);
  const int64_t n_idx = 8 << 20;  // 8M gathers (like C2's 8.35M nonzeros)
  int32_t* idx;
  cudaMalloc(&idx, n_idx * 4);
  auto make_idx = [&](int64_t row_bytes) {
    const int64_t nrows = fbytes / row_bytes;
    std::vector<int32_t> h(n_idx);
    uint64_t s = 12345;
    for (auto& x : h) {
      s = s * 6364136223846793005ULL + 1442695040888963407ULL;
      x = (int32_t)((s >> 33) % (uint64_t)nrows);
    }
    cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
    return nrows;
  };
  int64_t nr;
  nr = make_idx(256);
  run<16, 1, 4>("256B lpr16 vpl1 inf4", F, nr, idx, n_idx, out);
  run<16, 1, 8>("256B lpr16 vpl1 inf8", F, nr, idx, n_idx, out);
  run<8, 2, 8>("256B lpr8 vpl2 inf8", F, nr, idx, n_idx, out);
  nr = make_idx(512);
  run<32, 1, 4>("512B lpr32 vpl1 inf4", F, nr, idx, n_idx, out);
  run<32, 1, 8>("512B lpr32 vpl1 inf8", F, nr, idx, n_idx, out);
  run<16, 2, 4>("512B lpr16 vpl2 inf4", F, nr, idx, n_idx, out);
  run<16, 2, 8>("512B lpr16 vpl2 inf8", F, nr, idx, n_idx, out);
  run<8, 4, 4>("512B lpr8 vpl4 inf4", F, nr, idx, n_idx, out);
  run<8, 4, 8>("512B lpr8 vpl4 inf8", F, nr, idx, n_idx, out);
  nr = make_idx(1024);
  run<32, 2, 4>("1KB lpr32 vpl2 inf4", F, nr, idx, n_idx, out);
  run<32, 2, 8>("1KB lpr32 vpl2 inf8", F, nr, idx, n_idx, out);
  run<16, 4, 4>("1KB lpr16 vpl4 inf4", F, nr, idx, n_idx, out);
  nr = make_idx(2048);
  run<32, 4, 4>("2KB lpr32 vpl4 inf4", F, nr, idx, n_idx, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
