// Microbenchmark (not product code): can a column-chunked SpMM live in L2?
// Random gathers of a CH-byte chunk out of 1 KB rows (C2's fp32 feature rows,
// 612,500 rows = 627 MB), one chunk column per pass, all passes back to back:
// the working set of a pass is rows*CH bytes (78 MB at CH = 128). Compared
// against gathering the full 1 KB row once. 8.35M gathers per pass (C2 nnz).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather_probe l2_gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

template <int LPR, int INF>
__global__ void __launch_bounds__(512) gather(const uint4* __restrict__ F, int row_u4, int col_u4,
                                              const int32_t* __restrict__ idx, int64_t n_idx, int passes,
                                              uint4* __restrict__ out) {
  const int lane = threadIdx.x & 31, g = lane / LPR, gl = lane % LPR;
  constexpr int G = 32 / LPR;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t per = (n_idx + nwarps - 1) / nwarps;
  const int64_t b = warp * per, e = b + per < n_idx ? b + per : n_idx;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int p = 0; p < passes; ++p) {
    const int c0 = p * LPR + gl;
    for (int64_t k = b + g; k < e; k += G * INF) {
      uint4 v[INF];
#pragma unroll
      for (int u = 0; u < INF; ++u) {
        const int64_t kk = k + u * G;
        const int64_t row = kk < e ? idx[kk] : 0;
        v[u] = __ldg(F + row * row_u4 + c0);
      }
#pragma unroll
      for (int u = 0; u < INF; ++u) { acc.x ^= v[u].x; acc.y += v[u].y; acc.z ^= v[u].z; acc.w += v[u].w; }
    }
  }
  if (acc.x == 0x12345678) out[0] = acc;
  (void)col_u4;
}

template <int LPR, int INF>
void run(const char* name, const uint4* F, int row_u4, const int32_t* idx, int64_t n_idx, int passes, uint4* out,
         int blocks_per_sm, int threads) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * blocks_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<LPR, INF><<<blocks, threads>>>(F, row_u4, 0, idx, n_idx, passes, out);
  cudaEventRecord(a);
  const int it = 5;
  for (int i = 0; i < it; ++i) gather<LPR, INF><<<blocks, threads>>>(F, row_u4, 0, idx, n_idx, passes, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= it;
  const double bytes = (double)n_idx * passes * LPR * 16;
  printf("%-34s passes=%2d  %7.3f ms  gathered %7.1f GB/s\n", name, passes, ms, bytes / ms / 1e6);
}

int main() {
  const int64_t rows = 612500;
  const int row_u4 = 64;  // 1 KB rows
  uint4* F;
  cudaMalloc(&F, rows * row_u4 * 16);
  cudaMemset(F, 1, rows * row_u4 * 16);
  uint4* flush;
  cudaMalloc(&flush, 512 << 20);
  uint4* out;
  cudaMalloc(&out, 64);
  const int64_t n_idx = 8350000;
  int32_t* idx;
  cudaMalloc(&idx, n_idx * 4);
  std::vector<int32_t> h(n_idx);
  uint64_t s = 12345;
  for (auto& x : h) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    x = (int32_t)((s >> 33) % (uint64_t)rows);
  }
  cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
  // full 1 KB rows once (today's kernel's gather volume)
  run<32, 4>("full 1KB: 2x(32 lanes x16B)", F, row_u4, idx, n_idx, 2, out, 2, 512);
  // chunked passes, all chunks of the row: 1KB/CH passes
  run<2, 8>("CH=32B  lpr2 inf8", F, row_u4, idx, n_idx, 32, out, 2, 512);
  run<4, 8>("CH=64B  lpr4 inf8", F, row_u4, idx, n_idx, 16, out, 2, 512);
  run<4, 4>("CH=64B  lpr4 inf4", F, row_u4, idx, n_idx, 16, out, 2, 512);
  run<8, 4>("CH=128B lpr8 inf4", F, row_u4, idx, n_idx, 8, out, 2, 512);
  run<8, 8>("CH=128B lpr8 inf8", F, row_u4, idx, n_idx, 8, out, 2, 512);
  run<8, 8>("CH=128B lpr8 inf8 1blk", F, row_u4, idx, n_idx, 8, out, 1, 512);
  run<16, 4>("CH=256B lpr16 inf4", F, row_u4, idx, n_idx, 4, out, 2, 512);
  run<16, 8>("CH=256B lpr16 inf8", F, row_u4, idx, n_idx, 4, out, 2, 512);
  run<32, 4>("CH=512B lpr32 inf4", F, row_u4, idx, n_idx, 2, out, 2, 512);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
