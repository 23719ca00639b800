// Internal helpers shared by every translation unit of libggb.so.
#pragma once
#include <atomic>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ggb.h"

namespace ggb {

using bf16 = __nv_bfloat16;

// Errors map 1:1 onto the reference's exception types at the C++ mirror
// (cpp/gridgnn/ggb.hpp): kInval -> std::invalid_argument,
// kContract -> CommContract, kTimeout -> CommTimeout, others -> runtime_error.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const char* msg) {
  if (!ok) fail(GGB_EINVAL, msg);
}
inline void contract(bool ok, const char* msg) {
  if (!ok) fail(GGB_ECONTRACT, msg);
}

#define GGB_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      ::ggb::fail(GGB_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + \
                                 __FILE__ + ":" + std::to_string(__LINE__));               \
  } while (0)

#define GGB_LAUNCH_CHECK() GGB_CUDA(cudaGetLastError())

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

/// True the first time per CUDA device: kernel attributes set with
/// cudaFuncSetAttribute apply to the calling thread's current device, and one
/// process may drive several GPUs (the CLI runs a thread per rank).
inline bool first_on_device(std::atomic<uint64_t>& mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const uint64_t bit = uint64_t{1} << dev;
  return (mask.fetch_or(bit) & bit) == 0;
}
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

/// Grow-only device buffer; contents are not preserved on growth.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) {
    o.p = nullptr;
    o.bytes = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      bytes = o.bytes;
      o.p = nullptr;
      o.bytes = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void* reserve(size_t n) {
    if (n > bytes) {
      // per-step sizes (batch nonzeros, local rows) fluctuate by well under
      // a percent, and a cudaFree/cudaMalloc inside a step stalls the device:
      // large first allocations get 1/16 headroom, re-growth 1/4
      const bool regrow = bytes > 0;
      release();
      size_t want = n < 256 ? 256 : n;
      if (regrow)
        want += want / 4;
      else if (want >= (size_t(1) << 20))
        want += want / 16;
      GGB_CUDA(cudaMalloc(&p, want));
      bytes = want;
    }
    return p;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  template <class T>
  T* reserve_n(size_t n) {
    return static_cast<T*>(reserve(n * sizeof(T)));
  }
};

/// Pinned host staging for small device->host reads.
struct PinnedBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void* reserve(size_t n) {
    if (n > bytes) {
      if (p) cudaFreeHost(p);
      GGB_CUDA(cudaMallocHost(&p, n));
      bytes = n;
    }
    return p;
  }
};

/// A lazily created CUDA event owned by a host object.
struct EventHandle {
  cudaEvent_t e = nullptr;
  EventHandle() = default;
  EventHandle(const EventHandle&) = delete;
  EventHandle& operator=(const EventHandle&) = delete;
  ~EventHandle() {
    if (e) cudaEventDestroy(e);
  }
  cudaEvent_t get() {
    if (!e) GGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
  }
};

/// Reference block_partition (shardsample.cpp:8-17).
inline std::vector<int64_t> block_partition(int64_t n, int g) {
  require(g >= 1, "block_partition: g must be >= 1");
  std::vector<int64_t> off(static_cast<size_t>(g) + 1, 0);
  const int64_t base = n / g, extra = n % g;
  for (int k = 0; k < g; ++k) off[k + 1] = off[k] + base + (k < extra ? 1 : 0);
  return off;
}

// ---- grid + layout algebra (grid.hpp:11-73, tensor.hpp:14-44, pmm.hpp:31-63) ----
enum Axis : int { kD = 0, kX = 1, kY = 2, kZ = 3 };

struct Layout {
  int row, col;
  bool operator==(const Layout& o) const { return row == o.row && col == o.col; }
};

inline int third_axis(Layout l) { return 6 - l.row - l.col; }

inline Layout adjacency_layout(int layer) {
  switch ((layer - 1) % 3) {
    case 0: return {kZ, kX};
    case 1: return {kY, kZ};
    default: return {kX, kY};
  }
}
inline Layout feature_layout(int layer) {
  switch ((layer - 1) % 3) {
    case 0: return {kX, kY};
    case 1: return {kZ, kX};
    default: return {kY, kZ};
  }
}
inline Layout weight_layout_for(Layout h) { return {h.col, third_axis(h)}; }
inline Layout hagg_layout(int layer) { return {adjacency_layout(layer).row, feature_layout(layer).col}; }
inline Layout weight_layout(int layer) { return weight_layout_for(hagg_layout(layer)); }
constexpr Layout kInputFeatureLayout{kX, kZ};

struct Grid {
  int dims[4] = {1, 1, 1, 1};
  int total() const { return dims[0] * dims[1] * dims[2] * dims[3]; }
  void coord_of(int rank, int c[4]) const {
    c[3] = rank % dims[3];
    rank /= dims[3];
    c[2] = rank % dims[2];
    rank /= dims[2];
    c[1] = rank % dims[1];
    c[0] = rank / dims[1];
  }
  int rank_of(const int c[4]) const { return ((c[0] * dims[1] + c[1]) * dims[2] + c[2]) * dims[3] + c[3]; }
  int group_id(int axis, int rank) const {
    int c[4];
    coord_of(rank, c);
    int id = 0;
    for (int a = 0; a < 4; ++a) {
      if (a == axis) continue;
      id = id * dims[a] + c[a];
    }
    return id;
  }
};

}  // namespace ggb
