// Per-kernel-class device timing with CUDA events recorded on the launching
// stream, plus the algorithmic bytes / flops of every timed launch, so the
// bench can report achieved GB/s or TFLOP/s against the roofline live.
#pragma once

#include <vector>

#include "runtime.hpp"

namespace ggb {

enum ProfCat : int {
  kProfSample = 0,  // sampling + induced-subgraph CSR build
  kProfSpmmFwd,
  kProfSpmmBwd,
  kProfGemmFwd,
  kProfGemmDx,
  kProfGemmWgrad,
  kProfElementwise,  // other element-wise passes (casts, split row statistics)
  kProfOptimizer,
  kProfComm,
  kProfFwdRow,  // fused RMSNorm + ReLU + dropout + residual (k_fwd_row)
  kProfBwdRow,  // fused element-wise + RMSNorm backward (k_bwd_row)
  kProfCe,      // cross-entropy
  kProfCats
};

struct Prof {
  bool on = false;
  struct Mark {
    int cat;
    cudaEvent_t a, b;
    double bytes, flops;
  };
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> pool;
  double ms[kProfCats] = {}, bytes[kProfCats] = {}, flops[kProfCats] = {};
  int64_t count[kProfCats] = {};
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    GGB_CUDA(cudaEventCreate(&e));
    return e;
  }
  ~Prof() {
    for (auto& m : marks) {
      cudaEventDestroy(m.a);
      cudaEventDestroy(m.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
  }
};

Prof& prof_of(Ctx& ctx);

struct ProfScope {
  Ctx& ctx;
  Prof* p = nullptr;
  int cat;
  cudaEvent_t a = nullptr;
  double bytes, flops;
  cudaStream_t s;  // the stream the range is timed on (the context's unless given)
  ProfScope(Ctx& c, int cat_, double bytes_ = 0, double flops_ = 0, cudaStream_t stream = nullptr)
      : ctx(c), cat(cat_), bytes(bytes_), flops(flops_), s(stream ? stream : c.stream) {
    Prof& pr = prof_of(ctx);
    if (!pr.on) return;
    p = &pr;
    a = p->get();
    GGB_CUDA(cudaEventRecord(a, s));
  }
  /// close the timed range early (e.g. before a collective timed on its own)
  void end() {
    if (!p) return;
    cudaEvent_t b = p->get();
    cudaEventRecord(b, s);
    p->marks.push_back({cat, a, b, bytes, flops});
    p = nullptr;
  }
  ~ProfScope() { end(); }
};

// Synchronizes the stream and folds the recorded marks into the totals.
void prof_collect(Ctx& ctx);

}  // namespace ggb
