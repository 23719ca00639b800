#pragma once

#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>

#include "runtime.hpp"

namespace ggb {

struct Prefetcher {
  Ctx* consumer;
  const Graph* g;
  int64_t b;
  uint64_t seed, step0;
  Ctx sctx;  // sampling context: own stream + sampler scratch, same grid coords
  // batch slots: the producer may run up to kMaxSlots - 1 batches ahead
  // (GGB_PF_SLOTS, default 3: two builds in flight absorb a build that is
  // stretched by the training stream's kernels)
  static constexpr int kMaxSlots = 4;
  int nslots = 3;
  Batch slots[kMaxSlots];
  cudaEvent_t ready[kMaxSlots] = {}, released[kMaxSlots] = {};
  std::thread th;
  std::mutex m;
  std::condition_variable cv;
  int64_t produced = 0, consumed = 0, released_count = 0;
  bool stop = false, failed = false;
  std::exception_ptr err;
  // GGB_PF_TIMING=1: device time of each batch build on the sampling stream,
  // summed and printed at destruction (diagnostic; syncs on each batch)
  bool timing = false;
  cudaEvent_t tb[kMaxSlots] = {}, te[kMaxSlots] = {};
  double build_ms = 0.0;
  int64_t builds = 0;

  // dropout keep-bits generated ahead with each batch (drop_layers == 0: none)
  uint64_t run_seed = 0;
  int drop_layers = 0;
  int64_t d_h = 0;
  double rate = 0.0;

  Prefetcher(Ctx& consumer, const Graph& g, int64_t b, uint64_t seed, uint64_t first_step,
             uint64_t run_seed = 0, int drop_layers = 0, int64_t d_h = 0, double rate = 0.0);
  ~Prefetcher();
  void run();
  void make_masks(Batch& bt, uint64_t gstep);
  Batch* next();  // batch for step first_step + (number of previous calls)
};

}  // namespace ggb
