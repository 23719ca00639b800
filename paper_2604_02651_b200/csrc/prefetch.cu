// Sampling / training overlap: the reference's prefetch producer
// (train_run's producer thread + PrefetchQueue, model.hpp:556-581 and
// 631-656) as a native producer thread with its own CUDA stream and sampler
// scratch. A ring of batch slots (the reference's queue holds one batch
// beside the one in use; here up to nslots - 1 are built ahead); the
// hand-off is by CUDA events, so the compute stream never blocks the host:
//   producer: wait(released[slot]) on the sampling stream -> build batch k ->
//             record ready[slot];
//   consumer: next() records released[previous slot] on the compute stream,
//             then makes the compute stream wait on ready[slot].
// Batches are bit-identical to the non-prefetched ones (same seeds/steps), as
// in the reference (acceptance criterion 8).
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "comm.hpp"
#include "ops.hpp"
#include "prefetch.hpp"
#include "prof.hpp"
#include "rng.cuh"
#include "trainer.hpp"

namespace ggb {

Prefetcher::Prefetcher(Ctx& consumer_, const Graph& g_, int64_t b_, uint64_t seed_, uint64_t first_step,
                       uint64_t run_seed_, int drop_layers_, int64_t d_h_, double rate_)
    : consumer(&consumer_), g(&g_), b(b_), seed(seed_), step0(first_step), run_seed(run_seed_),
      drop_layers(rate_ > 0.0 ? drop_layers_ : 0), d_h(d_h_), rate(rate_) {
  require(b >= 2 && b <= g->n, "prefetch: need 2 <= b <= N");
  require(rate >= 0.0 && rate < 1.0, "prefetch: dropout rate must be in [0, 1)");
  sctx.grid = consumer->grid;
  sctx.rank = consumer->rank;
  for (int a = 0; a < 4; ++a) sctx.coord[a] = consumer->coord[a];
  sctx.device = consumer->device;
  sctx.num_sms = consumer->num_sms;
  {
    const char* e = std::getenv("GGB_SIDE_SMALL");
    sctx.side_stream = !(e && e[0] == '0');
  }
  GGB_CUDA(cudaSetDevice(sctx.device));
  // lowest scheduling priority: sampling (and mask hashing) fill idle SM
  // slots without displacing the training stream's CTAs (measured ~2% faster
  // per step than equal priority at 1 and 2 GPUs). GGB_PREFETCH_PRIORITY=same
  // gives the sampling stream the training stream's priority instead.
  int least = 0, greatest = 0, prio = 0;
  GGB_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  prio = least;
  const char* pe = std::getenv("GGB_PREFETCH_PRIORITY");
  if (pe && std::string(pe) == "same") GGB_CUDA(cudaStreamGetPriority(consumer->stream, &prio));
  GGB_CUDA(cudaStreamCreateWithPriority(&sctx.stream, cudaStreamNonBlocking, prio));
  sctx.own_stream = true;
  {
    const char* e = std::getenv("GGB_PF_SLOTS");
    const int v = e ? std::atoi(e) : 3;
    nslots = v >= 2 && v <= kMaxSlots ? v : 3;
  }
  for (int s = 0; s < nslots; ++s) {
    GGB_CUDA(cudaEventCreateWithFlags(&ready[s], cudaEventDisableTiming));
    GGB_CUDA(cudaEventCreateWithFlags(&released[s], cudaEventDisableTiming));
  }
  {
    const char* e = std::getenv("GGB_PF_TIMING");
    timing = e && e[0] == '1';
    if (timing)
      for (int s = 0; s < nslots; ++s) {
        GGB_CUDA(cudaEventCreate(&tb[s]));
        GGB_CUDA(cudaEventCreate(&te[s]));
      }
  }
  th = std::thread([this] { run(); });
}

Prefetcher::~Prefetcher() {
  {
    std::lock_guard<std::mutex> lk(m);
    stop = true;
  }
  cv.notify_all();
  if (th.joinable()) th.join();
  cudaSetDevice(sctx.device);
  cudaStreamSynchronize(sctx.stream);
  for (int s = 0; s < nslots; ++s) {
    cudaEventDestroy(ready[s]);
    cudaEventDestroy(released[s]);
    if (timing) {
      cudaEventDestroy(tb[s]);
      cudaEventDestroy(te[s]);
    }
  }
  if (timing && builds > 0)
    std::fprintf(stderr, "[prefetch] %lld batch builds, %.3f ms device time each\n", static_cast<long long>(builds),
                 build_ms / static_cast<double>(builds));
}

void Prefetcher::run() {
  try {
    GGB_CUDA(cudaSetDevice(sctx.device));
    for (int64_t k = 0;; ++k) {
      const int slot = static_cast<int>(k % nslots);
      {
        std::unique_lock<std::mutex> lk(m);
        // slot free once the consumer has released batch k - nslots
        cv.wait(lk, [&] { return stop || released_count >= k - nslots + 1; });
        if (stop) return;
      }
      if (k >= nslots) GGB_CUDA(cudaStreamWaitEvent(sctx.stream, released[slot], 0));
      if (timing) GGB_CUDA(cudaEventRecord(tb[slot], sctx.stream));
      const bool pre = preagg_enabled() && preagg_in_prefetch();
      build_step_batch(sctx, *g, b, seed, step0 + static_cast<uint64_t>(k), slots[slot], pre);
      if (pre && preagg_eligible(sctx, slots[slot])) preaggregate(sctx, slots[slot]);
      if (drop_layers > 0) make_masks(slots[slot], step0 + static_cast<uint64_t>(k));
      if (timing) GGB_CUDA(cudaEventRecord(te[slot], sctx.stream));
      GGB_CUDA(cudaEventRecord(ready[slot], sctx.stream));
      {
        std::lock_guard<std::mutex> lk(m);
        produced = k + 1;
      }
      cv.notify_all();
    }
  } catch (...) {
    std::lock_guard<std::mutex> lk(m);
    err = std::current_exception();
    failed = true;
    cv.notify_all();
  }
}

// Keep-bits of every layer's output block (feature_layout(l+1), the block
// the forward's fused RMSNorm/ReLU/dropout kernel writes) for global step
// gstep, keyed exactly as detail::dropout_key (model.hpp:164-171).
void Prefetcher::make_masks(Batch& bt, uint64_t gstep) {
  bt.masks.resize(static_cast<size_t>(drop_layers));
  const uint64_t thresh = static_cast<uint64_t>(std::ceil(rate * 0x1.0p53));
  for (int l = 1; l <= drop_layers; ++l) {
    const Layout out = feature_layout(l + 1);
    const auto& ro = bt.batch_off[out.row];
    const auto co = block_partition(d_h, sctx.grid.dims[out.col]);
    DropMask& dm = bt.masks[l - 1];
    dm.key = dropout_key(run_seed, sctx.coord[0], gstep, l);
    dm.thresh = thresh;
    dm.r0 = ro[sctx.coord[out.row]];
    dm.rows = ro[sctx.coord[out.row] + 1] - dm.r0;
    dm.c0 = co[sctx.coord[out.col]];
    dm.cols = co[sctx.coord[out.col] + 1] - dm.c0;
    dm.ldm = mask_words(std::max<int64_t>(dm.cols, 1));
    uint32_t* bits = dm.bits.reserve_n<uint32_t>(std::max<int64_t>(dm.rows, 1) * dm.ldm);
    dropout_keep(sctx, dm.key, dm.rows, dm.cols, dm.r0, dm.c0, thresh, bits, dm.ldm);
  }
}

Batch* Prefetcher::next() {
  std::unique_lock<std::mutex> lk(m);
  if (consumed > 0) {  // release the batch handed out last time, once its compute is done
    const int prev = static_cast<int>((consumed - 1) % nslots);
    GGB_CUDA(cudaEventRecord(released[prev], consumer->stream));
    released_count = consumed;
    cv.notify_all();
  }
  cv.wait(lk, [&] { return failed || produced > consumed; });
  if (failed && produced <= consumed) std::rethrow_exception(err);
  const int slot = static_cast<int>(consumed % nslots);
  GGB_CUDA(cudaStreamWaitEvent(consumer->stream, ready[slot], 0));
  if (timing) {
    float ms = 0.f;
    GGB_CUDA(cudaEventSynchronize(te[slot]));
    GGB_CUDA(cudaEventElapsedTime(&ms, tb[slot], te[slot]));
    build_ms += ms;
    ++builds;
  }
  consumer->h2d_bytes += slots[slot].h2d_bytes;  // the batch's PCIe feature reads count for the consumer
  ++consumed;
  return &slots[slot];
}

}  // namespace ggb
