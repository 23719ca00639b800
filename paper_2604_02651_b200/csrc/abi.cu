// extern "C" boundary of libggb.so (include/ggb.h). Every entry point
// catches, records the message in a thread-local slot and returns a status
// code; nothing throws across the ABI.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cstring>
#include <mutex>
#include <thread>

#include "comm.hpp"
#include "gendata.hpp"
#include "layers.hpp"
#include "dataset.hpp"
#include "dsio.hpp"
#include "prefetch.hpp"
#include "prof.hpp"
#include "trainer.hpp"

struct ggb_ctx_s : ggb::Ctx {};
struct ggb_graph_s : ggb::Graph {};
struct ggb_dataset_s : ggb::HostDataset {
  std::vector<int64_t> uv;  // the raw edge list the adjacency was normalized from
};
struct ggb_batch_s : ggb::Batch {};
struct ggb_state_s : ggb::State {};
struct ggb_prefetch_s : ggb::Prefetcher {
  using ggb::Prefetcher::Prefetcher;
};

namespace ggb {

Ctx::~Ctx() {
  comm.reset();
  prof.reset();
  if (own_stream && stream) cudaStreamDestroy(stream);
}

Prof& prof_of(Ctx& ctx) {
  if (!ctx.prof) ctx.prof = std::make_unique<Prof>();
  return *ctx.prof;
}

void prof_collect(Ctx& ctx) {
  Prof& p = prof_of(ctx);
  if (p.marks.empty()) return;
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
  // GGB_PROF_TRACE=<dir>: every timed range of this collect as a timeline row
  // (class, start relative to the first range, duration, bytes) per rank
  static const char* trace_dir = std::getenv("GGB_PROF_TRACE");
  FILE* tf = nullptr;
  if (trace_dir) {
    GGB_CUDA(cudaDeviceSynchronize());
    tf = std::fopen((std::string(trace_dir) + "/trace_rank" + std::to_string(ctx.rank) + ".txt").c_str(), "a");
    if (tf) std::fprintf(tf, "# collect\n");
  }
  for (auto& m : p.marks) {
    float ms = 0.f;
    GGB_CUDA(cudaEventElapsedTime(&ms, m.a, m.b));
    if (tf) {
      float t0 = 0.f;
      cudaEventElapsedTime(&t0, p.marks.front().a, m.a);
      std::fprintf(tf, "%d %.4f %.4f %.0f\n", m.cat, t0, ms, m.bytes);
    }
    p.ms[m.cat] += ms;
    p.bytes[m.cat] += m.bytes;
    p.flops[m.cat] += m.flops;
    p.count[m.cat] += 1;
    p.pool.push_back(m.a);
    p.pool.push_back(m.b);
  }
  if (tf) std::fclose(tf);
  p.marks.clear();
}

namespace {

thread_local std::string g_err;
thread_local DevBuf g_ws;  // unit-test GEMM workspace

template <class F>
int guard(F&& f) {
  try {
    f();
    return GGB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("out of host memory: ") + e.what();
    return GGB_EINTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return GGB_EINTERNAL;
  }
}

void use_device(const Ctx& c) { GGB_CUDA(cudaSetDevice(c.device)); }

template <class T>
void upload(DevBuf& b, const T* host, size_t n, cudaStream_t s) {
  b.reserve(std::max<size_t>(n, 1) * sizeof(T));
  if (n) GGB_CUDA(cudaMemcpyAsync(b.p, host, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

template <class F>
void parallel_rows(int64_t n, F&& f) {
  const int T = static_cast<int>(std::max(1u, std::min(std::thread::hardware_concurrency(), 32u)));
  if (n < 65536 || T == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = ceil_div(n, T);
  for (int t = 0; t < T; ++t) {
    const int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

// make_csr_shard (shardsample.cpp:19-45) on the host, then upload.
void build_shard(Ctx& ctx, int64_t n, const int64_t* rp, const int64_t* col, const double* val, int64_t r0,
                 int64_t r1, int64_t c0, int64_t c1, PlaneShard& sh) {
  sh.r0 = r0;
  sh.r1 = r1;
  sh.c0 = c0;
  sh.c1 = c1;
  const int64_t rows = r1 - r0;
  std::vector<int64_t> lo(static_cast<size_t>(rows)), hi(static_cast<size_t>(rows));
  std::vector<int64_t> out_rp(static_cast<size_t>(rows) + 1, 0);
  const bool full_cols = c0 == 0 && c1 == n;
  parallel_rows(rows, [&](int64_t a, int64_t b) {
    for (int64_t r = a; r < b; ++r) {
      const int64_t* s = col + rp[r0 + r];
      const int64_t* e = col + rp[r0 + r + 1];
      lo[r] = full_cols ? rp[r0 + r] : std::lower_bound(s, e, c0) - col;
      hi[r] = full_cols ? rp[r0 + r + 1] : std::lower_bound(s, e, c1) - col;
    }
  });
  for (int64_t r = 0; r < rows; ++r) out_rp[r + 1] = out_rp[r] + (hi[r] - lo[r]);
  sh.nnz = out_rp[rows];
  std::vector<int32_t> c32(static_cast<size_t>(sh.nnz));
  std::vector<double> v64;
  const bool contiguous = full_cols;  // values are one contiguous range
  if (!contiguous) v64.resize(static_cast<size_t>(sh.nnz));
  parallel_rows(rows, [&](int64_t a, int64_t b) {
    for (int64_t r = a; r < b; ++r) {
      const int64_t o = out_rp[r];
      for (int64_t k = lo[r]; k < hi[r]; ++k) c32[o + k - lo[r]] = static_cast<int32_t>(col[k]);
      if (!contiguous) std::copy(val + lo[r], val + hi[r], v64.begin() + o);
    }
  });
  upload(sh.row_ptr, out_rp.data(), out_rp.size(), ctx.stream);
  upload(sh.col, c32.data(), c32.size(), ctx.stream);
  if (contiguous)
    upload(sh.val, val + rp[r0], static_cast<size_t>(sh.nnz), ctx.stream);
  else
    upload(sh.val, v64.data(), v64.size(), ctx.stream);
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));  // host vectors go out of scope
}

void host_transpose(int64_t n, const int64_t* rp, const int64_t* col, const double* val, std::vector<int64_t>& trp,
                    std::vector<int64_t>& tcol, std::vector<double>& tval) {
  const int64_t nnz = rp[n];
  trp.assign(static_cast<size_t>(n) + 1, 0);
  for (int64_t k = 0; k < nnz; ++k) ++trp[col[k] + 1];
  for (int64_t v = 0; v < n; ++v) trp[v + 1] += trp[v];
  tcol.resize(static_cast<size_t>(nnz));
  tval.resize(static_cast<size_t>(nnz));
  std::vector<int64_t> cur(trp.begin(), trp.end() - 1);
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rp[r]; k < rp[r + 1]; ++k) {
      const int64_t s = cur[col[k]]++;
      tcol[s] = r;
      tval[s] = val[k];
    }
}

void graph_build(Ctx& ctx, Graph& g, int64_t n, const int64_t* rp, const int64_t* col, const double* val,
                 bool symmetric, int64_t d_in, const float* feats, int64_t n_classes, const int32_t* labels,
                 int layers) {
  require(n >= 1 && n < (int64_t{1} << 31) - 64, "graph: n must be in [1, 2^31)");
  require(layers >= 1, "graph: layers must be >= 1");
  require(rp[0] == 0, "graph: row_ptr must start at 0");
  g.ctx = &ctx;
  g.n = n;
  g.nnz = rp[n];
  g.d_in = d_in;
  g.n_classes = n_classes;
  g.layers = layers;
  g.planes = std::min(layers, 3);
  std::vector<int64_t> trp, tcol;
  std::vector<double> tval;
  const int64_t *Trp = rp, *Tcol = col;
  const double* Tval = val;
  struct Key {
    int t;
    int64_t r0, r1, c0, c1;
  };
  std::vector<Key> keys;
  g.shards.clear();
  g.fwd_of.assign(g.planes, -1);
  g.tr_of.assign(g.planes, -1);
  auto get = [&](int t, int64_t r0, int64_t r1, int64_t c0, int64_t c1) {
    // a symmetric matrix is its own transpose
    if (symmetric) t = 0;
    for (size_t k = 0; k < keys.size(); ++k)
      if (keys[k].t == t && keys[k].r0 == r0 && keys[k].r1 == r1 && keys[k].c0 == c0 && keys[k].c1 == c1)
        return static_cast<int>(k);
    if (t == 1 && trp.empty()) {
      host_transpose(n, rp, col, val, trp, tcol, tval);
      Trp = trp.data();
      Tcol = tcol.data();
      Tval = tval.data();
    }
    keys.push_back({t, r0, r1, c0, c1});
    g.shards.emplace_back();
    if (t == 0)
      build_shard(ctx, n, rp, col, val, r0, r1, c0, c1, g.shards.back());
    else
      build_shard(ctx, n, Trp, Tcol, Tval, r0, r1, c0, c1, g.shards.back());
    return static_cast<int>(keys.size() - 1);
  };
  for (int p = 0; p < g.planes; ++p) {
    const Layout lay = adjacency_layout(p + 1);
    const auto ro = block_partition(n, ctx.grid.dims[lay.row]);
    const auto co = block_partition(n, ctx.grid.dims[lay.col]);
    const int64_t r0 = ro[ctx.coord[lay.row]], r1 = ro[ctx.coord[lay.row] + 1];
    const int64_t c0 = co[ctx.coord[lay.col]], c1 = co[ctx.coord[lay.col] + 1];
    g.fwd_of[p] = get(0, r0, r1, c0, c1);
    g.tr_of[p] = get(1, c0, c1, r0, r1);
  }
  // feature Z-slice (kInputFeatureLayout.col) and labels
  const auto fo = block_partition(d_in, ctx.grid.dims[kInputFeatureLayout.col]);
  g.feat_c0 = fo[ctx.coord[kInputFeatureLayout.col]];
  g.feat_c1 = fo[ctx.coord[kInputFeatureLayout.col] + 1];
  const int64_t fw = g.feat_c1 - g.feat_c0;
  if (fw == d_in) {
    upload(g.features, feats, static_cast<size_t>(n * d_in), ctx.stream);
  } else {
    std::vector<float> sl(static_cast<size_t>(n * fw));
    for (int64_t v = 0; v < n; ++v) std::copy(feats + v * d_in + g.feat_c0, feats + v * d_in + g.feat_c1, sl.begin() + v * fw);
    upload(g.features, sl.data(), sl.size(), ctx.stream);
    GGB_CUDA(cudaStreamSynchronize(ctx.stream));
  }
  upload(g.labels, labels, static_cast<size_t>(n), ctx.stream);
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
  g.feat_ptr = g.features.as<float>();
  g.device_bytes = g.features.bytes + g.labels.bytes;
  for (auto& s : g.shards) g.device_bytes += s.row_ptr.bytes + s.col.bytes + s.val.bytes;
  for (auto& s : g.shards) shard_degree_profile(ctx, s);
}

// graph_build from a device-generated dataset (gendata.cu): the plane
// shards are cut on the device; a full-matrix shard takes the CSR buffers
// over, so a 1x1x1 grid holds exactly one copy of the adjacency.
void graph_build_device(Ctx& ctx, Graph& g, DevDataset& ds, int layers) {
  const int64_t n = ds.n;
  require(layers >= 1, "graph: layers must be >= 1");
  g.ctx = &ctx;
  g.n = n;
  g.nnz = ds.nnz;
  g.d_in = ds.d_in;
  g.n_classes = ds.n_classes;
  g.layers = layers;
  g.planes = std::min(layers, 3);
  g.shards.clear();
  g.fwd_of.assign(g.planes, -1);
  g.tr_of.assign(g.planes, -1);
  struct Key {
    int64_t r0, r1, c0, c1;
  };
  std::vector<Key> keys;
  auto get = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) {  // A == A^T: one key space
    for (size_t k = 0; k < keys.size(); ++k)
      if (keys[k].r0 == r0 && keys[k].r1 == r1 && keys[k].c0 == c0 && keys[k].c1 == c1) return static_cast<int>(k);
    keys.push_back({r0, r1, c0, c1});
    return static_cast<int>(keys.size() - 1);
  };
  for (int p = 0; p < g.planes; ++p) {
    const Layout lay = adjacency_layout(p + 1);
    const auto ro = block_partition(n, ctx.grid.dims[lay.row]);
    const auto co = block_partition(n, ctx.grid.dims[lay.col]);
    const int64_t r0 = ro[ctx.coord[lay.row]], r1 = ro[ctx.coord[lay.row] + 1];
    const int64_t c0 = co[ctx.coord[lay.col]], c1 = co[ctx.coord[lay.col] + 1];
    g.fwd_of[p] = get(r0, r1, c0, c1);
    g.tr_of[p] = get(c0, c1, r0, r1);
  }
  g.shards.resize(keys.size());
  int full = -1;
  for (size_t k = 0; k < keys.size(); ++k) {
    const Key& kk = keys[k];
    if (kk.r0 == 0 && kk.r1 == n && kk.c0 == 0 && kk.c1 == n) {
      full = static_cast<int>(k);
      continue;
    }
    build_shard_device(ctx, n, ds, kk.r0, kk.r1, kk.c0, kk.c1, g.shards[k]);
  }
  if (full >= 0) {
    PlaneShard& sh = g.shards[full];
    sh.r0 = sh.c0 = 0;
    sh.r1 = sh.c1 = n;
    sh.nnz = ds.nnz;
    sh.row_ptr = std::move(ds.row_ptr);
    sh.col = std::move(ds.col);
    sh.val = std::move(ds.val);
  }
  const auto fo = block_partition(ds.d_in, ctx.grid.dims[kInputFeatureLayout.col]);
  g.feat_c0 = fo[ctx.coord[kInputFeatureLayout.col]];
  g.feat_c1 = fo[ctx.coord[kInputFeatureLayout.col] + 1];
  const int64_t fw = g.feat_c1 - g.feat_c0;
  if (fw == ds.d_in) {
    g.features = std::move(ds.features);
  } else {
    float* dst = g.features.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(n * fw, 1)));
    GGB_CUDA(cudaMemcpy2DAsync(dst, fw * 4, ds.features.as<float>() + g.feat_c0, ds.d_in * 4, fw * 4, n,
                               cudaMemcpyDeviceToDevice, ctx.stream));
    GGB_CUDA(cudaStreamSynchronize(ctx.stream));
    ds.features.release();
  }
  g.labels = std::move(ds.labels);
  g.split = std::move(ds.split);
  g.value_free = ds.value_free;
  g.degree = std::move(ds.degree);
  g.feat_ptr = g.features.as<float>();
  g.device_bytes = g.features.bytes + g.labels.bytes + g.split.bytes + g.degree.bytes;
  for (auto& s : g.shards) g.device_bytes += s.row_ptr.bytes + s.col.bytes + s.val.bytes;
  for (auto& s : g.shards) shard_degree_profile(ctx, s);
}

template <class T>
void download(T* host, const void* dev, size_t n, cudaStream_t s) {
  if (n == 0 || !host) return;
  GGB_CUDA(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  GGB_CUDA(cudaStreamSynchronize(s));
}

// Split tags (Dataset::split, dataset.hpp:23), validated as load_dataset
// does (dataset.cpp:222-229).
void set_split(Graph& g, const uint8_t* split) {
  for (int64_t v = 0; v < g.n; ++v)
    if (split[v] > 3) fail(GGB_EINVAL, "graph_set_split: invalid split tag at vertex " + std::to_string(v));
  const size_t old = g.split.bytes;
  upload(g.split, split, static_cast<size_t>(g.n), g.ctx->stream);
  GGB_CUDA(cudaStreamSynchronize(g.ctx->stream));
  g.device_bytes += g.split.bytes - old;
}

}  // namespace
}  // namespace ggb

using namespace ggb;

extern "C" {

const char* ggb_last_error(void) { return g_err.c_str(); }
int ggb_version(void) { return 1; }

int ggb_get_unique_id(uint8_t out[128]) {
  return guard([&] { comm_get_unique_id(out); });
}

int ggb_device_count(int32_t* out) {
  return guard([&] {
    *out = 0;
    int n = 0;
    GGB_CUDA(cudaGetDeviceCount(&n));
    *out = n;
  });
}

int ggb_ctx_create(const int32_t dims[4], int32_t rank, int32_t device, const uint8_t* nccl_uid, void* stream,
                   ggb_ctx_t* out) {
  return guard([&] {
    require(dims && out, "ctx: null argument");
    for (int a = 0; a < 4; ++a) require(dims[a] >= 1, "DeviceGrid: dims must be >= 1");
    auto c = std::make_unique<ggb_ctx_s>();
    for (int a = 0; a < 4; ++a) c->grid.dims[a] = dims[a];
    require(rank >= 0 && rank < c->grid.total(), "ctx: rank out of range");
    c->rank = rank;
    c->grid.coord_of(rank, c->coord);
    c->device = device;
    GGB_CUDA(cudaSetDevice(device));
    GGB_CUDA(cudaFree(nullptr));  // establish the primary context
    int sms = 0;
    GGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    c->num_sms = sms;
    {  // GGB_SM_RESERVE=R: persistent kernels leave R SMs to the sampling stream
      const char* e = std::getenv("GGB_SM_RESERVE");
      const int r = e ? std::atoi(e) : 0;
      c->sm_reserve = r >= 0 && r < sms / 2 ? r : 0;
    }
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      GGB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    if (nccl_uid && c->grid.total() > 1) {
      c->comm = comm_create(c->grid, rank, nccl_uid);
      peer_setup(*c);  // every rank is here together: decide the peer-memory groups now
    }
    *out = c.release();
  });
}

int ggb_ctx_destroy(ggb_ctx_t ctx) {
  return guard([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    delete ctx;
  });
}

int ggb_ctx_set_stream(ggb_ctx_t ctx, void* stream) {
  return guard([&] {
    require(ctx != nullptr, "ctx: null");
    if (ctx->own_stream && ctx->stream) {
      GGB_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaStreamDestroy(ctx->stream);
      ctx->own_stream = false;
    }
    if (stream) {
      ctx->stream = static_cast<cudaStream_t>(stream);
    } else {
      GGB_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
    }
  });
}

int ggb_ctx_synchronize(ggb_ctx_t ctx) {
  return guard([&] {
    use_device(*ctx);
    sync_stream(*ctx, ctx->stream);  // with the collective watchdog (CommTimeout)
  });
}

int ggb_ctx_set_comm_timeout(ggb_ctx_t ctx, int64_t timeout_ms) {
  return guard([&] {
    require(timeout_ms > 0, "comm timeout must be positive");
    if (ctx->comm) ctx->comm->timeout_ms = timeout_ms;
  });
}

int ggb_ctx_counters(ggb_ctx_t ctx, uint64_t* counters) {
  return guard([&] {
    counters[0] = ctx->launches;
    counters[1] = ctx->h2d_bytes;
    counters[2] = ctx->d2h_bytes;
  });
}

int ggb_ctx_comm_stats(ggb_ctx_t ctx, int32_t grid_total, int32_t reset, uint64_t* out) {
  return guard([&] {
    require(out != nullptr, "comm_stats: null output");
    const CommStats& cs = ctx->stats;
    uint64_t v[GGB_COMM_STATS_LEN];
    for (int a = 0; a < 4; ++a) {
      for (int p = 0; p < kNumPhases; ++p) v[a * kNumPhases + p] = cs.bytes[a][p];
      v[4 * kNumPhases + a] = cs.allreduce_calls[a];
      v[4 * kNumPhases + 4 + a] = cs.allgather_calls[a];
    }
    if (grid_total) {  // Communicator::snapshot (comm.hpp:224-236): the sum over every rank of the grid
      use_device(*ctx);
      DevBuf tmp;
      uint64_t* d = tmp.reserve_n<uint64_t>(GGB_COMM_STATS_LEN);
      GGB_CUDA(cudaMemcpyAsync(d, v, sizeof(v), cudaMemcpyHostToDevice, ctx->stream));
      for (int a = 0; a < 4; ++a) all_reduce_u64(*ctx, a, d, GGB_COMM_STATS_LEN);
      GGB_CUDA(cudaMemcpyAsync(v, d, sizeof(v), cudaMemcpyDeviceToHost, ctx->stream));
      GGB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    for (int i = 0; i < GGB_COMM_STATS_LEN; ++i) out[i] = v[i];
    if (reset) ctx->stats = CommStats{};
  });
}

int ggb_ctx_profile(ggb_ctx_t ctx, int32_t enable) {
  return guard([&] {
    use_device(*ctx);
    prof_collect(*ctx);
    prof_of(*ctx).on = enable != 0;
  });
}

int ggb_ctx_profile_read(ggb_ctx_t ctx, double* ms, double* bytes, double* flops, int64_t* counts, int32_t reset) {
  return guard([&] {
    use_device(*ctx);
    prof_collect(*ctx);
    Prof& p = prof_of(*ctx);
    for (int c = 0; c < kProfCats; ++c) {
      if (ms) ms[c] = p.ms[c];
      if (bytes) bytes[c] = p.bytes[c];
      if (flops) flops[c] = p.flops[c];
      if (counts) counts[c] = p.count[c];
      if (reset) {
        p.ms[c] = p.bytes[c] = p.flops[c] = 0.0;
        p.count[c] = 0;
      }
    }
  });
}

int ggb_sample_vertices(ggb_ctx_t ctx, int64_t n, int64_t b, uint64_t seed, uint64_t step, int64_t* host_out) {
  return guard([&] {
    use_device(*ctx);
    require(b >= 1 && b <= n, "sample_vertices: need 1 <= b <= n");
    DevBuf out;
    int64_t* d = out.reserve_n<int64_t>(b);
    sample_set(*ctx, n, b, seed, step, d);
    download(host_out, d, static_cast<size_t>(b), ctx->stream);
  });
}

int ggb_sample_vertices_test_reject(ggb_ctx_t ctx, int64_t n, int64_t b, uint64_t seed, uint64_t step,
                                    uint64_t reject_mod, int64_t* host_out) {
  return guard([&] {
    use_device(*ctx);
    require(b >= 1 && b <= n, "sample_vertices: need 1 <= b <= n");
    DevBuf out;
    int64_t* d = out.reserve_n<int64_t>(b);
    sample_set(*ctx, n, b, seed, step, d, reject_mod);
    download(host_out, d, static_cast<size_t>(b), ctx->stream);
  });
}

int ggb_graph_create(ggb_ctx_t ctx, int64_t n, const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                     int32_t symmetric, int64_t d_in, const float* features, int64_t n_classes,
                     const int32_t* labels, int32_t layers, ggb_graph_t* out) {
  return guard([&] {
    use_device(*ctx);
    require(row_ptr && col_idx && values && features && labels && out, "graph: null argument");
    auto g = std::make_unique<ggb_graph_s>();
    graph_build(*ctx, *g, n, row_ptr, col_idx, values, symmetric != 0, d_in, features, n_classes, labels, layers);
    *out = g.release();
  });
}

int ggb_graph_generate_synthetic(ggb_ctx_t ctx, int64_t n, double avg_degree, int64_t d_in, int64_t n_classes,
                                 uint64_t seed, int32_t layers, ggb_graph_t* out) {
  return guard([&] {
    use_device(*ctx);
    HostDataset ds = generate_synthetic(n, avg_degree, d_in, n_classes, seed);
    auto g = std::make_unique<ggb_graph_s>();
    graph_build(*ctx, *g, n, ds.adj.row_ptr.data(), ds.adj.col.data(), ds.adj.val.data(), true, d_in,
                ds.features.data(), n_classes, ds.labels.data(), layers);
    set_split(*g, ds.split.data());
    *out = g.release();
  });
}

int ggb_graph_generate_synthetic_device(ggb_ctx_t ctx, int64_t n, double avg_degree, int64_t d_in,
                                        int64_t n_classes, uint64_t seed, int32_t layers, ggb_graph_t* out) {
  return guard([&] {
    require(out != nullptr, "graph: null handle slot");
    use_device(*ctx);
    auto g = std::make_unique<ggb_graph_s>();
    {
      DevDataset ds;
      // value-free shards (GGB_VALUE_FREE=0 keeps the fp64 value arrays): the
      // values are 1 / sqrt(deg_u deg_v) of the generated graph, recomputed
      // exactly in the batch extraction; 8 bytes per nonzero less HBM
      const char* vf = std::getenv("GGB_VALUE_FREE");
      ds.value_free = !(vf && vf[0] == '0');
      generate_synthetic_device(*ctx, n, avg_degree, d_in, n_classes, seed, ds);
      graph_build_device(*ctx, *g, ds, layers);
    }
    *out = g.release();
  });
}

int ggb_graph_export(ggb_graph_t g, int64_t* row_ptr, int64_t* col_idx, double* values, float* features,
                     int32_t* labels, uint8_t* split) {
  return guard([&] {
    require(g != nullptr, "graph_export: null graph");
    use_device(*g->ctx);
    cudaStream_t s = g->ctx->stream;
    const PlaneShard* full = nullptr;
    for (const auto& sh : g->shards)
      if (sh.r0 == 0 && sh.r1 == g->n && sh.c0 == 0 && sh.c1 == g->n) full = &sh;
    if (row_ptr || col_idx || values) {
      require(full != nullptr, "graph_export: no full-matrix shard on this rank (1x1x1 grids only)");
      download(row_ptr, full->row_ptr.p, static_cast<size_t>(g->n) + 1, s);
      if (col_idx) {
        std::vector<int32_t> c(static_cast<size_t>(full->nnz));
        download(c.data(), full->col.p, c.size(), s);
        std::copy(c.begin(), c.end(), col_idx);
      }
      if (values && g->value_free) {  // recompute 1 / sqrt(deg_u deg_v) (dataset.cpp:78-79)
        std::vector<int64_t> rp(static_cast<size_t>(g->n) + 1);
        std::vector<int32_t> c(static_cast<size_t>(full->nnz));
        download(rp.data(), full->row_ptr.p, rp.size(), s);
        download(c.data(), full->col.p, c.size(), s);
        for (int64_t u = 0; u < g->n; ++u)
          for (int64_t k = rp[u]; k < rp[u + 1]; ++k)
            values[k] = 1.0 / std::sqrt(static_cast<double>(rp[u + 1] - rp[u]) *
                                        static_cast<double>(rp[c[k] + 1] - rp[c[k]]));
      } else {
        download(values, full->val.p, static_cast<size_t>(full->nnz), s);
      }
    }
    if (features) {
      require(!g->features_on_host() && g->feat_c0 == 0 && g->feat_c1 == g->d_in,
              "graph_export: features are not a full device copy on this rank");
      download(features, g->features.p, static_cast<size_t>(g->n * g->d_in), s);
    }
    download(labels, g->labels.p, static_cast<size_t>(g->n), s);
    if (split) {
      require(g->split.bytes >= static_cast<size_t>(g->n), "graph_export: no split tags");
      download(split, g->split.p, static_cast<size_t>(g->n), s);
    }
  });
}

// ---- host datasets and their files (dataset.cpp:152-280) --------------
int ggb_dataset_load(const char* edges, const char* features, const char* labels, const char* split,
                     ggb_dataset_t* out) {
  return guard([&] {
    require(edges && features && labels && split && out, "dataset_load: null argument");
    auto d = std::make_unique<ggb_dataset_s>();
    static_cast<HostDataset&>(*d) = load_dataset(edges, features, labels, split, &d->uv);
    *out = d.release();
  });
}

int ggb_dataset_generate_synthetic(int64_t n, double avg_degree, int64_t d_in, int64_t n_classes, uint64_t seed,
                                   ggb_dataset_t* out) {
  return guard([&] {
    require(out != nullptr, "dataset: null handle slot");
    auto d = std::make_unique<ggb_dataset_s>();
    static_cast<HostDataset&>(*d) = generate_synthetic(n, avg_degree, d_in, n_classes, seed);
    d->uv = synthetic_edges(n, avg_degree, seed);
    *out = d.release();
  });
}

int ggb_rmat_edges(ggb_ctx_t ctx, int32_t scale, int64_t m, double a, double b, double c, uint64_t seed,
                   int64_t* host_uv) {
  return guard([&] {
    require(host_uv || m == 0, "rmat: null output");
    use_device(*ctx);
    DevBuf uv;
    int64_t* d = uv.reserve_n<int64_t>(static_cast<size_t>(std::max<int64_t>(2 * m, 1)));
    rmat_edges_device(*ctx, scale, m, a, b, c, seed, d);
    download(host_uv, d, static_cast<size_t>(2 * m), ctx->stream);
  });
}

int ggb_dataset_generate_rmat(ggb_ctx_t ctx, int32_t scale, int64_t m, double a, double b, double c, int64_t d_in,
                              int64_t n_classes, uint64_t seed, ggb_dataset_t* out) {
  return guard([&] {
    require(out != nullptr, "dataset: null handle slot");
    use_device(*ctx);
    auto d = std::make_unique<ggb_dataset_s>();
    d->uv.resize(static_cast<size_t>(2 * m));
    DevBuf uv;
    int64_t* dev = uv.reserve_n<int64_t>(static_cast<size_t>(std::max<int64_t>(2 * m, 1)));
    rmat_edges_device(*ctx, scale, m, a, b, c, seed, dev);
    download(d->uv.data(), dev, d->uv.size(), ctx->stream);
    static_cast<HostDataset&>(*d) = dataset_from_edges(int64_t{1} << scale, d->uv.data(), m, d_in, n_classes, seed);
    *out = d.release();
  });
}

int ggb_dataset_info(ggb_dataset_t d, int64_t* info) {
  return guard([&] {
    require(d && info, "dataset_info: null argument");
    info[0] = d->n;
    info[1] = static_cast<int64_t>(d->adj.col.size());
    info[2] = d->d_in;
    info[3] = d->n_classes;
    info[4] = static_cast<int64_t>(d->uv.size() / 2);
  });
}

int ggb_dataset_export(ggb_dataset_t d, int64_t* row_ptr, int64_t* col_idx, double* values, float* features,
                       int32_t* labels, uint8_t* split, int64_t* edges_uv) {
  return guard([&] {
    require(d != nullptr, "dataset_export: null dataset");
    auto cp = [](auto* dst, const auto& v) {
      if (dst) std::copy(v.begin(), v.end(), dst);
    };
    cp(row_ptr, d->adj.row_ptr);
    cp(col_idx, d->adj.col);
    cp(values, d->adj.val);
    cp(features, d->features);
    cp(labels, d->labels);
    cp(split, d->split);
    cp(edges_uv, d->uv);
  });
}

int ggb_dataset_save(ggb_dataset_t d, const char* edges, const char* features, const char* labels,
                     const char* split) {
  return guard([&] {
    require(d != nullptr, "dataset_save: null dataset");
    if (edges) save_edge_list(edges, d->uv.data(), static_cast<int64_t>(d->uv.size() / 2));
    if (features) save_features(features, d->n, d->d_in, d->features.data());
    if (labels) save_labels(labels, d->n, d->n_classes, d->labels.data());
    if (split) save_split(split, d->n, d->split.data());
  });
}

int ggb_graph_from_dataset(ggb_ctx_t ctx, ggb_dataset_t d, int32_t layers, ggb_graph_t* out) {
  return guard([&] {
    require(d && out, "graph_from_dataset: null argument");
    use_device(*ctx);
    auto g = std::make_unique<ggb_graph_s>();
    graph_build(*ctx, *g, d->n, d->adj.row_ptr.data(), d->adj.col.data(), d->adj.val.data(), true, d->d_in,
                d->features.data(), d->n_classes, d->labels.data(), layers);
    set_split(*g, d->split.data());
    *out = g.release();
  });
}

int ggb_dataset_destroy(ggb_dataset_t d) {
  return guard([&] { delete d; });
}

int ggb_graph_set_split(ggb_graph_t g, const uint8_t* split) {
  return guard([&] {
    require(g && split, "graph_set_split: null argument");
    use_device(*g->ctx);
    set_split(*g, split);
  });
}

int ggb_graph_destroy(ggb_graph_t g) {
  return guard([&] {
    if (g) cudaSetDevice(g->ctx->device);
    delete g;
  });
}

int ggb_graph_features_to_host(ggb_graph_t g) {
  return guard([&] {
    require(g != nullptr, "graph_features_to_host: null graph");
    use_device(*g->ctx);
    if (g->features_on_host()) return;
    const size_t bytes = g->features.bytes ? static_cast<size_t>(g->n) * (g->feat_c1 - g->feat_c0) * 4 : 0;
    require(bytes > 0, "graph_features_to_host: no device features");
    PinnedBuf& h = g->features_host;
    GGB_CUDA(cudaHostAlloc(&h.p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    h.bytes = bytes;
    GGB_CUDA(cudaMemcpyAsync(h.p, g->features.p, bytes, cudaMemcpyDeviceToHost, g->ctx->stream));
    GGB_CUDA(cudaStreamSynchronize(g->ctx->stream));
    void* dp = nullptr;
    GGB_CUDA(cudaHostGetDevicePointer(&dp, h.p, 0));
    g->feat_ptr = static_cast<const float*>(dp);
    g->device_bytes -= g->features.bytes;
    g->features.release();
  });
}

int ggb_graph_info(ggb_graph_t g, int64_t* info) {
  return guard([&] {
    info[0] = g->n;
    info[1] = g->nnz;
    info[2] = g->d_in;
    info[3] = g->n_classes;
    info[4] = static_cast<int64_t>(g->shards.size());
    info[5] = static_cast<int64_t>(g->device_bytes);
    info[6] = g->features_on_host() ? 1 : 0;
  });
}

int ggb_build_step_batch(ggb_ctx_t ctx, ggb_graph_t g, int64_t b, uint64_t group_seed, uint64_t step,
                         ggb_batch_t* inout) {
  return guard([&] {
    use_device(*ctx);
    require(inout != nullptr, "batch: null handle slot");
    std::unique_ptr<ggb_batch_s> fresh;
    ggb_batch_s* bt = *inout;
    if (!bt) {
      fresh = std::make_unique<ggb_batch_s>();
      bt = fresh.get();
    }
    build_step_batch(*ctx, *g, b, group_seed, step, *bt);
    if (fresh) *inout = fresh.release();
  });
}

int ggb_prefetch_create(ggb_ctx_t ctx, ggb_graph_t g, int64_t b, uint64_t group_seed, uint64_t first_step,
                        uint64_t run_seed, int32_t layers, int64_t d_h, double dropout_rate,
                        ggb_prefetch_t* out) {
  return guard([&] {
    use_device(*ctx);
    require(g && out, "prefetch: null argument");
    *out = new ggb_prefetch_s(*ctx, *g, b, group_seed, first_step, run_seed, layers, d_h, dropout_rate);
  });
}

int ggb_prefetch_next(ggb_prefetch_t pf, ggb_batch_t* batch_out) {
  return guard([&] {
    use_device(*pf->consumer);
    *batch_out = reinterpret_cast<ggb_batch_t>(pf->next());  // owned by the prefetcher
  });
}

int ggb_prefetch_destroy(ggb_prefetch_t pf) {
  return guard([&] { delete pf; });
}

int ggb_batch_destroy(ggb_batch_t batch) {
  return guard([&] {
    if (batch && batch->ctx) cudaSetDevice(batch->ctx->device);
    delete batch;
  });
}

int ggb_batch_info(ggb_batch_t bt, int64_t* info) {
  return guard([&] {
    if (bt->ctx) use_device(*bt->ctx);
    settle_totals(*bt);
    info[0] = bt->b;
    info[1] = bt->n;
    info[2] = bt->planes;
    info[3] = bt->x_r0;
    info[4] = bt->x_r1;
    info[5] = bt->x_c0;
    info[6] = bt->x_c1;
    info[7] = static_cast<int64_t>(bt->nnz_extracted);
    info[8] = static_cast<int64_t>(bt->nnz_kept);
  });
}

int ggb_batch_sample(ggb_batch_t bt, int64_t* host_out) {
  return guard([&] {
    use_device(*bt->ctx);
    download(host_out, bt->sample.p, static_cast<size_t>(bt->b), bt->ctx->stream);
  });
}

int ggb_batch_offsets(ggb_batch_t bt, int32_t axis, int64_t* host_out) {
  return guard([&] {
    require(axis >= 1 && axis <= 3, "batch_offsets: axis must be X, Y or Z");
    std::copy(bt->batch_off[axis].begin(), bt->batch_off[axis].end(), host_out);
  });
}

int ggb_batch_plane(ggb_batch_t bt, int32_t plane, int32_t transposed, int64_t* dims, int64_t* row_ptr,
                    int64_t* col_idx, double* values) {
  return guard([&] {
    require(plane >= 0 && plane < bt->planes, "batch_plane: plane out of range");
    use_device(*bt->ctx);
    settle_totals(*bt);
    const BatchCsr& c = bt->csrs[transposed ? bt->csrt_of[plane] : bt->csr_of[plane]];
    dims[0] = c.n_rows;
    dims[1] = c.n_cols;
    dims[2] = c.nnz;
    dims[3] = c.r0;
    dims[4] = c.r1;
    dims[5] = c.c0;
    dims[6] = c.c1;
    cudaStream_t s = bt->ctx->stream;
    download(row_ptr, c.row_ptr.p, static_cast<size_t>(c.n_rows + 1), s);
    if (col_idx) {
      std::vector<int32_t> c32(static_cast<size_t>(c.nnz));
      download(c32.data(), c.col.p, c32.size(), s);
      for (int64_t k = 0; k < c.nnz; ++k) col_idx[k] = c32[k];
    }
    download(values, c.val64.p, static_cast<size_t>(c.nnz), s);
  });
}

int ggb_batch_x_in(ggb_batch_t bt, float* host_out) {
  return guard([&] {
    Ctx& ctx = *bt->ctx;
    use_device(ctx);
    const int64_t n = (bt->x_r1 - bt->x_r0) * (bt->x_c1 - bt->x_c0);
    DevBuf tmp;
    float* d = tmp.reserve_n<float>(std::max<int64_t>(n, 1));
    gather_x_in_fp32(ctx, *bt, d);
    download(host_out, d, static_cast<size_t>(n), ctx.stream);
  });
}

int ggb_batch_labels(ggb_batch_t bt, int32_t* host_out) {
  return guard([&] {
    use_device(*bt->ctx);
    download(host_out, bt->labels.p, static_cast<size_t>(bt->b), bt->ctx->stream);
  });
}

int ggb_state_create(ggb_ctx_t ctx, const ggb_model_config* cfg, uint64_t seed, ggb_state_t* out) {
  return guard([&] {
    use_device(*ctx);
    require(cfg && out, "state: null argument");
    auto st = std::make_unique<ggb_state_s>();
    state_init(*ctx, *st, *cfg, seed);
    GGB_CUDA(cudaStreamSynchronize(ctx->stream));
    *out = st.release();
  });
}

int ggb_state_destroy(ggb_state_t st) {
  return guard([&] {
    if (st && st->ctx) cudaSetDevice(st->ctx->device);
    delete st;
  });
}

int ggb_state_set_compute(ggb_state_t st, int32_t mode) {
  return guard([&] {
    require(mode == kAccurate || mode == kFast, "compute mode must be ACCURATE or FAST");
    st->compute = mode;
  });
}

int ggb_state_num_params(ggb_state_t st) { return st ? static_cast<int>(st->params.size()) : -1; }

int ggb_state_param_info(ggb_state_t st, int32_t idx, int64_t* info) {
  return guard([&] {
    require(idx >= 0 && idx < static_cast<int>(st->params.size()), "param index out of range");
    const Block& b = st->params[idx].blk;
    info[0] = b.g_rows;
    info[1] = b.g_cols;
    info[2] = b.r0;
    info[3] = b.r1;
    info[4] = b.c0;
    info[5] = b.c1;
  });
}

static float* which_buf(State& st, int which) {
  switch (which) {
    case 0: return st.W.as<float>();
    case 1: return st.G.as<float>();
    case 2: return st.M.as<float>();
    case 3: return st.V.as<float>();
    default: fail(GGB_EINVAL, "param: which must be 0..3");
  }
}

int ggb_state_param_get(ggb_state_t st, int32_t idx, int32_t which, float* host_out) {
  return guard([&] {
    require(idx >= 0 && idx < static_cast<int>(st->params.size()), "param index out of range");
    use_device(*st->ctx);
    const ParamSlot& p = st->params[idx];
    download(host_out, which_buf(*st, which) + p.off, static_cast<size_t>(p.n), st->ctx->stream);
  });
}

int ggb_state_param_set(ggb_state_t st, int32_t idx, int32_t which, const float* host_in) {
  return guard([&] {
    require(idx >= 0 && idx < static_cast<int>(st->params.size()), "param index out of range");
    use_device(*st->ctx);
    const ParamSlot& p = st->params[idx];
    GGB_CUDA(cudaMemcpyAsync(which_buf(*st, which) + p.off, host_in, p.n * 4, cudaMemcpyHostToDevice,
                             st->ctx->stream));
    if (which == 0) refresh_bf16(*st);
    GGB_CUDA(cudaStreamSynchronize(st->ctx->stream));
  });
}

int ggb_train_step(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t bt, int32_t precision, uint64_t run_seed,
                   uint64_t global_step, double rmsnorm_eps, float* loss_out) {
  return guard([&] {
    use_device(*ctx);
    contract(st->ctx == ctx && bt->ctx && bt->ctx->device == ctx->device && bt->ctx->rank == ctx->rank,
             "train_step: handles belong to another rank");
    {  // train_step's phases (model.hpp:466-476)
      PhaseScope ps(*ctx, kPhaseForward);
      forward(*st, *bt, precision, true, run_seed, global_step, rmsnorm_eps);
      cross_entropy(*st, *bt);
    }
    {
      PhaseScope ps(*ctx, kPhaseBackward);
      backward(*st, *bt, precision);
    }
    if (loss_out) {
      GGB_CUDA(cudaMemcpyAsync(loss_out, st->loss.p, sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
      sync_stream(*ctx, ctx->stream);  // with the collective watchdog
      ctx->d2h_bytes += sizeof(float);
    }
  });
}

int ggb_loss_to_host_async(ggb_ctx_t ctx, ggb_state_t st, float* host_dst) {
  return guard([&] {
    use_device(*ctx);
    contract(st->ctx == ctx && st->have_forward, "loss_to_host_async: no train_step of this state on this rank");
    require(host_dst != nullptr, "loss_to_host_async: null destination");
    GGB_CUDA(cudaMemcpyAsync(host_dst, st->loss.p, sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->d2h_bytes += sizeof(float);
  });
}

int ggb_loss(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t bt, float* loss_out) {
  return guard([&] {
    use_device(*ctx);
    contract(st->ctx == ctx && st->have_forward, "loss: no forward of this state on this rank");
    {
      PhaseScope ps(*ctx, kPhaseForward);
      cross_entropy(*st, *bt);
    }
    if (loss_out) {
      GGB_CUDA(cudaMemcpyAsync(loss_out, st->loss.p, sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
      sync_stream(*ctx, ctx->stream);  // with the collective watchdog
      ctx->d2h_bytes += sizeof(float);
    }
  });
}

int ggb_backward(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t bt, int32_t precision) {
  return guard([&] {
    use_device(*ctx);
    contract(st->ctx == ctx, "backward: state belongs to another rank");
    PhaseScope ps(*ctx, kPhaseBackward);
    backward(*st, *bt, precision);
  });
}

int ggb_device_alloc(ggb_ctx_t ctx, size_t bytes, void** out) {
  return guard([&] {
    require(out != nullptr, "device_alloc: null slot");
    use_device(*ctx);
    *out = nullptr;
    GGB_CUDA(cudaMalloc(out, std::max<size_t>(bytes, 16)));
  });
}

int ggb_device_free(ggb_ctx_t ctx, void* p) {
  return guard([&] {
    use_device(*ctx);
    GGB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (p) GGB_CUDA(cudaFree(p));
  });
}

int ggb_memcpy_h2d(ggb_ctx_t ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    use_device(*ctx);
    if (bytes == 0) return;
    GGB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    GGB_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->h2d_bytes += bytes;
  });
}

int ggb_memcpy_d2h(ggb_ctx_t ctx, void* dst, const void* src, size_t bytes) {
  return guard([&] {
    use_device(*ctx);
    if (bytes == 0) return;
    GGB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    GGB_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->d2h_bytes += bytes;
  });
}

int ggb_contract(ggb_ctx_t ctx, const ggb_block* a, const ggb_block* b, const ggb_block* c, int32_t precision) {
  return guard([&] {
    require(a && b && c, "contract: null block");
    use_device(*ctx);
    layer_contract(*ctx, *a, *b, *c, precision);
  });
}

int ggb_spmm(ggb_ctx_t ctx, const ggb_csr_block* a, const ggb_block* f, const ggb_block* h, int32_t precision) {
  return guard([&] {
    require(a && f && h, "spmm: null block");
    use_device(*ctx);
    layer_spmm(*ctx, *a, *f, *h, precision);
  });
}

int ggb_transposed(ggb_ctx_t ctx, const ggb_block* t, const ggb_block* out) {
  return guard([&] {
    require(t && out, "transposed: null block");
    use_device(*ctx);
    layer_transposed(*ctx, *t, *out);
  });
}

int ggb_gather_full(ggb_ctx_t ctx, const ggb_block* t, float* full, int64_t ld_full) {
  return guard([&] {
    require(t && full && ld_full >= t->g_cols, "gather_full: bad output");
    use_device(*ctx);
    layer_gather_full(*ctx, *t, full, ld_full);
  });
}

int ggb_reshard(ggb_ctx_t ctx, const ggb_block* src, const ggb_block* dst) {
  return guard([&] {
    require(src && dst, "reshard: null block");
    use_device(*ctx);
    layer_reshard(*ctx, *src, *dst);
  });
}

int ggb_rmsnorm_fwd(ggb_ctx_t ctx, const ggb_block* x, const float* gamma, double eps, const ggb_block* y,
                    float* rms) {
  return guard([&] {
    require(x && y && gamma, "rmsnorm: null argument");
    use_device(*ctx);
    layer_rmsnorm_fwd(*ctx, *x, gamma, eps, *y, rms);
  });
}

int ggb_rmsnorm_bwd(ggb_ctx_t ctx, const ggb_block* x, const float* gamma, const float* rms, const ggb_block* dy,
                    const ggb_block* dx, float* dgamma) {
  return guard([&] {
    require(x && gamma && rms && dy && dx && dgamma, "rmsnorm_bwd: missing cache");
    use_device(*ctx);
    layer_rmsnorm_bwd(*ctx, *x, gamma, rms, *dy, *dx, dgamma);
  });
}

int ggb_fused_elementwise_fwd(ggb_ctx_t ctx, const ggb_block* x, const ggb_block* h_prev, double rate,
                              uint64_t mask_key, int32_t training, const ggb_block* out, uint32_t* keep_bits) {
  return guard([&] {
    require(x && out, "fused_elementwise: null block");
    use_device(*ctx);
    layer_fused_fwd(*ctx, *x, h_prev, rate, mask_key, training, *out, keep_bits);
  });
}

int ggb_fused_elementwise_bwd(ggb_ctx_t ctx, const ggb_block* dy, const uint32_t* keep_bits, float keep_scale,
                              const ggb_block* dx) {
  return guard([&] {
    require(dy && dx, "fused_elementwise_bwd: null block");
    contract(keep_bits != nullptr, "fused_elementwise_bwd: missing cache");
    use_device(*ctx);
    layer_fused_bwd(*ctx, *dy, keep_bits, keep_scale, *dx);
  });
}

int64_t ggb_mask_words(int64_t cols) { return mask_words(std::max<int64_t>(cols, 1)); }

int ggb_cross_entropy(ggb_ctx_t ctx, const ggb_block* logits, const int32_t* labels, float* loss,
                      const ggb_block* grad) {
  return guard([&] {
    require(logits && labels && loss && grad, "cross_entropy: null argument");
    use_device(*ctx);
    layer_cross_entropy(*ctx, *logits, labels, loss, *grad);
  });
}

int ggb_batch_csr_block(ggb_batch_t bt, int32_t plane, int32_t transposed, ggb_csr_block* out) {
  return guard([&] {
    require(bt && out && plane >= 0 && plane < bt->planes, "batch_csr_block: plane out of range");
    const Layout lay = adjacency_layout(plane + 1);
    const BatchCsr& c = bt->csrs[transposed ? bt->csrt_of[plane] : bt->csr_of[plane]];
    const int ra = transposed ? lay.col : lay.row, ca = transposed ? lay.row : lay.col;
    out->row_axis = ra;
    out->col_axis = ca;
    out->g_rows = bt->b;
    out->g_cols = bt->b;
    out->row_off = bt->batch_off[ra].data();
    out->col_off = bt->batch_off[ca].data();
    out->row_ptr = c.row_ptr.as<int64_t>();
    out->col = c.col.as<int32_t>();
    out->val = c.val.as<float>();
  });
}

int ggb_last_loss_device(ggb_state_t st, const float** dev_ptr) {
  return guard([&] {
    require(st->loss.p != nullptr, "no loss computed yet");
    *dev_ptr = st->loss.as<float>();
  });
}

int ggb_state_logits(ggb_state_t st, int64_t* dims, float* host_out) {
  return guard([&] {
    require(st->have_forward, "no forward pass yet");
    const Block& b = st->logits_blk;
    dims[0] = b.r0;
    dims[1] = b.r1;
    dims[2] = b.c0;
    dims[3] = b.c1;
    use_device(*st->ctx);
    download(host_out, st->logits.p, static_cast<size_t>(b.rows() * b.cols()), st->ctx->stream);
  });
}

int ggb_forward(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t bt, int32_t precision, int32_t training,
                uint64_t run_seed, uint64_t global_step, double rmsnorm_eps) {
  return guard([&] {
    use_device(*ctx);
    forward(*st, *bt, precision, training != 0, run_seed, global_step, rmsnorm_eps);
  });
}

int ggb_evaluate_full_graph(ggb_ctx_t ctx, ggb_state_t st, ggb_batch_t eval_batch, ggb_graph_t g,
                            int32_t precision, double rmsnorm_eps, uint64_t* counts) {
  return guard([&] {
    require(st && eval_batch && g && counts, "evaluate_full_graph: null argument");
    use_device(*ctx);
    evaluate_full_graph(*st, *eval_batch, *g, precision, rmsnorm_eps, counts);
  });
}

int ggb_dp_sync(ggb_ctx_t ctx, ggb_state_t st) {
  return guard([&] {
    use_device(*ctx);
    dp_sync(*st);
  });
}

int ggb_optimizer_step(ggb_ctx_t ctx, ggb_state_t st, int32_t optimizer, double lr) {
  return guard([&] {
    use_device(*ctx);
    optimizer_step(*st, optimizer, lr);
  });
}

int ggb_gemm_bf16(ggb_ctx_t ctx, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda, const void* bt,
                  int64_t ldb, float* c, int64_t ldc, void* c_bf16, int64_t ldcb) {
  return guard([&] {
    use_device(*ctx);
    gemm_bf16(*ctx, m, n, k, static_cast<const bf16*>(a), lda, static_cast<const bf16*>(bt), ldb, c, ldc,
              static_cast<bf16*>(c_bf16), ldcb);
  });
}

int ggb_gemm_split_bf16(ggb_ctx_t ctx, int64_t m, int64_t n, int64_t k, const void* a_hi, const void* a_lo,
                        int64_t lda, const void* bt_hi, const void* bt_lo, int64_t ldb, float* c, int64_t ldc) {
  return guard([&] {
    use_device(*ctx);
    gemm_split(*ctx, m, n, k, static_cast<const bf16*>(a_hi), static_cast<const bf16*>(a_lo), lda,
               static_cast<const bf16*>(bt_hi), static_cast<const bf16*>(bt_lo), ldb, c, ldc, nullptr, 0);
  });
}

int ggb_gemm_wgrad_bf16(ggb_ctx_t ctx, int64_t m, int64_t kw, int64_t nw, const void* x, int64_t ldx,
                        const void* dy, int64_t lddy, float* dw, int64_t lddw) {
  return guard([&] {
    use_device(*ctx);
    gemm_wgrad_bf16(*ctx, m, kw, nw, static_cast<const bf16*>(x), ldx, static_cast<const bf16*>(dy), lddy, dw, lddw,
                    g_ws);
  });
}

int ggb_spmm_csr(ggb_ctx_t ctx, int64_t rows, const int64_t* row_ptr, const int32_t* col, const float* val,
                 const void* f, int64_t ldf, int64_t fcols, float* out, int64_t ldo, void* out_bf16, int64_t ldob,
                 int32_t accumulate) {
  return guard([&] {
    use_device(*ctx);
    LongRowsScope lrs(*ctx, true);  // test entry: the merge-path kernel (any row-length profile)
    spmm_csr(*ctx, rows, row_ptr, col, val, static_cast<const bf16*>(f), ldf, fcols, out, ldo,
             static_cast<bf16*>(out_bf16), ldob, accumulate);
  });
}

int ggb_spmm_csr_f32(ggb_ctx_t ctx, int64_t rows, const int64_t* row_ptr, const int32_t* col, const float* val,
                     const float* f, int64_t ldf, int64_t fcols, float* out, int64_t ldo, void* out_hi,
                     void* out_lo, int64_t ldob, int32_t accumulate) {
  return guard([&] {
    use_device(*ctx);
    LongRowsScope lrs(*ctx, true);
    spmm_csr_f32(*ctx, rows, row_ptr, col, val, f, ldf, fcols, out, ldo, static_cast<bf16*>(out_hi),
                 static_cast<bf16*>(out_lo), ldob, accumulate);
  });
}

}  // extern "C"
