// TEST INFRASTRUCTURE ONLY — never linked into the product (libggb.so).
//
// Neutral extern "C" surface over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place with -Dgridgnn=gridgnn_ref
// by oracle/Makefile). Tests, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs call these through ctypes.
//
// Every entry point drives the reference's own public API:
//   sample_vertices            proj/src/sampling.cpp:11-33
//   generate_synthetic, ...    proj/src/dataset.cpp:47-150
//   make_rank_context          proj/include/gridgnn/model.hpp:217-234
//   build_step_batch           proj/include/gridgnn/model.hpp:250-309
//   forward/train_step         proj/include/gridgnn/model.hpp:335-478
//   dp_sync/optimizer_step     proj/include/gridgnn/model.hpp:423-456
// and mirrors acceptance.cpp:171-190 (serial_step) for the step harness.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "gridgnn/comm.hpp"
#include "gridgnn/dataset.hpp"
#include "gridgnn/model.hpp"
#include "gridgnn/pmm.hpp"
#include "gridgnn/rng.hpp"
#include "gridgnn/sampling.hpp"
#include "gridgnn/shardsample.hpp"

using namespace gridgnn;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const CommContract& e) {
    g_err = e.what();
    return 2;
  } catch (const CommTimeout& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

template <class Body>
void run_ranks(Communicator& comm, Body&& body) {
  std::vector<std::thread> threads;
  std::vector<std::exception_ptr> errs(static_cast<std::size_t>(comm.grid().total()));
  for (int r = 0; r < comm.grid().total(); ++r)
    threads.emplace_back([&, r] {
      try {
        RankComm rc(comm, r);
        body(rc);
      } catch (...) {
        errs[static_cast<std::size_t>(r)] = std::current_exception();
      }
    });
  for (auto& t : threads) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

struct RefBatch {
  StepBatch<float> sb;
  std::vector<std::uint64_t> counters;  // per plane extracted, kept
};

ModelConfig make_cfg(const std::int64_t* mc, const double* md) {
  // mc = {layers, d_in, d_h, d_out, use_rmsnorm, use_dropout, use_residual}
  ModelConfig c;
  c.layers = static_cast<int>(mc[0]);
  c.d_in = mc[1];
  c.d_h = mc[2];
  c.d_out = mc[3];
  c.use_rmsnorm = mc[4] != 0;
  c.use_dropout = mc[5] != 0;
  c.use_residual = mc[6] != 0;
  c.dropout_rate = md[0];
  return c;
}

template <class Real>
void put_tile(const ShardedTensor<Real>& t, float* global) {
  for (index_t i = t.r0; i < t.r1; ++i)
    for (index_t j = t.c0; j < t.c1; ++j)
      global[i * t.g_cols + j] = static_cast<float>(t.local.at(i - t.r0, j - t.c0));
}

template <class Real>
void put_vec(const VecParam<Real>& g, const std::vector<Real>& v, float* global) {
  for (index_t j = g.c0; j < g.c1; ++j) global[j] = static_cast<float>(v[static_cast<std::size_t>(j - g.c0)]);
}

/// Global size of the flattened parameter export (win, [wl, gamma] x L, wout).
std::int64_t param_total(const ModelConfig& c) {
  std::int64_t n = c.d_in * c.d_h + c.d_h * c.d_out;
  n += static_cast<std::int64_t>(c.layers) * (c.d_h * c.d_h + (c.use_rmsnorm ? c.d_h : 0));
  return n;
}

/// Writes the assembled global values of every parameter (or its gradient /
/// Adam moment) in param_views order into out.
template <class Real>
void export_params(const std::vector<ModelState<Real>>& states, int which, float* out) {
  const auto& c = states.front().cfg;
  std::int64_t off = 0;
  auto pick = [which](const Param<Real>& p) -> const ShardedTensor<Real>& {
    return which == 1 ? p.g : p.w;
  };
  for (const auto& st : states) put_tile(pick(st.win), out + off);
  off += c.d_in * c.d_h;
  for (int l = 0; l < c.layers; ++l) {
    for (const auto& st : states) put_tile(pick(st.wl[static_cast<std::size_t>(l)]), out + off);
    off += c.d_h * c.d_h;
    if (c.use_rmsnorm) {
      for (const auto& st : states) {
        const auto& gm = st.gamma[static_cast<std::size_t>(l)];
        put_vec(gm, which == 1 ? gm.g : gm.w, out + off);
      }
      off += c.d_h;
    }
  }
  for (const auto& st : states) put_tile(pick(st.wout), out + off);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_sample_vertices(std::int64_t n, std::int64_t b, std::uint64_t seed, std::uint64_t step,
                        std::int64_t* out) {
  return guard([&] {
    auto s = sample_vertices(n, b, seed, step);
    std::memcpy(out, s.vertices.data(), s.vertices.size() * sizeof(std::int64_t));
  });
}

std::uint64_t ref_splitmix64(std::uint64_t x) { return rng::splitmix64(x); }
std::uint64_t ref_hash_combine(std::uint64_t a, std::uint64_t b) { return rng::hash_combine(a, b); }
double ref_element_unit(std::uint64_t k, std::uint64_t i, std::uint64_t j) {
  return rng::element_unit(k, i, j);
}
float ref_bf16_round(float x) { return bf16_round(x); }
std::uint64_t ref_dropout_key(std::uint64_t seed, int dp, std::uint64_t gstep, int layer) {
  return detail::dropout_key(seed, dp, gstep, layer);
}

int ref_block_partition(std::int64_t n, int g, std::int64_t* out) {
  return guard([&] {
    auto v = block_partition(n, g);
    std::memcpy(out, v.data(), v.size() * sizeof(std::int64_t));
  });
}

// ---- datasets ---------------------------------------------------------------

void* ref_dataset_synthetic(std::int64_t n, double avg_degree, std::int64_t d_in,
                            std::int64_t n_classes, std::uint64_t seed) {
  Dataset* out = nullptr;
  if (guard([&] { out = new Dataset(generate_synthetic(n, avg_degree, d_in, n_classes, seed)); }) != 0)
    return nullptr;
  return out;
}

/// Dataset from a raw edge list through the reference's own normalization
/// (dataset.cpp:47-83); features/labels/split supplied by the caller.
void* ref_dataset_from_edges(std::int64_t n, const std::int64_t* uv, std::int64_t m,
                             std::int64_t d_in, const float* features, std::int64_t n_classes,
                             const std::int32_t* labels, const std::uint8_t* split) {
  Dataset* out = nullptr;
  if (guard([&] {
        std::vector<std::pair<index_t, index_t>> edges(static_cast<std::size_t>(m));
        for (std::int64_t e = 0; e < m; ++e) edges[static_cast<std::size_t>(e)] = {uv[2 * e], uv[2 * e + 1]};
        auto ds = std::make_unique<Dataset>();
        ds->adjacency = normalize_adjacency(edges, n);
        ds->n = n;
        ds->d_in = d_in;
        ds->n_classes = n_classes;
        ds->features.assign(features, features + n * d_in);
        ds->labels.assign(labels, labels + n);
        ds->split.resize(static_cast<std::size_t>(n));
        for (std::int64_t v = 0; v < n; ++v) ds->split[static_cast<std::size_t>(v)] = static_cast<SplitTag>(split[v]);
        out = ds.release();
      }) != 0)
    return nullptr;
  return out;
}

/// load_dataset (dataset.cpp:178-239): the reference's own readers.
void* ref_dataset_load(const char* edges, const char* features, const char* labels, const char* split) {
  Dataset* out = nullptr;
  if (guard([&] { out = new Dataset(load_dataset(edges, features, labels, split)); }) != 0) return nullptr;
  return out;
}

/// The CLI's `gen` command (gridgnn_main.cpp:313-324): synthetic_edges +
/// generate_synthetic written with the reference's save_* (dataset.cpp:241-280).
int ref_save_synthetic(std::int64_t n, double avg_degree, std::int64_t d_in, std::int64_t n_classes,
                       std::uint64_t seed, const char* edges_path, const char* features_path,
                       const char* labels_path, const char* split_path) {
  return guard([&] {
    const auto edges = synthetic_edges(n, avg_degree, seed);
    const Dataset ds = generate_synthetic(n, avg_degree, d_in, n_classes, seed);
    save_edge_list(edges_path, edges);
    save_features(features_path, ds.n, ds.d_in, ds.features);
    save_labels(labels_path, ds.n, ds.n_classes, ds.labels);
    save_split(split_path, ds.split);
  });
}

void ref_dataset_free(void* ds) { delete static_cast<Dataset*>(ds); }

void ref_dataset_info(void* p, std::int64_t* out) {
  auto* ds = static_cast<Dataset*>(p);
  out[0] = ds->n;
  out[1] = ds->adjacency.nnz();
  out[2] = ds->d_in;
  out[3] = ds->n_classes;
}

void ref_dataset_export(void* p, std::int64_t* row_ptr, std::int64_t* col, double* val, float* feats,
                        std::int32_t* labels, std::uint8_t* split) {
  auto* ds = static_cast<Dataset*>(p);
  if (row_ptr) std::memcpy(row_ptr, ds->adjacency.row_ptr.data(), ds->adjacency.row_ptr.size() * 8);
  if (col) std::memcpy(col, ds->adjacency.col_idx.data(), ds->adjacency.col_idx.size() * 8);
  if (val) std::memcpy(val, ds->adjacency.values.data(), ds->adjacency.values.size() * 8);
  if (feats) std::memcpy(feats, ds->features.data(), ds->features.size() * 4);
  if (labels) std::memcpy(labels, ds->labels.data(), ds->labels.size() * 4);
  if (split)
    for (std::size_t v = 0; v < ds->split.size(); ++v) split[v] = static_cast<std::uint8_t>(ds->split[v]);
}

std::int64_t ref_synthetic_edges(std::int64_t n, double avg_degree, std::uint64_t seed,
                                 std::int64_t* uv_out) {
  std::int64_t m = -1;
  guard([&] {
    auto e = synthetic_edges(n, avg_degree, seed);
    m = static_cast<std::int64_t>(e.size());
    if (uv_out)
      for (std::size_t k = 0; k < e.size(); ++k) {
        uv_out[2 * k] = e[k].first;
        uv_out[2 * k + 1] = e[k].second;
      }
  });
  return m;
}

// ---- step batches (build_step_batch for one rank) ----------------------------

void* ref_step_batch(void* dsp, const int* dims, int rank, int layers, std::int64_t b,
                     std::uint64_t group_seed, std::uint64_t step) {
  auto* ds = static_cast<Dataset*>(dsp);
  RefBatch* out = nullptr;
  if (guard([&] {
        DeviceGrid grid(dims[0], dims[1], dims[2], dims[3]);
        const Coord4 coord = grid.coord_of(rank);
        RankContext ctx = make_rank_context(grid, coord, *ds, layers);
        RankStats stats;
        auto rb = std::make_unique<RefBatch>();
        rb->sb = build_step_batch<float>(grid, coord, ctx, *ds, b, group_seed, step, &stats);
        rb->counters = {stats.sampled_nnz_extracted, stats.sampled_nnz_kept};
        out = rb.release();
      }) != 0)
    return nullptr;
  return out;
}

void ref_batch_free(void* p) { delete static_cast<RefBatch*>(p); }

void ref_batch_sample(void* p, std::int64_t* out) {
  auto* rb = static_cast<RefBatch*>(p);
  std::memcpy(out, rb->sb.sample.vertices.data(), rb->sb.sample.vertices.size() * 8);
}

void ref_batch_counters(void* p, std::uint64_t* out) {
  auto* rb = static_cast<RefBatch*>(p);
  out[0] = rb->counters[0];
  out[1] = rb->counters[1];
}

int ref_batch_offsets(void* p, int axis, std::int64_t* out) {
  auto* rb = static_cast<RefBatch*>(p);
  const auto& v = rb->sb.batch_off[static_cast<std::size_t>(axis)];
  std::memcpy(out, v.data(), v.size() * 8);
  return static_cast<int>(v.size());
}

int ref_batch_num_planes(void* p) { return static_cast<int>(static_cast<RefBatch*>(p)->sb.a.size()); }

/// dims = {n_rows, n_cols, nnz, r0, r1, c0, c1}; arrays may be null (query).
void ref_batch_plane(void* p, int plane, int transposed, std::int64_t* dims, std::int64_t* row_ptr,
                     std::int64_t* col, double* val) {
  auto* rb = static_cast<RefBatch*>(p);
  const ShardedSparse& s = transposed ? rb->sb.a_t[static_cast<std::size_t>(plane)]
                                      : rb->sb.a[static_cast<std::size_t>(plane)];
  dims[0] = s.local.n_rows;
  dims[1] = s.local.n_cols;
  dims[2] = s.local.nnz();
  dims[3] = s.r0;
  dims[4] = s.r1;
  dims[5] = s.c0;
  dims[6] = s.c1;
  if (row_ptr) std::memcpy(row_ptr, s.local.row_ptr.data(), s.local.row_ptr.size() * 8);
  if (col) std::memcpy(col, s.local.col_idx.data(), s.local.col_idx.size() * 8);
  if (val) std::memcpy(val, s.local.values.data(), s.local.values.size() * 8);
}

/// dims = {r0, r1, c0, c1}; values row-major (r1-r0) x (c1-c0).
void ref_batch_x_in(void* p, std::int64_t* dims, float* out) {
  auto* rb = static_cast<RefBatch*>(p);
  const auto& x = rb->sb.x_in;
  dims[0] = x.r0;
  dims[1] = x.r1;
  dims[2] = x.c0;
  dims[3] = x.c1;
  if (out) std::memcpy(out, x.local.v.data(), x.local.v.size() * 4);
}

void ref_batch_labels(void* p, std::int32_t* out) {
  auto* rb = static_cast<RefBatch*>(p);
  std::memcpy(out, rb->sb.labels.data(), rb->sb.labels.size() * 4);
}

// ---- training ----------------------------------------------------------------

std::int64_t ref_param_total(const std::int64_t* mc, const double* md) {
  return param_total(make_cfg(mc, md));
}

/// Runs `n_steps` of the train_run step body (model.hpp:646-685, no eval, no
/// prefetch) on `dims`, one thread per rank, starting at global step
/// `step0`. Outputs: per-step loss (rank 0), the assembled logits of the LAST
/// step's training forward (b x d_out, optional), the assembled gradients of
/// the last step before dp_sync/optimizer (optional) and the final weights
/// (optional). prec: 0 fp32, 1 bf16 round-trip. optimizer: 0 sgd, 1 adam,
/// -1 none (gradients only).
int ref_train(void* dsp, const int* dims, const std::int64_t* mc, const double* md,
              std::int64_t b, std::uint64_t seed, std::uint64_t step0, int n_steps, int prec,
              int optimizer, double lr, double eps, float* losses, float* logits_out,
              float* grads_out, float* weights_out) {
  auto* ds = static_cast<Dataset*>(dsp);
  return guard([&] {
    const ModelConfig mcfg = make_cfg(mc, md);
    DeviceGrid grid(dims[0], dims[1], dims[2], dims[3]);
    Communicator comm(grid);
    const Precision p = prec ? Precision::kBf16Roundtrip : Precision::kFp32;
    std::vector<ModelState<float>> states(static_cast<std::size_t>(grid.total()));
    std::vector<ShardedTensor<float>> logits(static_cast<std::size_t>(grid.total()));
    run_ranks(comm, [&](RankComm& rc) {
      const int dp = grid.dp_group(rc.rank());
      const std::uint64_t group_seed = rng::hash_combine(seed, static_cast<std::uint64_t>(dp));
      RankContext ctx = make_rank_context(grid, rc.coord(), *ds, mcfg.layers);
      auto st = init_state<float>(grid, rc.coord(), mcfg, seed);
      for (int s = 0; s < n_steps; ++s) {
        const std::uint64_t gstep = step0 + static_cast<std::uint64_t>(s);
        auto batch = build_step_batch<float>(grid, rc.coord(), ctx, *ds, b, group_seed, gstep);
        auto cache = forward(rc, st, batch, p, true, seed, gstep, eps);
        auto ce = parallel_cross_entropy(rc, cache.logits, batch.labels);
        backward(rc, st, cache, batch, ce.grad_logits, p);
        if (rc.rank() == 0 && losses) losses[s] = ce.loss;
        if (s == n_steps - 1) logits[static_cast<std::size_t>(rc.rank())] = cache.logits;
        if (s == n_steps - 1) states[static_cast<std::size_t>(rc.rank())] = st;  // grads pre-sync
        if (optimizer >= 0) {
          dp_sync(rc, st);
          optimizer_step(st, optimizer == 0 ? Optimizer::kSgd : Optimizer::kAdam, lr);
        }
      }
      if (weights_out) {
        // keep grads of the last step in states[], but weights after the update
        auto& keep = states[static_cast<std::size_t>(rc.rank())];
        keep.win.w = st.win.w;
        for (std::size_t l = 0; l < st.wl.size(); ++l) keep.wl[l].w = st.wl[l].w;
        for (std::size_t l = 0; l < st.gamma.size(); ++l) keep.gamma[l].w = st.gamma[l].w;
        keep.wout.w = st.wout.w;
      }
    });
    if (logits_out)
      for (const auto& t : logits) put_tile(t, logits_out);
    if (grads_out) export_params(states, 1, grads_out);
    if (weights_out) export_params(states, 0, weights_out);
  });
}

/// train_run's per-epoch evaluation (model.hpp:621-626,686-688): n_steps
/// training steps from step 0 (group seeds, dp_sync, optimizer), then
/// evaluate_full_graph on the eval batch build_step_batch(b = n, seed, step 0).
/// counts = {correct train/val/test, total train/val/test}; eval_logits
/// (n x d_out, nullable) = the eval forward's logits.
int ref_train_eval(void* dsp, const int* dims, const std::int64_t* mc, const double* md,
                   std::int64_t b, std::uint64_t seed, int n_steps, int prec, int optimizer, double lr,
                   double eps, std::uint64_t* counts, float* eval_logits) {
  auto* ds = static_cast<Dataset*>(dsp);
  return guard([&] {
    const ModelConfig mcfg = make_cfg(mc, md);
    DeviceGrid grid(dims[0], dims[1], dims[2], dims[3]);
    Communicator comm(grid);
    const Precision p = prec ? Precision::kBf16Roundtrip : Precision::kFp32;
    std::vector<ShardedTensor<float>> logits(static_cast<std::size_t>(grid.total()));
    std::vector<EvalCounts> res(static_cast<std::size_t>(grid.total()));
    run_ranks(comm, [&](RankComm& rc) {
      const int dp = grid.dp_group(rc.rank());
      const std::uint64_t group_seed = rng::hash_combine(seed, static_cast<std::uint64_t>(dp));
      RankContext ctx = make_rank_context(grid, rc.coord(), *ds, mcfg.layers);
      const auto eval_batch = build_step_batch<float>(grid, rc.coord(), ctx, *ds, ds->n, seed, 0, nullptr);
      auto st = init_state<float>(grid, rc.coord(), mcfg, seed);
      for (int s = 0; s < n_steps; ++s) {
        const auto gstep = static_cast<std::uint64_t>(s);
        auto batch = build_step_batch<float>(grid, rc.coord(), ctx, *ds, b, group_seed, gstep);
        auto cache = forward(rc, st, batch, p, true, seed, gstep, eps);
        auto ce = parallel_cross_entropy(rc, cache.logits, batch.labels);
        backward(rc, st, cache, batch, ce.grad_logits, p);
        dp_sync(rc, st);
        optimizer_step(st, optimizer == 0 ? Optimizer::kSgd : Optimizer::kAdam, lr);
      }
      res[static_cast<std::size_t>(rc.rank())] = evaluate_full_graph(rc, st, eval_batch, *ds, p, eps);
      if (eval_logits)
        logits[static_cast<std::size_t>(rc.rank())] = forward(rc, st, eval_batch, p, false, 0, 0, eps).logits;
    });
    for (int i = 0; i < 3; ++i) {
      counts[i] = res[0].correct[static_cast<std::size_t>(i)];
      counts[3 + i] = res[0].total[static_cast<std::size_t>(i)];
    }
    if (eval_logits)
      for (int r = 0; r < grid.total(); ++r)
        if (grid.dp_group(r) == 0) put_tile(logits[static_cast<std::size_t>(r)], eval_logits);
  });
}

/// CommStats of the train_run step loop (model.hpp:646-685): n_steps of
/// [build_step_batch -> train_step (forward/backward phases) -> dp_sync ->
/// optimizer_step], then (eval != 0) evaluate_full_graph on the b = n eval
/// batch outside any phase. out[28] = Communicator::snapshot(): bytes[axis]
/// [phase] (20), all-reduce calls (4), all-gather calls (4), axes D,X,Y,Z.
int ref_comm_stats(void* dsp, const int* dims, const std::int64_t* mc, const double* md, std::int64_t b,
                   std::uint64_t seed, int n_steps, int prec, int eval, std::uint64_t* out) {
  auto* ds = static_cast<Dataset*>(dsp);
  return guard([&] {
    const ModelConfig mcfg = make_cfg(mc, md);
    DeviceGrid grid(dims[0], dims[1], dims[2], dims[3]);
    Communicator comm(grid);
    const Precision p = prec ? Precision::kBf16Roundtrip : Precision::kFp32;
    run_ranks(comm, [&](RankComm& rc) {
      const int dp = grid.dp_group(rc.rank());
      const std::uint64_t group_seed = rng::hash_combine(seed, static_cast<std::uint64_t>(dp));
      RankContext ctx = make_rank_context(grid, rc.coord(), *ds, mcfg.layers);
      auto st = init_state<float>(grid, rc.coord(), mcfg, seed);
      for (int s = 0; s < n_steps; ++s) {
        const auto gstep = static_cast<std::uint64_t>(s);
        StepBatch<float> batch;
        {
          PhaseScope ps(rc, Phase::kSampling);
          batch = build_step_batch<float>(grid, rc.coord(), ctx, *ds, b, group_seed, gstep, &rc.stats());
        }
        train_step(rc, st, batch, p, seed, gstep, 1e-6);
        dp_sync(rc, st);
        optimizer_step(st, Optimizer::kAdam, 1e-3);
      }
      if (eval) {
        const auto eval_batch = build_step_batch<float>(grid, rc.coord(), ctx, *ds, ds->n, seed, 0, nullptr);
        evaluate_full_graph(rc, st, eval_batch, *ds, p, 1e-6);
      }
    });
    const CommStats snap = comm.snapshot();
    for (int a = 0; a < 4; ++a) {
      for (int q = 0; q < kNumPhases; ++q) out[a * kNumPhases + q] = snap.bytes[a][q];
      out[20 + a] = snap.allreduce_calls[a];
      out[24 + a] = snap.allgather_calls[a];
    }
  });
}

/// Initial weights (init_state on the 1x1x1x1 grid), flattened in
/// param_views order.
int ref_init_weights(const std::int64_t* mc, const double* md, std::uint64_t seed, float* out) {
  return guard([&] {
    const ModelConfig mcfg = make_cfg(mc, md);
    DeviceGrid grid(1, 1, 1, 1);
    std::vector<ModelState<float>> st{init_state<float>(grid, {0, 0, 0, 0}, mcfg, seed)};
    export_params(st, 0, out);
  });
}

/// CPU baseline: the train_run step body (model.hpp:646-685, without the
/// per-epoch eval) timed per step with steady_clock, one std::thread per rank
/// as train_run does (model.hpp:724-733). step_ms[k] = max over ranks of the
/// k-th timed step; phase_ms = {sample, fwd, bwd, dpsync, opt} summed over the
/// timed steps on rank 0. Runs `warmup` untimed steps first.
int ref_bench(void* dsp, const int* dims, const std::int64_t* mc, const double* md, std::int64_t b,
              std::uint64_t seed, int warmup, int steps, int prec, double* step_ms,
              double* phase_ms) {
  auto* ds = static_cast<Dataset*>(dsp);
  return guard([&] {
    const ModelConfig mcfg = make_cfg(mc, md);
    DeviceGrid grid(dims[0], dims[1], dims[2], dims[3]);
    Communicator comm(grid);
    const Precision p = prec ? Precision::kBf16Roundtrip : Precision::kFp32;
    const int R = grid.total();
    std::vector<std::vector<double>> per(static_cast<std::size_t>(R),
                                         std::vector<double>(static_cast<std::size_t>(steps), 0.0));
    std::vector<double> ph(5, 0.0);
    run_ranks(comm, [&](RankComm& rc) {
      using clock = std::chrono::steady_clock;
      auto ms = [](clock::time_point t0) {
        return std::chrono::duration<double, std::milli>(clock::now() - t0).count();
      };
      const int dp = grid.dp_group(rc.rank());
      const std::uint64_t group_seed = rng::hash_combine(seed, static_cast<std::uint64_t>(dp));
      RankContext ctx = make_rank_context(grid, rc.coord(), *ds, mcfg.layers);
      auto st = init_state<float>(grid, rc.coord(), mcfg, seed);
      for (int s = 0; s < warmup + steps; ++s) {
        rc.barrier();
        const auto t_step = clock::now();
        auto t0 = clock::now();
        auto batch = build_step_batch<float>(grid, rc.coord(), ctx, *ds, b, group_seed,
                                             static_cast<std::uint64_t>(s), &rc.stats());
        const double t_s = ms(t0);
        t0 = clock::now();
        auto cache = forward(rc, st, batch, p, true, seed, static_cast<std::uint64_t>(s), 1e-6);
        auto ce = parallel_cross_entropy(rc, cache.logits, batch.labels);
        const double t_f = ms(t0);
        t0 = clock::now();
        backward(rc, st, cache, batch, ce.grad_logits, p);
        const double t_b = ms(t0);
        t0 = clock::now();
        dp_sync(rc, st);
        const double t_d = ms(t0);
        t0 = clock::now();
        optimizer_step(st, Optimizer::kAdam, 1e-3);
        const double t_o = ms(t0);
        if (s >= warmup) {
          per[static_cast<std::size_t>(rc.rank())][static_cast<std::size_t>(s - warmup)] = ms(t_step);
          if (rc.rank() == 0) {
            ph[0] += t_s;
            ph[1] += t_f;
            ph[2] += t_b;
            ph[3] += t_d;
            ph[4] += t_o;
          }
        }
      }
    });
    for (int s = 0; s < steps; ++s) {
      double m = 0.0;
      for (int r = 0; r < R; ++r) m = std::max(m, per[static_cast<std::size_t>(r)][static_cast<std::size_t>(s)]);
      step_ms[s] = m;
    }
    if (phase_ms)
      for (int k = 0; k < 5; ++k) phase_ms[k] = ph[static_cast<std::size_t>(k)];
  });
}


// ---- layer operators (pmm.hpp:76-401) on the one-rank grid ------------------
// Each runs the reference operator on full-matrix shards (offsets {0, n}) of a
// 1x1x1x1 grid, layout (X, Y) for dense operands.
}  // extern "C"

namespace {
ShardedTensor<float> full_shard(Layout lay, std::int64_t rows, std::int64_t cols, const float* v) {
  DeviceGrid g(1, 1, 1, 1);
  auto t = make_sharded<float>(g, g.coord_of(0), lay, rows, cols, {0, rows}, {0, cols});
  if (v) std::copy(v, v + rows * cols, t.local.v.begin());
  return t;
}
template <class Body>
void one_rank(Body&& body) {
  Communicator comm(DeviceGrid(1, 1, 1, 1));
  RankComm rc(comm, 0);
  body(rc);
}
}  // namespace

extern "C" {

int ref_contract(std::int64_t m, std::int64_t k, std::int64_t n, const float* a, const float* b, int prec, float* c) {
  return guard([&] {
    one_rank([&](RankComm& rc) {
      auto A = full_shard({Axis::X, Axis::Y}, m, k, a);
      auto B = full_shard({Axis::Y, Axis::Z}, k, n, b);
      auto C = contract(rc, A, B, prec ? Precision::kBf16Roundtrip : Precision::kFp32);
      std::copy(C.local.v.begin(), C.local.v.end(), c);
    });
  });
}

int ref_spmm(std::int64_t rows, std::int64_t cols, const std::int64_t* rp, const std::int64_t* col, const double* val,
             const float* f, std::int64_t n, int prec, float* h) {
  return guard([&] {
    one_rank([&](RankComm& rc) {
      ShardedSparse A;
      A.layout = {Axis::Z, Axis::X};
      A.g_rows = rows;
      A.g_cols = cols;
      A.row_off = {0, rows};
      A.col_off = {0, cols};
      A.r1 = rows;
      A.c1 = cols;
      A.local.n_rows = rows;
      A.local.n_cols = cols;
      A.local.row_ptr.assign(rp, rp + rows + 1);
      A.local.col_idx.assign(col, col + rp[rows]);
      A.local.values.assign(val, val + rp[rows]);
      auto F = full_shard({Axis::X, Axis::Y}, cols, n, f);
      auto H = spmm(rc, A, F, prec ? Precision::kBf16Roundtrip : Precision::kFp32);
      std::copy(H.local.v.begin(), H.local.v.end(), h);
    });
  });
}

int ref_rmsnorm(std::int64_t m, std::int64_t n, const float* x, const float* gamma, float eps, const float* dy,
                float* y, float* rms, float* dx, float* dgamma) {
  return guard([&] {
    one_rank([&](RankComm& rc) {
      auto X = full_shard({Axis::X, Axis::Y}, m, n, x);
      auto r = parallel_rmsnorm_fwd(rc, X, std::span<const float>(gamma, static_cast<std::size_t>(n)), eps);
      std::copy(r.y.local.v.begin(), r.y.local.v.end(), y);
      std::copy(r.rms.begin(), r.rms.end(), rms);
      if (dy) {
        auto DY = full_shard({Axis::X, Axis::Y}, m, n, dy);
        auto g = parallel_rmsnorm_bwd(rc, X, std::span<const float>(gamma, static_cast<std::size_t>(n)), r.rms, DY);
        std::copy(g.dx.local.v.begin(), g.dx.local.v.end(), dx);
        std::copy(g.dgamma.begin(), g.dgamma.end(), dgamma);
      }
    });
  });
}

int ref_fused(std::int64_t m, std::int64_t n, const float* x, const float* h_prev, double rate, std::uint64_t key,
              int training, const float* dy, float* out, float* scale, float* dx) {
  return guard([&] {
    auto X = full_shard({Axis::X, Axis::Y}, m, n, x);
    ShardedTensor<float> H;
    if (h_prev) H = full_shard({Axis::X, Axis::Y}, m, n, h_prev);
    auto r = fused_elementwise_fwd<float>(X, h_prev ? &H : nullptr, rate, key, training != 0);
    std::copy(r.out.local.v.begin(), r.out.local.v.end(), out);
    std::copy(r.scale.v.begin(), r.scale.v.end(), scale);
    if (dy) {
      auto DY = full_shard({Axis::X, Axis::Y}, m, n, dy);
      auto d = fused_elementwise_bwd(DY, r.scale);
      std::copy(d.local.v.begin(), d.local.v.end(), dx);
    }
  });
}

int ref_cross_entropy(std::int64_t m, std::int64_t n, const float* logits, const std::int32_t* labels, float* loss,
                      float* grad) {
  return guard([&] {
    one_rank([&](RankComm& rc) {
      auto L = full_shard({Axis::X, Axis::Z}, m, n, logits);
      auto r = parallel_cross_entropy(rc, L, std::vector<std::int32_t>(labels, labels + m));
      *loss = r.loss;
      std::copy(r.grad_logits.local.v.begin(), r.grad_logits.local.v.end(), grad);
    });
  });
}

}  // extern "C"
