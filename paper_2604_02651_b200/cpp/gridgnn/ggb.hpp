// gridgnn drop-in (header-only C++20) over the C ABI of libggb.so.
//
// Restores the reference's hot-path C++ surface (namespace gridgnn,
// /root/reference/proj/include/gridgnn) on top of the B200 implementation:
// the same names, by-value results and exception types
//   std::invalid_argument  <- GGB_EINVAL
//   gridgnn::CommContract  <- GGB_ECONTRACT   (comm.hpp:44-46)
//   gridgnn::CommTimeout   <- GGB_ETIMEOUT    (comm.hpp:41-43)
//   std::runtime_error     <- CUDA / NCCL failures
// Device state lives behind RAII handles; host copies are materialized only
// by the accessors (the reference's "parity mode" field access).
#pragma once

#include <array>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/ggb.h"

namespace gridgnn {

using index_t = std::int64_t;

struct CommTimeout : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CommContract : std::logic_error {
  using std::logic_error::logic_error;
};

enum class Precision { kFp32 = GGB_FP32, kBf16Roundtrip = GGB_BF16_WIRE };  // comm.hpp:22
enum class Optimizer { kSgd = GGB_SGD, kAdam = GGB_ADAM };                 // model.hpp:45
enum class Axis : int { D = 0, X = 1, Y = 2, Z = 3 };                       // grid.hpp:11
enum class SplitTag : std::uint8_t { kTrain = 0, kVal = 1, kTest = 2, kUnused = 3 };  // dataset.hpp:12

namespace detail {
inline void check(int rc) {
  if (rc == GGB_OK) return;
  const std::string msg = ggb_last_error();
  switch (rc) {
    case GGB_EINVAL: throw std::invalid_argument(msg);
    case GGB_ECONTRACT: throw CommContract(msg);
    case GGB_ETIMEOUT: throw CommTimeout(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

/// grid.hpp:18-73 (lexicographic rank = ((d*gx + x)*gy + y)*gz + z).
struct DeviceGrid {
  std::int32_t dims[4] = {1, 1, 1, 1};
  DeviceGrid() = default;
  DeviceGrid(int gd, int gx, int gy, int gz) : dims{gd, gx, gy, gz} {
    for (int d : dims)
      if (d < 1) throw std::invalid_argument("DeviceGrid: dims must be >= 1");
  }
  int total() const { return dims[0] * dims[1] * dims[2] * dims[3]; }
  int dim(Axis a) const { return dims[static_cast<int>(a)]; }
  int dp_group(int rank) const { return rank / (dims[1] * dims[2] * dims[3]); }
};

/// sampling.hpp:13-19
struct SampleSet {
  std::vector<index_t> vertices;
  index_t batch_size = 0, graph_size = 0;
  std::uint64_t seed = 0, step = 0;
};

/// csr.hpp:13-24 (int64 indices, fp64 values)
struct CsrMatrix {
  index_t n_rows = 0, n_cols = 0;
  std::vector<index_t> row_ptr{0};
  std::vector<index_t> col_idx;
  std::vector<double> values;
  index_t nnz() const { return static_cast<index_t>(col_idx.size()); }
  bool operator==(const CsrMatrix&) const = default;
};

/// model.hpp:26-43
struct ModelConfig {
  int layers = 2;
  index_t d_in = 0, d_h = 64, d_out = 0;
  double dropout_rate = 0.1;
  bool use_rmsnorm = true, use_dropout = true, use_residual = true;
  ggb_model_config c() const {
    return {layers, d_in, d_h, d_out, dropout_rate, use_rmsnorm, use_dropout, use_residual};
  }
};

inline std::vector<index_t> block_partition(index_t n, int g) {  // shardsample.cpp:8-17
  if (g < 1) throw std::invalid_argument("block_partition: g must be >= 1");
  std::vector<index_t> off(static_cast<size_t>(g) + 1, 0);
  for (int k = 0; k < g; ++k) off[k + 1] = off[k] + n / g + (k < n % g ? 1 : 0);
  return off;
}

inline index_t steps_per_epoch(index_t n, index_t b, int gd) {  // model.hpp:539-542
  const index_t per = b * gd;
  return (n + per - 1) / per;
}

enum class Phase : int { kSampling = 0, kForward, kBackward, kDpSync, kOther };  // comm.hpp:24
inline constexpr int kNumPhases = 5;

/// CommStats (comm.hpp:94-117): the reference's byte accounting of the
/// logical collectives (ring-equivalent all-reduce volume, full all-gather
/// payload, singleton groups free).
struct CommStats {
  std::array<std::array<std::uint64_t, kNumPhases>, 4> bytes{};
  std::array<std::uint64_t, 4> allreduce_calls{};
  std::array<std::uint64_t, 4> allgather_calls{};
  std::uint64_t bytes_on(Axis a) const {
    std::uint64_t s = 0;
    for (auto b : bytes[static_cast<std::size_t>(static_cast<int>(a))]) s += b;
    return s;
  }
  std::uint64_t phase_bytes(Phase p) const {
    std::uint64_t s = 0;
    for (const auto& ax : bytes) s += ax[static_cast<std::size_t>(static_cast<int>(p))];
    return s;
  }
  std::uint64_t sampling_bytes() const { return phase_bytes(Phase::kSampling); }
  std::uint64_t total_bytes() const {
    std::uint64_t s = 0;
    for (const auto& ax : bytes)
      for (auto b : ax) s += b;
    return s;
  }
  CommStats operator-(const CommStats& o) const {
    CommStats d;
    for (int a = 0; a < 4; ++a) {
      for (int p = 0; p < kNumPhases; ++p) d.bytes[a][p] = bytes[a][p] - o.bytes[a][p];
      d.allreduce_calls[a] = allreduce_calls[a] - o.allreduce_calls[a];
      d.allgather_calls[a] = allgather_calls[a] - o.allgather_calls[a];
    }
    return d;
  }
};

/// One rank on one GPU (replaces Communicator + RankComm, comm.hpp:203-408).
class RankComm {
 public:
  /// nccl_uid: 128 bytes from unique_id() on rank 0 (nullptr: virtual rank,
  /// multi-rank collectives throw CommContract).
  RankComm(const DeviceGrid& grid, int rank, int device = 0, const std::uint8_t* nccl_uid = nullptr,
           void* stream = nullptr)
      : grid_(grid), rank_(rank) {
    detail::check(ggb_ctx_create(grid.dims, rank, device, nccl_uid, stream, &h_));
  }
  ~RankComm() {
    if (h_) ggb_ctx_destroy(h_);
  }
  RankComm(const RankComm&) = delete;
  RankComm& operator=(const RankComm&) = delete;
  static std::vector<std::uint8_t> unique_id() {
    std::vector<std::uint8_t> id(128);
    detail::check(ggb_get_unique_id(id.data()));
    return id;
  }
  int rank() const { return rank_; }
  const DeviceGrid& grid() const { return grid_; }
  /// grid.hpp Coord4 of this rank: rank = ((d*gx + x)*gy + y)*gz + z
  std::array<int, 4> coord() const {
    std::array<int, 4> c{};
    int r = rank_;
    for (int a = 3; a >= 0; --a) {
      c[static_cast<size_t>(a)] = r % grid_.dims[a];
      r /= grid_.dims[a];
    }
    return c;
  }
  void synchronize() { detail::check(ggb_ctx_synchronize(h_)); }
  ggb_ctx_t handle() const { return h_; }
  /// This rank's counters (RankStats), or with grid_total the sum over the
  /// grid (Communicator::snapshot; collective, every rank calls it).
  CommStats comm_stats(bool grid_total = false, bool reset = false) {
    std::uint64_t v[GGB_COMM_STATS_LEN];
    detail::check(ggb_ctx_comm_stats(h_, grid_total ? 1 : 0, reset ? 1 : 0, v));
    CommStats s;
    for (int a = 0; a < 4; ++a) {
      for (int p = 0; p < kNumPhases; ++p) s.bytes[a][p] = v[a * kNumPhases + p];
      s.allreduce_calls[a] = v[20 + a];
      s.allgather_calls[a] = v[24 + a];
    }
    return s;
  }
  CommStats snapshot() { return comm_stats(true); }

 private:
  DeviceGrid grid_;
  int rank_;
  ggb_ctx_t h_ = nullptr;
};

/// sampling.hpp:33 — sampled on the GPU, bit-exact with the reference.
inline SampleSet sample_vertices(RankComm& rc, index_t n, index_t b, std::uint64_t seed, std::uint64_t step) {
  SampleSet s;
  if (b <= 0 || b > n) throw std::invalid_argument("sample_vertices: need 1 <= b <= n");
  s.vertices.resize(static_cast<size_t>(b));
  detail::check(ggb_sample_vertices(rc.handle(), n, b, seed, step, s.vertices.data()));
  s.batch_size = b;
  s.graph_size = n;
  s.seed = seed;
  s.step = step;
  return s;
}

/// Host Dataset (dataset.hpp:16-29) with the reference's file formats
/// (load_dataset / save_*, dataset.cpp:152-280) and generator; no GPU needed.
class Dataset {
 public:
  explicit Dataset(ggb_dataset_t h) : h_(h) {}
  Dataset(Dataset&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Dataset(const Dataset&) = delete;
  Dataset& operator=(const Dataset&) = delete;
  ~Dataset() {
    if (h_) ggb_dataset_destroy(h_);
  }
  /// save_edge_list + save_features + save_labels + save_split (the CLI's gen output)
  void save(const std::string& edges, const std::string& features, const std::string& labels,
            const std::string& split) const {
    detail::check(ggb_dataset_save(h_, edges.c_str(), features.c_str(), labels.c_str(), split.c_str()));
  }
  index_t n() const { return info(0); }
  index_t nnz() const { return info(1); }
  index_t d_in() const { return info(2); }
  index_t n_classes() const { return info(3); }
  ggb_dataset_t handle() const { return h_; }

 private:
  index_t info(int k) const {
    index_t v[5];
    detail::check(ggb_dataset_info(h_, v));
    return v[k];
  }
  ggb_dataset_t h_ = nullptr;
};

/// load_dataset (dataset.cpp:178-239): the same files, validation and messages.
inline Dataset load_dataset(const std::string& graph_path, const std::string& feature_path,
                            const std::string& label_path, const std::string& split_path) {
  ggb_dataset_t h = nullptr;
  detail::check(ggb_dataset_load(graph_path.c_str(), feature_path.c_str(), label_path.c_str(), split_path.c_str(), &h));
  return Dataset(h);
}

/// generate_synthetic (dataset.cpp:85-131) on the host, bit-identical.
inline Dataset generate_synthetic(index_t n, double avg_degree, index_t d_in, index_t n_classes, std::uint64_t seed) {
  ggb_dataset_t h = nullptr;
  detail::check(ggb_dataset_generate_synthetic(n, avg_degree, d_in, n_classes, seed, &h));
  return Dataset(h);
}

/// Dataset + RankContext resident in HBM (dataset.hpp:16-29, model.hpp:212-234).
class DeviceDataset {
 public:
  /// make_rank_context from a host Dataset (its split tags included).
  DeviceDataset(RankComm& rc, const Dataset& ds, int layers) {
    detail::check(ggb_graph_from_dataset(rc.handle(), ds.handle(), layers, &h_));
  }
  /// generate_synthetic built on the GPU.
  static DeviceDataset generate_on_device(RankComm& rc, index_t n, double avg_degree, index_t d_in,
                                          index_t n_classes, std::uint64_t seed, int layers) {
    ggb_graph_t h = nullptr;
    detail::check(ggb_graph_generate_synthetic_device(rc.handle(), n, avg_degree, d_in, n_classes, seed, layers, &h));
    return DeviceDataset(h);
  }
  DeviceDataset(DeviceDataset&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  /// keep the features in host memory, as the reference's Dataset does
  void features_to_host() { detail::check(ggb_graph_features_to_host(h_)); }
  DeviceDataset(RankComm& rc, const CsrMatrix& adjacency, index_t d_in, const std::vector<float>& features,
                index_t n_classes, const std::vector<std::int32_t>& labels, int layers, bool symmetric = true,
                const std::vector<SplitTag>* split = nullptr) {
    detail::check(ggb_graph_create(rc.handle(), adjacency.n_rows, adjacency.row_ptr.data(), adjacency.col_idx.data(),
                                   adjacency.values.data(), symmetric, d_in, features.data(), n_classes, labels.data(),
                                   layers, &h_));
    if (split) set_split(*split);
  }
  /// generate_synthetic (dataset.cpp:85-131), built natively.
  DeviceDataset(RankComm& rc, index_t n, double avg_degree, index_t d_in, index_t n_classes, std::uint64_t seed,
                int layers) {
    detail::check(ggb_graph_generate_synthetic(rc.handle(), n, avg_degree, d_in, n_classes, seed, layers, &h_));
  }
  ~DeviceDataset() {
    if (h_) ggb_graph_destroy(h_);
  }
  DeviceDataset(const DeviceDataset&) = delete;
  DeviceDataset& operator=(const DeviceDataset&) = delete;
  /// Dataset::split (dataset.hpp:23); generate_synthetic sets it itself.
  void set_split(const std::vector<SplitTag>& split) {
    if (static_cast<index_t>(split.size()) != n()) throw std::invalid_argument("set_split: one tag per vertex");
    detail::check(ggb_graph_set_split(h_, reinterpret_cast<const std::uint8_t*>(split.data())));
  }
  ggb_graph_t handle() const { return h_; }
  index_t n() const { return info(0); }
  index_t nnz() const { return info(1); }

 private:
  explicit DeviceDataset(ggb_graph_t h) : h_(h) {}
  index_t info(int k) const {
    index_t v[7];
    detail::check(ggb_graph_info(h_, v));
    return v[k];
  }
  ggb_graph_t h_ = nullptr;
};

/// StepBatch (model.hpp:238-246) resident in HBM; accessors copy to the host.
class StepBatch {
 public:
  StepBatch() = default;
  ~StepBatch() {
    if (h_ && own_) ggb_batch_destroy(h_);
  }
  StepBatch(const StepBatch&) = delete;
  StepBatch& operator=(const StepBatch&) = delete;
  StepBatch(StepBatch&& o) noexcept : h_(o.h_), own_(o.own_) { o.h_ = nullptr; }
  StepBatch& operator=(StepBatch&& o) noexcept {
    if (this != &o) {
      if (h_ && own_) ggb_batch_destroy(h_);
      h_ = o.h_;
      own_ = o.own_;
      o.h_ = nullptr;
    }
    return *this;
  }
  ggb_batch_t handle() const { return h_; }
  ggb_batch_t* slot() { return &h_; }
  static StepBatch borrow(ggb_batch_t h) {
    StepBatch b;
    b.h_ = h;
    b.own_ = false;
    return b;
  }

  SampleSet sample() const {
    SampleSet s;
    index_t info[9];
    detail::check(ggb_batch_info(h_, info));
    s.vertices.resize(static_cast<size_t>(info[0]));
    detail::check(ggb_batch_sample(h_, s.vertices.data()));
    s.batch_size = info[0];
    s.graph_size = info[1];
    return s;
  }
  std::vector<index_t> batch_off(Axis a) const {
    std::vector<index_t> v(64);
    detail::check(ggb_batch_offsets(h_, static_cast<int>(a), v.data()));
    return v;
  }
  /// a[p] (transposed == false) or a_t[p]: local CSR block (MiniBatchShard a_loc / a_t_loc)
  CsrMatrix plane(int p, bool transposed) const {
    index_t dims[7];
    detail::check(ggb_batch_plane(h_, p, transposed, dims, nullptr, nullptr, nullptr));
    CsrMatrix m;
    m.n_rows = dims[0];
    m.n_cols = dims[1];
    m.row_ptr.resize(static_cast<size_t>(dims[0] + 1));
    m.col_idx.resize(static_cast<size_t>(dims[2]));
    m.values.resize(static_cast<size_t>(dims[2]));
    detail::check(ggb_batch_plane(h_, p, transposed, dims, m.row_ptr.data(), m.col_idx.data(), m.values.data()));
    return m;
  }
  /// {nnz_extracted, nnz_kept} work counters (MiniBatchShard, shardsample.hpp:111-113)
  std::array<std::uint64_t, 2> counters() const {
    index_t info[9];
    detail::check(ggb_batch_info(h_, info));
    return {static_cast<std::uint64_t>(info[7]), static_cast<std::uint64_t>(info[8])};
  }
  std::vector<std::int32_t> labels() const {
    std::vector<std::int32_t> v(static_cast<size_t>(sample_size()));
    detail::check(ggb_batch_labels(h_, v.data()));
    return v;
  }

 private:
  index_t sample_size() const {
    index_t info[9];
    detail::check(ggb_batch_info(h_, info));
    return info[0];
  }
  ggb_batch_t h_ = nullptr;
  bool own_ = true;
};

/// build_step_batch (model.hpp:250-309): communication-free. Reuses the
/// batch's device buffers when passed back in.
inline void build_step_batch(RankComm& rc, const DeviceDataset& ds, index_t b, std::uint64_t group_seed,
                             std::uint64_t step, StepBatch& inout) {
  detail::check(ggb_build_step_batch(rc.handle(), ds.handle(), b, group_seed, step, inout.slot()));
}
inline StepBatch build_step_batch(RankComm& rc, const DeviceDataset& ds, index_t b, std::uint64_t group_seed,
                                  std::uint64_t step) {
  StepBatch sb;
  build_step_batch(rc, ds, b, group_seed, step, sb);
  return sb;
}

/// ModelState (model.hpp:87-105) resident in HBM.
class ModelState {
 public:
  ModelState(RankComm& rc, const ModelConfig& cfg, std::uint64_t seed) : cfg_(cfg) {  // init_state
    const ggb_model_config c = cfg.c();
    detail::check(ggb_state_create(rc.handle(), &c, seed, &h_));
  }
  ~ModelState() {
    if (h_) ggb_state_destroy(h_);
  }
  ModelState(const ModelState&) = delete;
  ModelState& operator=(const ModelState&) = delete;
  ggb_state_t handle() const { return h_; }
  const ModelConfig& cfg() const { return cfg_; }
  int num_params() const { return ggb_state_num_params(h_); }
  /// param_views order (model.hpp:107-133): which 0 weight, 1 grad, 2 m, 3 v
  std::vector<float> param(int idx, int which = 0) const {
    index_t info[6];
    detail::check(ggb_state_param_info(h_, idx, info));
    std::vector<float> v(static_cast<size_t>((info[3] - info[2]) * (info[5] - info[4])));
    detail::check(ggb_state_param_get(h_, idx, which, v.data()));
    return v;
  }

 private:
  ModelConfig cfg_;
  ggb_state_t h_ = nullptr;
};

inline ModelState init_state(RankComm& rc, const ModelConfig& cfg, std::uint64_t seed) { return {rc, cfg, seed}; }

/// train_step (model.hpp:459-478): forward + cross-entropy + backward.
inline float train_step(RankComm& rc, ModelState& st, const StepBatch& batch, Precision prec, std::uint64_t run_seed,
                        std::uint64_t global_step, double rmsnorm_eps = 1e-6) {
  float loss = 0.f;
  detail::check(ggb_train_step(rc.handle(), st.handle(), batch.handle(), static_cast<int>(prec), run_seed,
                               global_step, rmsnorm_eps, &loss));
  return loss;
}

inline void dp_sync(RankComm& rc, ModelState& st) { detail::check(ggb_dp_sync(rc.handle(), st.handle())); }

inline void optimizer_step(RankComm& rc, ModelState& st, Optimizer opt, double lr) {
  detail::check(ggb_optimizer_step(rc.handle(), st.handle(), static_cast<int>(opt), lr));
}

/// EvalCounts (model.hpp:480-490).
struct EvalCounts {
  std::array<std::uint64_t, 3> correct{};  // train, val, test
  std::array<std::uint64_t, 3> total{};
  double accuracy(SplitTag s) const {
    const auto i = static_cast<std::size_t>(s);
    return total[i] == 0 ? 0.0 : static_cast<double>(correct[i]) / static_cast<double>(total[i]);
  }
};

/// train_run's eval batch: every vertex, seed = run seed, step 0 (model.hpp:625).
inline StepBatch build_eval_batch(RankComm& rc, const DeviceDataset& ds, std::uint64_t seed) {
  return build_step_batch(rc, ds, ds.n(), seed, 0);
}

/// evaluate_full_graph (model.hpp:493-537): dropout-off forward over the eval
/// batch, argmax per vertex (ties to the lowest class id), per-split counts
/// summed over the grid (identical on every rank).
inline EvalCounts evaluate_full_graph(RankComm& rc, ModelState& st, const StepBatch& eval_batch,
                                      const DeviceDataset& ds, Precision prec, double rmsnorm_eps = 1e-6) {
  std::uint64_t c[6];
  detail::check(ggb_evaluate_full_graph(rc.handle(), st.handle(), eval_batch.handle(), ds.handle(),
                                        static_cast<int>(prec), rmsnorm_eps, c));
  EvalCounts out;
  for (int i = 0; i < 3; ++i) {
    out.correct[static_cast<std::size_t>(i)] = c[i];
    out.total[static_cast<std::size_t>(i)] = c[3 + i];
  }
  return out;
}

/// The train_run producer thread + PrefetchQueue (model.hpp:556-581).
class Prefetcher {
 public:
  Prefetcher(RankComm& rc, const DeviceDataset& ds, index_t b, std::uint64_t group_seed, std::uint64_t first_step,
             std::uint64_t run_seed = 0, const ModelConfig* cfg = nullptr) {
    const int layers = (cfg && cfg->use_dropout) ? cfg->layers : 0;
    detail::check(ggb_prefetch_create(rc.handle(), ds.handle(), b, group_seed, first_step, run_seed, layers,
                                      cfg ? cfg->d_h : 0, cfg ? cfg->dropout_rate : 0.0, &h_));
  }
  ~Prefetcher() {
    if (h_) ggb_prefetch_destroy(h_);
  }
  Prefetcher(const Prefetcher&) = delete;
  Prefetcher& operator=(const Prefetcher&) = delete;
  StepBatch next() {
    ggb_batch_t b = nullptr;
    detail::check(ggb_prefetch_next(h_, &b));
    return StepBatch::borrow(b);
  }

 private:
  ggb_prefetch_t h_ = nullptr;
};

struct TrainConfig {  // model.hpp:47-58 (the fields of the step loop)
  DeviceGrid grid;
  index_t batch = 0;
  int epochs = 1;
  std::uint64_t seed = 0;
  Precision precision = Precision::kFp32;
  bool prefetch = false;
  Optimizer optimizer = Optimizer::kAdam;
  double lr = 1e-3;
  double rmsnorm_eps = 1e-6;
  bool evaluate = true;  // per-epoch evaluate_full_graph, as train_run always does
};

/// EpochMetrics (metrics.hpp:13-29). Timings are host wall-clock around the
/// device calls (sampling wait, train_step = forward + CE + backward, which
/// the device runs back to back, so t_bwd_ms stays 0; dp_sync). Byte columns:
/// the epoch's CommStats delta summed over the grid (model.hpp:706-716).
struct EpochMetrics {
  int epoch = 0;
  std::int64_t step = 0;
  double loss = 0.0;
  double train_acc = 0.0, val_acc = 0.0, test_acc = 0.0;
  double t_sample_ms = 0.0, t_fwd_ms = 0.0, t_bwd_ms = 0.0, t_dpsync_ms = 0.0;
  std::uint64_t bytes_x = 0, bytes_y = 0, bytes_z = 0, bytes_d = 0;
};

/// TrainReport (metrics.hpp:31-44) of one rank.
struct TrainReport {
  std::vector<EpochMetrics> epochs;
  std::vector<double> step_losses;
  std::uint64_t sampled_nnz_extracted = 0;
  std::uint64_t sampled_nnz_kept = 0;
  CommStats comm_total;  // grid total at the end of the run
  double wall_ms = 0.0;
  double final_train_acc() const { return epochs.empty() ? 0.0 : epochs.back().train_acc; }
  double final_val_acc() const { return epochs.empty() ? 0.0 : epochs.back().val_acc; }
  double final_test_acc() const { return epochs.empty() ? 0.0 : epochs.back().test_acc; }
};

/// metrics_csv_string / write_metrics_csv (metrics.cpp:10-32): the same
/// fixed columns and exact (%.17g) number formatting.
inline std::string metrics_csv_string(const TrainReport& report) {
  std::string out =
      "epoch,step,loss,train_acc,val_acc,test_acc,t_sample_ms,t_fwd_ms,t_bwd_ms,"
      "t_dpsync_ms,bytes_x,bytes_y,bytes_z,bytes_d\n";
  char buf[512];
  for (const auto& e : report.epochs) {
    std::snprintf(buf, sizeof(buf),
                  "%d,%lld,%.17g,%.17g,%.17g,%.17g,%.3f,%.3f,%.3f,%.3f,%llu,%llu,%llu,%llu\n", e.epoch,
                  static_cast<long long>(e.step), e.loss, e.train_acc, e.val_acc, e.test_acc, e.t_sample_ms,
                  e.t_fwd_ms, e.t_bwd_ms, e.t_dpsync_ms, static_cast<unsigned long long>(e.bytes_x),
                  static_cast<unsigned long long>(e.bytes_y), static_cast<unsigned long long>(e.bytes_z),
                  static_cast<unsigned long long>(e.bytes_d));
    out += buf;
  }
  return out;
}

inline void write_metrics_csv(const std::string& path, const TrainReport& report) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot open metrics file for writing: " + path);
  const std::string s = metrics_csv_string(report);
  const bool ok = std::fwrite(s.data(), 1, s.size(), f) == s.size();
  std::fclose(f);
  if (!ok) throw std::runtime_error("failed writing metrics file: " + path);
}

/// train_run of one rank (model.hpp:588-747; the reference runs one thread per
/// rank, here one process per GPU): S = steps_per_epoch steps per epoch, per
/// step [batch -> train_step -> dp_sync -> optimizer_step], then the per-epoch
/// full-graph evaluation.
inline TrainReport train_run(RankComm& rc, const DeviceDataset& ds, const ModelConfig& mcfg,
                             const TrainConfig& tcfg) {
  using clock = std::chrono::steady_clock;
  auto ms_since = [](clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(clock::now() - t0).count();
  };
  const auto run_start = clock::now();
  if (tcfg.batch < 2 || tcfg.batch > ds.n()) throw std::invalid_argument("train_run: batch size must be in [2, N]");
  if (tcfg.epochs < 1) throw std::invalid_argument("train_run: epochs must be >= 1");
  const int dp = tcfg.grid.dp_group(rc.rank());
  const std::uint64_t group_seed = [&] {  // rng::hash_combine(seed, dp) (model.hpp:620-621)
    auto sm = [](std::uint64_t x) {
      x += 0x9e3779b97f4a7c15ULL;
      x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
      x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
      return x ^ (x >> 31);
    };
    const std::uint64_t b = static_cast<std::uint64_t>(dp);
    return sm(tcfg.seed ^ (0x9e3779b97f4a7c15ULL + (b << 6) + (b >> 2)));
  }();
  const index_t S = steps_per_epoch(ds.n(), tcfg.batch, tcfg.grid.dims[0]);
  ModelState st(rc, mcfg, tcfg.seed);
  TrainReport report;
  StepBatch eval_batch;
  if (tcfg.evaluate) eval_batch = build_eval_batch(rc, ds, tcfg.seed);
  std::unique_ptr<Prefetcher> pf;
  if (tcfg.prefetch) pf = std::make_unique<Prefetcher>(rc, ds, tcfg.batch, group_seed, 0, tcfg.seed, &mcfg);
  StepBatch batch;
  std::uint64_t gstep = 0;
  const CommStats run_start_stats = rc.snapshot();  // the reference's Communicator starts at zero
  CommStats prev_snapshot = run_start_stats;
  for (int epoch = 0; epoch < tcfg.epochs; ++epoch) {
    EpochMetrics row;
    double loss_sum = 0.0;
    for (index_t s = 0; s < S; ++s, ++gstep) {
      auto t0 = clock::now();
      StepBatch borrowed;
      const StepBatch* cur = &batch;
      if (pf) {
        borrowed = pf->next();
        cur = &borrowed;
      } else {
        build_step_batch(rc, ds, tcfg.batch, group_seed, gstep, batch);
      }
      const auto cnt = cur->counters();
      report.sampled_nnz_extracted += cnt[0];
      report.sampled_nnz_kept += cnt[1];
      row.t_sample_ms += ms_since(t0);
      t0 = clock::now();
      const double loss = train_step(rc, st, *cur, tcfg.precision, tcfg.seed, gstep, tcfg.rmsnorm_eps);
      row.t_fwd_ms += ms_since(t0);
      report.step_losses.push_back(loss);
      loss_sum += loss;
      t0 = clock::now();
      dp_sync(rc, st);
      rc.synchronize();
      row.t_dpsync_ms += ms_since(t0);
      optimizer_step(rc, st, tcfg.optimizer, tcfg.lr);
    }
    row.epoch = epoch + 1;
    row.step = static_cast<std::int64_t>(gstep);
    row.loss = loss_sum / static_cast<double>(S);
    if (tcfg.evaluate) {
      const EvalCounts c = evaluate_full_graph(rc, st, eval_batch, ds, tcfg.precision, tcfg.rmsnorm_eps);
      row.train_acc = c.accuracy(SplitTag::kTrain);
      row.val_acc = c.accuracy(SplitTag::kVal);
      row.test_acc = c.accuracy(SplitTag::kTest);
    }
    const CommStats snap = rc.snapshot();
    row.bytes_x = snap.bytes_on(Axis::X) - prev_snapshot.bytes_on(Axis::X);
    row.bytes_y = snap.bytes_on(Axis::Y) - prev_snapshot.bytes_on(Axis::Y);
    row.bytes_z = snap.bytes_on(Axis::Z) - prev_snapshot.bytes_on(Axis::Z);
    row.bytes_d = snap.bytes_on(Axis::D) - prev_snapshot.bytes_on(Axis::D);
    prev_snapshot = snap;
    report.epochs.push_back(row);
  }
  rc.synchronize();
  report.comm_total = prev_snapshot - run_start_stats;
  report.wall_ms = ms_since(run_start);
  return report;
}

/// Every rank of `grid` as a host thread driving its own GPU (rank r on
/// device r mod #devices), NCCL between the threads' contexts — the
/// reference's Communicator runs its ranks on threads of one process too.
/// body(rc) runs per rank; the first exception of any rank is rethrown after
/// every thread joined.
inline void run_ranks(const DeviceGrid& grid, const std::function<void(RankComm&)>& body) {
  std::int32_t ndev = 0;
  detail::check(ggb_device_count(&ndev));
  const int world = grid.total();
  if (ndev < 1) throw std::runtime_error("no CUDA device");
  if (world > ndev)
    throw std::invalid_argument("grid of " + std::to_string(world) + " ranks on " + std::to_string(ndev) +
                                " GPU(s): one rank per GPU");
  std::vector<std::uint8_t> uid;
  if (world > 1) uid = RankComm::unique_id();
  std::mutex m;
  std::exception_ptr err;
  std::vector<std::thread> threads;
  for (int r = 0; r < world; ++r)
    threads.emplace_back([&, r] {
      try {
        RankComm rc(grid, r, r % ndev, world > 1 ? uid.data() : nullptr);
        body(rc);
      } catch (...) {
        std::lock_guard<std::mutex> lk(m);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& t : threads) t.join();
  if (err) std::rethrow_exception(err);
}

/// train_run_fp32 (model.hpp:544-545, src/model.cpp:5-8): the whole grid of
/// tcfg.grid trained on `ds`; rank 0's report (the reference returns the
/// report of its rank 0 thread too).
inline TrainReport train_run_fp32(const Dataset& ds, const ModelConfig& mcfg, const TrainConfig& tcfg) {
  TrainReport out;
  std::mutex m;
  run_ranks(tcfg.grid, [&](RankComm& rc) {
    DeviceDataset dds(rc, ds, mcfg.layers);
    TrainReport rep = train_run(rc, dds, mcfg, tcfg);
    if (rc.rank() == 0) {
      std::lock_guard<std::mutex> lk(m);
      out = std::move(rep);
    }
  });
  return out;
}

/// reference_train (model.hpp:549-552): the same run on the degenerate
/// grid with the same DP replica count, fp32 sums.
inline TrainReport reference_train(const Dataset& ds, const ModelConfig& mcfg, TrainConfig tcfg) {
  tcfg.grid = DeviceGrid(tcfg.grid.dims[0], 1, 1, 1);
  tcfg.precision = Precision::kFp32;
  return train_run_fp32(ds, mcfg, tcfg);
}

}  // namespace gridgnn
