// gridgnn: the reference CLI's train / verify / sample-stats / gen commands
// (proj/tools/gridgnn_main.cpp: same subcommands, options, config-file form
// and report lines) over the B200 library through the C++ drop-in header.
//
// The reference multiplexes every rank of the grid onto host threads of one
// process; here every rank is a host thread driving its own GPU (rank r on
// device r mod #devices), with NCCL communicators created from one in-process
// unique id. One-process grids keep every collective on NCCL (CUDA IPC peer
// memory needs one process per GPU: bench.py / torchrun).
//
// Options: --key value or --key=value; flags --prefetch / --no-prefetch,
// --rmsnorm / --no-rmsnorm, --residual / --no-residual; --config FILE holds
// `key = value` lines (flag names without dashes), overridden by the
// command line.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <fstream>
#include <functional>
#include <map>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "gridgnn/dataset.hpp"
#include "gridgnn/metrics.hpp"
#include "gridgnn/model.hpp"
#include "gridgnn/pmm.hpp"
#include "gridgnn/sampling.hpp"

namespace gg = gridgnn;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// RunConfig of the reference CLI: the same fields and defaults.
struct RunConfig {
  std::string grid = "1x1x1x1";
  std::int64_t batch_size = 0;  // 0: n/4, floored at 2
  int epochs = 10;
  std::uint64_t seed = 1;
  std::string precision = "fp32";
  bool prefetch = false;
  std::string out;
  int layers = 2;
  std::int64_t d_h = 64;
  double dropout = 0.1;
  bool rmsnorm = true, residual = true;
  double lr = 1e-3;
  std::string optimizer = "adam";
  std::string edges, features, labels, split;
  std::int64_t n = 256;
  double avg_degree = 8.0;
  std::int64_t d_in = 128, classes = 32;
  std::uint64_t data_seed = 7;
  std::int64_t draws = 100000;
  double perturb = 0.0;
};

std::string trim(const std::string& s) {
  const auto a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return "";
  return s.substr(a, s.find_last_not_of(" \t\r\n") - a + 1);
}

bool parse_bool(const std::string& v, const std::string& key) {
  if (v == "true" || v == "1" || v == "yes" || v == "on") return true;
  if (v == "false" || v == "0" || v == "no" || v == "off") return false;
  throw UsageError("--" + key + ": expected a boolean, got '" + v + "'");
}

// One option: key (without dashes) and value text; flags arrive as "true"/"false".
void set_option(RunConfig& rc, const std::string& cmd, const std::string& key, const std::string& v) {
  auto num = [&](auto& dst, bool positive, bool nonneg) {
    std::istringstream is(v);
    std::remove_reference_t<decltype(dst)> x{};
    if (!(is >> x) || !is.eof()) throw UsageError("--" + key + ": not a number: '" + v + "'");
    if ((positive && !(x > 0)) || (nonneg && x < 0)) throw UsageError("--" + key + ": out of range: " + v);
    dst = x;
  };
  auto file = [&](std::string& dst) {
    if (!std::ifstream(v).good()) throw UsageError("--" + key + ": File does not exist: " + v);
    dst = v;
  };
  if (key == "grid") rc.grid = v;
  else if (key == "batch-size") num(rc.batch_size, false, true);
  else if (key == "epochs") num(rc.epochs, true, false);
  else if (key == "seed") num(rc.seed, false, false);
  else if (key == "precision") rc.precision = v;
  else if (key == "prefetch") rc.prefetch = parse_bool(v, key);
  else if (key == "out") rc.out = v;
  else if (key == "layers") num(rc.layers, true, false);
  else if (key == "hidden-dim") num(rc.d_h, true, false);
  else if (key == "dropout") {
    num(rc.dropout, false, true);
    if (rc.dropout >= 1.0) throw UsageError("--dropout: must be in [0, 1)");
  } else if (key == "rmsnorm") rc.rmsnorm = parse_bool(v, key);
  else if (key == "residual") rc.residual = parse_bool(v, key);
  else if (key == "lr") num(rc.lr, true, false);
  else if (key == "optimizer") {
    if (v != "adam" && v != "sgd") throw UsageError("--optimizer: expected adam or sgd: " + v);
    rc.optimizer = v;
  } else if (key == "edges") file(rc.edges);
  else if (key == "features") file(rc.features);
  else if (key == "labels") file(rc.labels);
  else if (key == "split") file(rc.split);
  else if (key == "n") num(rc.n, true, false);
  else if (key == "avg-degree") num(rc.avg_degree, false, true);
  else if (key == "d-in") num(rc.d_in, true, false);
  else if (key == "classes") num(rc.classes, true, false);
  else if (key == "data-seed") num(rc.data_seed, false, false);
  else if (key == "draws" && cmd == "sample-stats") num(rc.draws, true, false);
  else if (key == "perturb" && cmd == "verify") num(rc.perturb, false, false);
  else throw UsageError("The following argument was not expected: --" + key);
}

const char* kFlags[] = {"prefetch", "rmsnorm", "residual"};

RunConfig parse_args(const std::string& cmd, int argc, char** argv) {
  RunConfig rc;
  std::vector<std::pair<std::string, std::string>> opts;
  std::string config;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + a);
    a = a.substr(2);
    std::string key = a, val;
    const auto eq = a.find('=');
    if (eq != std::string::npos) {
      key = a.substr(0, eq);
      val = a.substr(eq + 1);
    } else {
      bool flag = false;
      for (const char* f : kFlags) {
        if (key == f) opts.emplace_back(key, "true"), flag = true;
        else if (key == std::string("no-") + f) opts.emplace_back(f, "false"), flag = true;
      }
      if (flag) continue;
      if (i + 1 >= argc) throw UsageError("--" + key + " requires an argument");
      val = argv[++i];
    }
    if (key == "config") config = val;
    else opts.emplace_back(key, val);
  }
  if (!config.empty()) {  // file values first, the command line overrides them
    std::ifstream in(config);
    if (!in) throw UsageError("--config: cannot open " + config);
    std::string line;
    while (std::getline(in, line)) {
      line = trim(line.substr(0, line.find('#')));
      if (line.empty() || line[0] == '[') continue;
      const auto eq = line.find('=');
      if (eq == std::string::npos) throw UsageError("--config: expected key = value: " + line);
      set_option(rc, cmd, trim(line.substr(0, eq)), trim(line.substr(eq + 1)));
    }
  }
  for (const auto& [k, v] : opts) set_option(rc, cmd, k, v);
  return rc;
}

gg::DeviceGrid parse_grid(const std::string& s) {
  int d[4];
  char extra;
  if (std::sscanf(s.c_str(), "%dx%dx%dx%d%c", &d[0], &d[1], &d[2], &d[3], &extra) != 4)
    throw UsageError("--grid: expected GdxGxxGyxGz, e.g. 2x2x2x1: " + s);
  for (int x : d)
    if (x < 1) throw UsageError("--grid: grid dims must be >= 1: " + s);
  return gg::DeviceGrid(d[0], d[1], d[2], d[3]);
}

gg::Precision parse_precision(const std::string& s) {
  if (s == "fp32") return gg::Precision::kFp32;
  if (s == "bf16comm") return gg::Precision::kBf16Roundtrip;
  throw UsageError("--precision: expected fp32 or bf16comm: " + s);
}

gg::Dataset load_or_generate(const RunConfig& rc) {
  if (!rc.edges.empty()) return gg::load_dataset(rc.edges, rc.features, rc.labels, rc.split);
  return gg::generate_synthetic(rc.n, rc.avg_degree, rc.d_in, rc.classes, rc.data_seed);
}

gg::index_t effective_batch(const RunConfig& rc, gg::index_t n) {
  gg::index_t b = rc.batch_size;
  if (b == 0) b = n / 4;
  return std::min<gg::index_t>(std::max<gg::index_t>(b, 2), n);
}

gg::ModelConfig model_config(const RunConfig& rc, const gg::Dataset& ds) {
  gg::ModelConfig m;
  m.layers = rc.layers;
  m.d_in = ds.d_in();
  m.d_h = rc.d_h;
  m.d_out = ds.n_classes();
  m.dropout_rate = rc.dropout;
  m.use_dropout = rc.dropout > 0.0;
  m.use_rmsnorm = rc.rmsnorm;
  m.use_residual = rc.residual;
  return m;
}

gg::TrainConfig train_config(const RunConfig& rc, gg::index_t n) {
  gg::TrainConfig t;
  t.grid = parse_grid(rc.grid);
  t.batch = effective_batch(rc, n);
  t.epochs = rc.epochs;
  t.seed = rc.seed;
  t.precision = parse_precision(rc.precision);
  t.prefetch = rc.prefetch;
  t.optimizer = rc.optimizer == "sgd" ? gg::Optimizer::kSgd : gg::Optimizer::kAdam;
  t.lr = rc.lr;
  return t;
}

// train_run on every rank of the grid; rank 0's report. make: the rank's
// DeviceDataset (make_rank_context of the run's dataset).
gg::TrainReport train_on_grid(const gg::ModelConfig& mcfg, const gg::TrainConfig& tcfg,
                              const std::function<gg::DeviceDataset(gg::RankComm&)>& make) {
  gg::TrainReport out;
  std::mutex m;
  gg::run_ranks(tcfg.grid, [&](gg::RankComm& rc) {
    gg::DeviceDataset dds = make(rc);
    gg::TrainReport rep = gg::train_run(rc, dds, mcfg, tcfg);
    if (rc.rank() == 0) {
      std::lock_guard<std::mutex> lk(m);
      out = std::move(rep);
    }
  });
  return out;
}


int cmd_train(const RunConfig& rc) {
  const gg::Dataset ds = load_or_generate(rc);
  const gg::ModelConfig mcfg = model_config(rc, ds);
  const gg::TrainConfig tcfg = train_config(rc, ds.n());
  const gg::TrainReport rep = gg::train_run_fp32(ds, mcfg, tcfg);
  const std::string out = rc.out.empty() ? "metrics.csv" : rc.out;
  gg::write_metrics_csv(out, rep);
  std::printf("wrote %s (%zu epochs)\n", out.c_str(), rep.epochs.size());
  std::printf("final: train_acc=%.4f val_acc=%.4f test_acc=%.4f loss=%.6f\n", rep.final_train_acc(),
              rep.final_val_acc(), rep.final_test_acc(), rep.epochs.empty() ? 0.0 : rep.epochs.back().loss);
  const auto& t = rep.comm_total;
  std::printf("comm bytes: x=%llu y=%llu z=%llu d=%llu  wall=%.1f ms\n",
              static_cast<unsigned long long>(t.bytes_on(gg::Axis::X)),
              static_cast<unsigned long long>(t.bytes_on(gg::Axis::Y)),
              static_cast<unsigned long long>(t.bytes_on(gg::Axis::Z)),
              static_cast<unsigned long long>(t.bytes_on(gg::Axis::D)), rep.wall_ms);
  return 0;
}

// The device-path counterpart of the reference's fp64 finite-difference
// check: directional derivatives (L(W + hD) - L(W - hD)) / 2h of the device
// forward against <g, D> of the device backward, D = the gradient direction
// plus a random one (tests/test_gpu_finite_diff.py states the same check).
double directional_gradient_check(gg::RankComm& rc, const gg::DeviceDataset& dds, const gg::ModelConfig& mcfg,
                                  gg::index_t b, std::uint64_t seed) {
  gg::ModelState st(rc, mcfg, seed);
  gg::StepBatch batch = gg::build_step_batch(rc, dds, b, seed, 0);
  gg::train_step(rc, st, batch, gg::Precision::kFp32, seed, 0);
  const int np = st.num_params();
  std::vector<std::vector<float>> w0(np), g(np);
  for (int i = 0; i < np; ++i) {
    w0[i] = st.param(i, 0);
    g[i] = st.param(i, 1);
  }
  auto loss_at = [&](const std::vector<std::vector<double>>& d, double h) {
    for (int i = 0; i < np; ++i) {
      std::vector<float> w(w0[i]);
      for (size_t k = 0; k < w.size(); ++k) w[k] += static_cast<float>(h * d[i][k]);
      gg::detail::check(ggb_state_param_set(st.handle(), i, 0, w.data()));
    }
    gg::detail::check(ggb_forward(rc.handle(), st.handle(), batch.handle(), GGB_FP32, 1, seed, 0, 1e-6));
    float l = 0.f;
    gg::detail::check(ggb_loss(rc.handle(), st.handle(), batch.handle(), &l));
    return static_cast<double>(l);
  };
  std::mt19937_64 gen(seed);
  std::normal_distribution<double> nd;
  double gn = 0.0, worst = 0.0;
  for (const auto& v : g)
    for (float x : v) gn += static_cast<double>(x) * x;
  gn = std::sqrt(gn);
  for (int draw = 0; draw < 3; ++draw) {
    std::vector<std::vector<double>> d(np);
    double rn = 0.0;
    for (int i = 0; i < np; ++i) {
      d[i].resize(g[i].size());
      for (double& x : d[i]) x = nd(gen), rn += x * x;
    }
    rn = std::sqrt(rn);
    double dn = 0.0, want = 0.0;
    for (int i = 0; i < np; ++i)
      for (size_t k = 0; k < d[i].size(); ++k) {
        d[i][k] = g[i][k] / gn + d[i][k] / rn;
        dn += d[i][k] * d[i][k];
      }
    dn = std::sqrt(dn);
    for (int i = 0; i < np; ++i)
      for (size_t k = 0; k < d[i].size(); ++k) {
        d[i][k] /= dn;
        want += static_cast<double>(g[i][k]) * d[i][k];
      }
    double best = 1e300;
    for (double h : {3e-2, 1e-2, 3e-3}) {
      const double fd = (loss_at(d, h) - loss_at(d, -h)) / (2 * h);
      best = std::min(best, std::abs(fd - want) / std::max(std::abs(want), 1e-8));
    }
    worst = std::max(worst, best);
  }
  for (int i = 0; i < np; ++i) gg::detail::check(ggb_state_param_set(st.handle(), i, 0, w0[i].data()));
  return worst;
}

int cmd_verify(const RunConfig& rc) {
  int failures = 0;
  auto report = [&](const char* name, bool ok, const std::string& detail) {
    std::printf("%-34s %s%s%s\n", name, ok ? "PASS" : "FAIL", detail.empty() ? "" : "  ", detail.c_str());
    if (!ok) ++failures;
  };
  {  // rotation schedule: adjacency planes cycle ZX, YZ, XY (pmm.hpp:31-38)
    bool ok = true;
    const gg::Plane want[] = {gg::Plane::ZX, gg::Plane::YZ, gg::Plane::XY};
    for (int l = 1; l <= 9; ++l) ok = ok && gg::plane_of(gg::adjacency_layout(l)) == want[(l - 1) % 3];
    report("rotation schedule", ok, "");
  }
  {  // sharded vs serial trainer on the same batches (DP replicas kept)
    RunConfig small = rc;
    small.n = 48;
    small.classes = 4;
    small.d_in = 12;
    small.d_h = 8;
    small.epochs = 3;
    small.dropout = 0.0;
    gg::Dataset ds = load_or_generate(small);
    const gg::ModelConfig mcfg = model_config(small, ds);
    gg::TrainConfig tcfg = train_config(small, ds.n());
    gg::TrainConfig tref = tcfg;
    tref.grid = gg::DeviceGrid(tcfg.grid.dims[0], 1, 1, 1);
    tref.precision = gg::Precision::kFp32;
    const gg::TrainReport ref = gg::train_run_fp32(ds, mcfg, tref);
    // the run under test, optionally with one input feature offset (the
    // reference's check-failure hook)
    gg::Dataset ds_run = load_or_generate(small);
    std::vector<std::int64_t> rp(static_cast<size_t>(ds_run.n() + 1)), ci(static_cast<size_t>(ds_run.nnz()));
    std::vector<double> val(ci.size());
    std::vector<float> f(static_cast<size_t>(ds_run.n() * ds_run.d_in()));
    std::vector<std::int32_t> lab(static_cast<size_t>(ds_run.n()));
    std::vector<std::uint8_t> sp(static_cast<size_t>(ds_run.n()));
    gg::detail::check(ggb_dataset_export(ds_run.handle(), rp.data(), ci.data(), val.data(), f.data(), lab.data(),
                                         sp.data(), nullptr));
    f[0] += static_cast<float>(rc.perturb);
    gg::CsrMatrix a;
    a.n_rows = a.n_cols = ds_run.n();
    a.row_ptr = rp;
    a.col_idx = ci;
    a.values = val;
    std::vector<gg::SplitTag> split(sp.size());
    for (size_t i = 0; i < sp.size(); ++i) split[i] = static_cast<gg::SplitTag>(sp[i]);
    const gg::TrainReport got = train_on_grid(mcfg, tcfg, [&](gg::RankComm& r) {
      return gg::DeviceDataset(r, a, ds_run.d_in(), f, ds_run.n_classes(), lab, mcfg.layers, true, &split);
    });
    double max_diff = 0.0;
    bool ok = got.step_losses.size() == ref.step_losses.size();
    for (size_t i = 0; ok && i < ref.step_losses.size(); ++i)
      max_diff = std::max(max_diff, std::abs(got.step_losses[i] - ref.step_losses[i]) /
                                        std::max(std::abs(ref.step_losses[i]), 1e-12));
    // the reference compares its fp32 CPU runs at 1e-4 absolute; the device
    // path's bar is the north star's loss tolerance, 1e-3 relative
    ok = ok && max_diff < 1e-3;
    char buf[128];
    std::snprintf(buf, sizeof buf, "grid %s, max step-loss rel diff %.3g", small.grid.c_str(), max_diff);
    report("sharded vs serial trainer", ok, buf);
  }
  {  // gradient check: directional derivatives of the device forward vs its backward
    RunConfig small = rc;
    small.n = 400;
    small.classes = 3;
    small.d_in = 6;
    small.d_h = 8;
    gg::Dataset ds = load_or_generate(small);
    gg::ModelConfig mcfg = model_config(small, ds);
    mcfg.use_dropout = false;
    mcfg.dropout_rate = 0.0;
    double worst = 0.0;
    gg::run_ranks(gg::DeviceGrid(1, 1, 1, 1), [&](gg::RankComm& r) {
      gg::DeviceDataset dds(r, ds, mcfg.layers);
      worst = directional_gradient_check(r, dds, mcfg, ds.n() / 2, rc.seed);
    });
    char buf[96];
    std::snprintf(buf, sizeof buf, "max relative error %.3g (fp32 device path, bar 1e-2)", worst);
    report("gradient check (directional)", worst < 1e-2, buf);
  }
  if (failures) std::printf("%d check(s) failed\n", failures);
  return failures ? 1 : 0;
}

// Inclusion frequency and aggregation bias of the sampler + induced-subgraph
// rescaling over many draws (the reference's sample-stats), with batches
// built by the device pipeline on one GPU.
int cmd_sample_stats(const RunConfig& rc) {
  const gg::Dataset ds = load_or_generate(rc);
  const gg::index_t n = ds.n();
  const gg::index_t b = effective_batch(rc, n);
  const auto draws = static_cast<std::uint64_t>(rc.draws);
  std::vector<std::int64_t> rp(static_cast<size_t>(n + 1)), ci(static_cast<size_t>(ds.nnz()));
  std::vector<double> val(ci.size());
  gg::detail::check(ggb_dataset_export(ds.handle(), rp.data(), ci.data(), val.data(), nullptr, nullptr, nullptr,
                                       nullptr));
  // unit signal: the aggregation is the rescaled adjacency row sum
  std::vector<double> full(static_cast<size_t>(n), 0.0);
  for (gg::index_t r = 0; r < n; ++r)
    for (std::int64_t e = rp[r]; e < rp[r + 1]; ++e) full[static_cast<size_t>(r)] += val[static_cast<size_t>(e)];
  std::vector<std::uint64_t> included(static_cast<size_t>(n), 0);
  std::vector<double> agg(static_cast<size_t>(n), 0.0);
  gg::run_ranks(gg::DeviceGrid(1, 1, 1, 1), [&](gg::RankComm& r) {
    gg::DeviceDataset dds(r, ds, 1);
    gg::StepBatch batch;
    for (std::uint64_t d = 0; d < draws; ++d) {
      gg::build_step_batch(r, dds, b, rc.seed, d, batch);
      const gg::SampleSet s = batch.sample();
      const gg::CsrMatrix a = batch.plane(0, false);
      for (gg::index_t i = 0; i < b; ++i) {
        const auto v = static_cast<size_t>(s.vertices[static_cast<size_t>(i)]);
        ++included[v];
        double h = 0.0;
        for (auto e = a.row_ptr[static_cast<size_t>(i)]; e < a.row_ptr[static_cast<size_t>(i) + 1]; ++e)
          h += a.values[static_cast<size_t>(e)];
        agg[v] += h;
      }
    }
  });
  const double p = static_cast<double>(b) / static_cast<double>(n);
  double max_freq_dev = 0.0, max_bias = 0.0;
  for (gg::index_t v = 0; v < n; ++v) {
    const auto vi = static_cast<size_t>(v);
    const double freq = static_cast<double>(included[vi]) / static_cast<double>(draws);
    max_freq_dev = std::max(max_freq_dev, std::abs(freq - p) / p);
    if (included[vi] == 0) continue;
    const double mean = agg[vi] / static_cast<double>(included[vi]);
    max_bias = std::max(max_bias, std::abs(mean - full[vi]) / std::max(std::abs(full[vi]), 1e-12));
  }
  std::printf("n=%lld B=%lld draws=%llu\n", static_cast<long long>(n), static_cast<long long>(b),
              static_cast<unsigned long long>(draws));
  std::printf("inclusion frequency: target %.6f, max relative deviation %.4g\n", p, max_freq_dev);
  std::printf("aggregation bias: max relative deviation of conditional mean %.4g%s\n", max_bias,
              b == n ? " (B=N: every batch is the full graph)" : "");
  return 0;
}

int cmd_gen(const RunConfig& rc) {
  const gg::Dataset ds = gg::generate_synthetic(rc.n, rc.avg_degree, rc.d_in, rc.classes, rc.data_seed);
  const std::string prefix = rc.out.empty() ? "synthetic" : rc.out;
  ds.save(prefix + ".edges", prefix + ".sgnf", prefix + ".sgnl", prefix + ".sgns");
  std::printf("wrote %s.{edges,sgnf,sgnl,sgns}: n=%lld d_in=%lld classes=%lld\n", prefix.c_str(),
              static_cast<long long>(ds.n()), static_cast<long long>(ds.d_in()),
              static_cast<long long>(ds.n_classes()));
  return 0;
}

void usage() {
  std::fprintf(stderr,
               "Deterministic multi-axis-parallel GCN training on B200\n"
               "Usage: gridgnn SUBCOMMAND [OPTIONS]\n"
               "Subcommands:\n"
               "  train         Train a model and write a metrics CSV\n"
               "  verify        Run oracle and gradient checks\n"
               "  sample-stats  Report sampling frequency and aggregation bias\n"
               "  gen           Write a synthetic dataset to disk\n");
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2 || std::string(argv[1]) == "--help" || std::string(argv[1]) == "-h") {
    usage();
    return argc < 2 ? 106 : 0;
  }
  const std::string cmd = argv[1];
  if (cmd != "train" && cmd != "verify" && cmd != "sample-stats" && cmd != "gen") {
    usage();
    std::fprintf(stderr, "The following argument was not expected: %s\n", cmd.c_str());
    return 109;
  }
  try {
    const RunConfig rc = parse_args(cmd, argc, argv);
    if (cmd == "train") return cmd_train(rc);
    if (cmd == "verify") return cmd_verify(rc);
    if (cmd == "sample-stats") return cmd_sample_stats(rc);
    return cmd_gen(rc);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
    return 105;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
