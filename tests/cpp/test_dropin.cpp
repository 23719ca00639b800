#include <algorithm>
// Acceptance-style checks of the C++ drop-in (paper_2604_02651_b200/cpp/gridgnn/ggb.hpp),
// written like the reference's acceptance.cpp: one PASS/FAIL line per
// check, exit status = number of failures. The reference-side answers come
// from the unmodified reference compiled in place (oracle/_ref, through the
// neutral C shim) — test infrastructure only.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../paper_2604_02651_b200/cpp/gridgnn/ggb.hpp"

extern "C" {  // oracle/ref_shim.cpp
int ref_sample_vertices(std::int64_t n, std::int64_t b, std::uint64_t seed, std::uint64_t step, std::int64_t* out);
void* ref_dataset_synthetic(std::int64_t n, double avg_degree, std::int64_t d_in, std::int64_t n_classes,
                            std::uint64_t seed);
void ref_dataset_free(void*);
void* ref_step_batch(void* ds, const int* dims, int rank, int layers, std::int64_t b, std::uint64_t group_seed,
                     std::uint64_t step);
void ref_batch_free(void*);
void ref_batch_plane(void* p, int plane, int transposed, std::int64_t* dims, std::int64_t* row_ptr, std::int64_t* col,
                     double* val);
int ref_train(void* ds, const int* dims, const std::int64_t* mc, const double* md, std::int64_t b, std::uint64_t seed,
              std::uint64_t step0, int n_steps, int prec, int optimizer, double lr, double eps, float* losses,
              float* logits_out, float* grads_out, float* weights_out);
int ref_train_eval(void* ds, const int* dims, const std::int64_t* mc, const double* md, std::int64_t b,
                   std::uint64_t seed, int n_steps, int prec, int optimizer, double lr, double eps,
                   std::uint64_t* counts, float* eval_logits);
}

using namespace gridgnn;

static int g_fail = 0;
static void report(int idx, const char* name, bool ok, const std::string& detail) {
  std::printf("%2d %-44s %s  %s\n", idx, name, ok ? "PASS" : "FAIL", detail.c_str());
  if (!ok) ++g_fail;
}

int main() {
  RankComm rc(DeviceGrid(1, 1, 1, 1), 0);

  // 1. sample_vertices known answers (test_sampling.cpp:13-26)
  {
    bool ok = sample_vertices(rc, 100, 5, 7, 3).vertices == std::vector<index_t>{7, 35, 43, 44, 54};
    ok = ok && sample_vertices(rc, 5, 5, 123, 0).vertices == std::vector<index_t>{0, 1, 2, 3, 4};
    ok = ok && sample_vertices(rc, 100, 10, 7, 4).vertices == sample_vertices(rc, 100, 10, 11, 0).vertices;
    std::vector<index_t> want(612500);
    ref_sample_vertices(2450000, 612500, 9, 4, want.data());
    ok = ok && sample_vertices(rc, 2450000, 612500, 9, 4).vertices == want;
    bool threw = false;
    try {
      sample_vertices(rc, 10, 11, 0, 0);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    report(1, "sample_vertices == reference", ok && threw, "incl. products-shaped batch, errors");
  }

  // 2. build_step_batch == reference on a 2x2x2 grid (every rank, virtual contexts)
  const index_t n = 20000, b = 5000;
  const int layers = 3;
  void* rds = ref_dataset_synthetic(n, 16.0, 12, 6, 7);
  {
    bool ok = true;
    const int dims[4] = {1, 2, 2, 2};
    for (int rank = 0; rank < 16; ++rank) {
      RankComm vr(DeviceGrid(1, 2, 2, 2), rank % 8);
      // ranks 0-7: native host generator; 8-15: built on the GPU with device shard cuts
      DeviceDataset ds = rank < 8 ? DeviceDataset(vr, n, 16.0, 12, 6, 7, layers)
                                  : DeviceDataset::generate_on_device(vr, n, 16.0, 12, 6, 7, layers);
      StepBatch sb = build_step_batch(vr, ds, b, 11, 3);
      void* rb = ref_step_batch(rds, dims, rank % 8, layers, b, 11, 3);
      for (int p = 0; p < 3; ++p)
        for (int t = 0; t < 2; ++t) {
          index_t d[7];
          ref_batch_plane(rb, p, t, d, nullptr, nullptr, nullptr);
          CsrMatrix want;
          want.n_rows = d[0];
          want.n_cols = d[1];
          want.row_ptr.resize(static_cast<size_t>(d[0] + 1));
          want.col_idx.resize(static_cast<size_t>(d[2]));
          want.values.resize(static_cast<size_t>(d[2]));
          ref_batch_plane(rb, p, t, d, want.row_ptr.data(), want.col_idx.data(), want.values.data());
          ok = ok && sb.plane(p, t != 0) == want;
        }
      ref_batch_free(rb);
    }
    report(2, "shard assembly bit-exact (2x2x2, 8 ranks)", ok,
           "a_loc and a_t_loc, fp64 values; host- and device-built graphs");
  }

  // 3. train_run losses track the reference (1x1x1x1, Adam, 6 steps)
  {
    DeviceDataset ds(rc, n, 16.0, 12, 6, 7, layers);
    ModelConfig mcfg;
    mcfg.layers = layers;
    mcfg.d_in = 12;
    mcfg.d_h = 64;
    mcfg.d_out = 6;
    TrainConfig tcfg;
    tcfg.batch = b;
    tcfg.epochs = 2;
    tcfg.seed = 1;
    const TrainReport rep = train_run(rc, ds, mcfg, tcfg);
    const std::vector<double>& losses = rep.step_losses;
    const std::int64_t mc[7] = {layers, 12, 64, 6, 1, 1, 1};
    const double md[1] = {0.1};
    const int dims[4] = {1, 1, 1, 1};
    std::vector<float> want(losses.size());
    ref_train(rds, dims, mc, md, b, 1, 0, static_cast<int>(losses.size()), 0, 1, 1e-3, 1e-6, want.data(), nullptr,
              nullptr, nullptr);
    double worst = 0.0;
    for (size_t k = 0; k < losses.size(); ++k)
      worst = std::max(worst, std::abs(losses[k] - want[k]) / std::abs(static_cast<double>(want[k])));
    report(3, "train_run losses vs reference (rel <= 1e-3)", worst <= 1e-3, "max rel " + std::to_string(worst));

    // 4. prefetch is transparent (acceptance criterion 8)
    tcfg.prefetch = true;
    const TrainReport pl = train_run(rc, ds, mcfg, tcfg);
    report(4, "prefetch on/off identical losses", pl.step_losses == losses, "");

    // 5. per-epoch evaluate_full_graph tracks the reference's (model.hpp:686-700)
    std::uint64_t counts[6];
    ref_train_eval(rds, dims, mc, md, b, 1, static_cast<int>(losses.size()), 0, 1, 1e-3, 1e-6, counts, nullptr);
    const EpochMetrics& last = rep.epochs.back();
    const double acc[3] = {last.train_acc, last.val_acc, last.test_acc};
    double dev = 0.0;
    for (int s = 0; s < 3; ++s)
      dev = std::max(dev, std::abs(acc[s] - static_cast<double>(counts[s]) / static_cast<double>(counts[3 + s])));
    // metrics.cpp:10-32 format: header + one row per epoch
    const std::string csv = metrics_csv_string(rep);
    const bool csv_ok = csv.rfind("epoch,step,loss,train_acc,val_acc,test_acc,", 0) == 0 &&
                        std::count(csv.begin(), csv.end(), '\n') == 3;
    report(5, "full-graph eval accuracy vs reference", dev <= 5e-3 && rep.epochs.size() == 2 && csv_ok,
           "max |acc diff| " + std::to_string(dev) + ", test acc " + std::to_string(last.test_acc));
  }
  ref_dataset_free(rds);
  return g_fail;
}
