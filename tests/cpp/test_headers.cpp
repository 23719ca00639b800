// Every reference header name resolves against the drop-in
// (paper_2604_02651_b200/cpp/gridgnn) and the reference's top-level entry
// points keep their signatures: a translation unit written against
// proj/include/gridgnn compiles and links unchanged for these calls.
#include <cstdio>
#include <type_traits>

#include "gridgnn/comm.hpp"
#include "gridgnn/csr.hpp"
#include "gridgnn/dataset.hpp"
#include "gridgnn/grid.hpp"
#include "gridgnn/metrics.hpp"
#include "gridgnn/model.hpp"
#include "gridgnn/pmm.hpp"
#include "gridgnn/sampling.hpp"
#include "gridgnn/shardsample.hpp"
#include "gridgnn/tensor.hpp"

namespace gg = gridgnn;

// model.hpp:544-552
static_assert(std::is_same_v<decltype(&gg::train_run_fp32),
                             gg::TrainReport (*)(const gg::Dataset&, const gg::ModelConfig&, const gg::TrainConfig&)>);
static_assert(std::is_same_v<decltype(&gg::reference_train),
                             gg::TrainReport (*)(const gg::Dataset&, const gg::ModelConfig&, gg::TrainConfig)>);
// metrics.cpp:10-32, model.hpp:539-542, shardsample.cpp:8-17
static_assert(std::is_same_v<decltype(&gg::write_metrics_csv), void (*)(const std::string&, const gg::TrainReport&)>);
static_assert(std::is_same_v<decltype(&gg::steps_per_epoch), gg::index_t (*)(gg::index_t, gg::index_t, int)>);

int main(int argc, char**) {
  if (argc > 1) {  // the calls themselves (run only with a GPU)
    gg::Dataset ds = gg::generate_synthetic(256, 8.0, 16, 4, 7);
    gg::ModelConfig m;
    m.d_in = ds.d_in();
    m.d_out = ds.n_classes();
    gg::TrainConfig t;
    t.batch = 64;
    t.epochs = 2;
    t.seed = 1;
    const gg::TrainReport r = gg::train_run_fp32(ds, m, t);
    const gg::TrainReport o = gg::reference_train(ds, m, t);
    std::printf("%zu %zu %.6f %.6f\n", r.epochs.size(), o.epochs.size(), r.step_losses.back(), o.step_losses.back());
    return r.step_losses == o.step_losses ? 0 : 1;
  }
  std::printf("headers ok\n");
  return 0;
}
