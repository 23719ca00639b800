// Host dataset (Dataset, dataset.hpp:16-29) as built natively by dataset.cpp.
#pragma once

#include <cstdint>
#include <vector>

#include "common.hpp"

namespace ggb {

struct HostCsr {
  int64_t n = 0;
  std::vector<int64_t> row_ptr, col;
  std::vector<double> val;
};

struct HostDataset {
  int64_t n = 0, d_in = 0, n_classes = 0;
  HostCsr adj;
  std::vector<float> features;
  std::vector<int32_t> labels;
  std::vector<uint8_t> split;
};

std::vector<int64_t> synthetic_edges(int64_t n, double avg_degree, uint64_t seed);
HostCsr normalize_adjacency(const int64_t* uv, int64_t m, int64_t n);
void synthetic_features(int64_t n, int64_t d_in, uint64_t seed, float* out);
void degree_labels(int64_t n, const int64_t* row_ptr, int64_t n_classes, int32_t* labels);
void split_tags(int64_t n, uint64_t seed, uint8_t* split);
HostDataset generate_synthetic(int64_t n, double avg_degree, int64_t d_in, int64_t n_classes,
                               uint64_t seed);
/// generate_synthetic with the ER edge stream replaced by the given edge list
/// (normalized adjacency, N(0,1) features, degree-quantile labels, 60/20/20 split)
HostDataset dataset_from_edges(int64_t n, const int64_t* uv, int64_t m, int64_t d_in, int64_t n_classes,
                               uint64_t seed);

}  // namespace ggb
