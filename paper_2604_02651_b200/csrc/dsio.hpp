// Dataset files (dsio.cpp): the reference's edge list and SGNF/SGNL/SGNS
// formats (dataset.cpp:152-280).
#pragma once

#include <string>
#include <vector>

#include "dataset.hpp"

namespace ggb {

/// load_edge_list (dataset.cpp:152-176): flat (u, v) pairs; *n_out = max id + 1.
std::vector<int64_t> read_edge_list(const std::string& path, int64_t* n_out);
/// load_dataset (dataset.cpp:178-239); the raw edge list is returned in *uv_out if given.
HostDataset load_dataset(const std::string& graph_path, const std::string& feature_path,
                         const std::string& label_path, const std::string& split_path, std::vector<int64_t>* uv_out);
void save_edge_list(const std::string& path, const int64_t* uv, int64_t m);
void save_features(const std::string& path, int64_t n, int64_t d_in, const float* features);
void save_labels(const std::string& path, int64_t n, int64_t n_classes, const int32_t* labels);
void save_split(const std::string& path, int64_t n, const uint8_t* split);

}  // namespace ggb
