// Device-built synthetic dataset (gendata.cu): the reference's
// generate_synthetic (dataset.cpp:85-131) on the GPU.
#pragma once

#include "runtime.hpp"

namespace ggb {

/// Dataset (dataset.hpp:16-29) resident in HBM: the normalized adjacency as a
/// column-sorted CSR (int64 row_ptr, int32 col, fp64 val), fp32 features
/// [n][d_in], int32 labels, uint8 split tags.
struct DevDataset {
  int64_t n = 0, d_in = 0, n_classes = 0, nnz = 0;
  DevBuf row_ptr, col, val, features, labels, split;
  // value-free CSR: no fp64 value array; the row degrees (self-loop included)
  // give every value as 1 / sqrt(deg_u deg_v) (dataset.cpp:78-79), exactly
  bool value_free = false;
  DevBuf degree;  // int32 [n]
};

void generate_synthetic_device(Ctx& ctx, int64_t n, double avg_degree, int64_t d_in, int64_t n_classes,
                               uint64_t seed, DevDataset& ds);
/// R-MAT edge list (Graph500 quadrant probabilities a, b, c; 2^scale
/// vertices, m draws) into uv_dev [2m] int64 (gendata.cu k_rmat).
void rmat_edges_device(Ctx& ctx, int scale, int64_t m, double a, double b, double c, uint64_t seed, int64_t* uv_dev);
/// make_csr_shard (shardsample.cpp:19-45) of the device CSR.
void build_shard_device(Ctx& ctx, int64_t n, const DevDataset& ds, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                        PlaneShard& sh);

}  // namespace ggb
