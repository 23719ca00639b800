// gridgnn/shardsample.hpp drop-in (reference: include/gridgnn/shardsample.hpp:14-119):
// the index vocabulary of the communication-free sampler (Alg. 2).
//
// On the B200 the per-shard phases — extract_rows, filter_and_remap,
// assemble_shard and the RemapTable lookups (shardsample.cpp:58-122) — are
// fused into the device batch build (ggb_build_step_batch: warp-per-row
// extraction with bitmap membership and a popcount rank table instead of the
// step-tagged table; exact same CSR blocks), so they have no separate entry
// points. What callers use to interpret batches — the partition offsets and
// the positions of a range inside the sorted sample — is here; make_csr_shard
// prepares a static shard on the host (the input side of ggb_graph_create).
#pragma once

#include <algorithm>

#include "ggb.hpp"

namespace gridgnn {

/// rows [r0, r1) with local row ids, column ids kept GLOBAL within [c0, c1) (shardsample.hpp:18-25)
struct CsrShard {
  index_t r0 = 0, r1 = 0, c0 = 0, c1 = 0;
  CsrMatrix local;
};

inline CsrShard make_csr_shard(const CsrMatrix& a, index_t r0, index_t r1, index_t c0, index_t c1) {
  if (r0 < 0 || r1 < r0 || r1 > a.n_rows || c0 < 0 || c1 < c0 || c1 > a.n_cols)
    throw std::invalid_argument("make_csr_shard: range out of bounds");
  CsrShard s{r0, r1, c0, c1, {}};
  s.local.n_rows = r1 - r0;
  s.local.n_cols = a.n_cols;
  s.local.row_ptr.assign(1, 0);
  for (index_t r = r0; r < r1; ++r) {
    const auto b = a.col_idx.begin() + a.row_ptr[static_cast<std::size_t>(r)];
    const auto e = a.col_idx.begin() + a.row_ptr[static_cast<std::size_t>(r) + 1];
    const auto lo = std::lower_bound(b, e, c0), hi = std::lower_bound(lo, e, c1);  // columns are sorted
    s.local.col_idx.insert(s.local.col_idx.end(), lo, hi);
    const auto v0 = a.values.begin() + (lo - a.col_idx.begin());
    s.local.values.insert(s.local.values.end(), v0, v0 + (hi - lo));
    s.local.row_ptr.push_back(static_cast<index_t>(s.local.col_idx.size()));
  }
  return s;
}

/// S_r = sample[row_lo, row_hi), S_c = sample[col_lo, col_hi) (shardsample.hpp:59-65)
struct LocalRanges {
  index_t row_lo = 0, row_hi = 0;
  index_t col_lo = 0, col_hi = 0;
};

inline LocalRanges locate_ranges(const SampleSet& s, index_t r0, index_t r1, index_t c0, index_t c1) {
  const auto b = s.vertices.begin(), e = s.vertices.end();
  auto pos = [&](index_t v) { return static_cast<index_t>(std::lower_bound(b, e, v) - b); };
  return {pos(r0), pos(r1), pos(c0), pos(c1)};
}

/// positions of the partition offsets inside the sorted sample (shardsample.hpp:118-119)
inline std::vector<index_t> sample_partition(const SampleSet& s, const std::vector<index_t>& offsets) {
  std::vector<index_t> out;
  out.reserve(offsets.size());
  for (index_t o : offsets)
    out.push_back(static_cast<index_t>(std::lower_bound(s.vertices.begin(), s.vertices.end(), o) - s.vertices.begin()));
  return out;
}

}  // namespace gridgnn
