// Native synthetic dataset builder, bit-identical to the reference
// generate_synthetic (src/dataset.cpp:85-150) and normalize_adjacency
// (src/dataset.cpp:47-83), parallelized over host threads:
//  * edges: the reference's sequential Stream, two next_below(n) draws per
//    pair (a counter RNG, so it is a tight loop);
//  * normalization: per-row buckets, per-row sort + dedup on worker threads;
//  * features: Marsaglia polar attempts consume draw pairs (2a, 2a+1), so a
//    parallel count of accepted attempts per chunk followed by a prefix gives
//    every output its exact position in the reference sequence;
//  * labels: a stable counting sort by degree == std::stable_sort by (deg, id).
// This runs once per dataset and is not part of the training step.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "dataset.hpp"
#include "rng.cuh"

namespace ggb {
namespace {

int workers() {
  const unsigned h = std::thread::hardware_concurrency();
  return static_cast<int>(std::max(1u, std::min(h, 64u)));
}

template <class F>
void parallel_for(int64_t n, F&& f) {
  const int T = workers();
  if (n < 4096 || T == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = ceil_div(n, T);
  for (int t = 0; t < T; ++t) {
    const int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& x : th) x.join();
}

struct Stream {
  uint64_t state;
  uint64_t next_u64() { return splitmix64_step(); }
  uint64_t splitmix64_step() {
    state += kGolden;
    uint64_t x = state;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  }
  uint64_t next_below(uint64_t bound) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x;
    do {
      x = next_u64();
    } while (x >= limit);
    return x % bound;
  }
};

}  // namespace

std::vector<int64_t> synthetic_edges(int64_t n, double avg_degree, uint64_t seed) {
  require(n >= 1, "synthetic_edges: n must be >= 1");
  require(avg_degree >= 0, "synthetic_edges: avg_degree must be >= 0");
  Stream s{hash_combine(seed, 0xe0e0)};
  const uint64_t target = static_cast<uint64_t>(avg_degree * static_cast<double>(n) / 2.0);
  std::vector<int64_t> uv;
  uv.reserve(2 * target);
  if (n > 1)
    for (uint64_t e = 0; e < target; ++e) {
      const int64_t u = static_cast<int64_t>(s.next_below(static_cast<uint64_t>(n)));
      const int64_t v = static_cast<int64_t>(s.next_below(static_cast<uint64_t>(n)));
      if (u != v) {
        uv.push_back(u);
        uv.push_back(v);
      }
    }
  return uv;
}

HostCsr normalize_adjacency(const int64_t* uv, int64_t m, int64_t n) {
  require(n > 0, "normalize_adjacency: n must be positive");
  std::vector<int64_t> cnt(static_cast<size_t>(n) + 1, 0);
  for (int64_t e = 0; e < m; ++e) {
    const int64_t u = uv[2 * e], v = uv[2 * e + 1];
    require(u >= 0 && u < n && v >= 0 && v < n, "normalize_adjacency: vertex id out of range");
    if (u == v) continue;
    ++cnt[u + 1];
    ++cnt[v + 1];
  }
  for (int64_t v = 0; v < n; ++v) cnt[v + 1] += 1 + cnt[v];  // + one self-loop per row
  std::vector<int32_t> bucket(static_cast<size_t>(cnt[n]));
  std::vector<int64_t> cur(cnt.begin(), cnt.end() - 1);
  for (int64_t v = 0; v < n; ++v) bucket[cur[v]++] = static_cast<int32_t>(v);
  for (int64_t e = 0; e < m; ++e) {
    const int64_t u = uv[2 * e], v = uv[2 * e + 1];
    if (u == v) continue;
    bucket[cur[u]++] = static_cast<int32_t>(v);
    bucket[cur[v]++] = static_cast<int32_t>(u);
  }
  // sort + dedup each row in place; record the deduplicated length
  std::vector<int64_t> deg(static_cast<size_t>(n));
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      int32_t* b = bucket.data() + cnt[r];
      int32_t* e = bucket.data() + cnt[r + 1];
      std::sort(b, e);
      deg[r] = std::unique(b, e) - b;
    }
  });
  HostCsr a;
  a.n = n;
  a.row_ptr.assign(static_cast<size_t>(n) + 1, 0);
  for (int64_t v = 0; v < n; ++v) a.row_ptr[v + 1] = a.row_ptr[v] + deg[v];
  a.col.resize(static_cast<size_t>(a.row_ptr[n]));
  a.val.resize(static_cast<size_t>(a.row_ptr[n]));
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    for (int64_t r = lo; r < hi; ++r) {
      const int32_t* b = bucket.data() + cnt[r];
      const int64_t o = a.row_ptr[r];
      for (int64_t k = 0; k < deg[r]; ++k) {
        const int64_t c = b[k];
        a.col[o + k] = c;
        a.val[o + k] = 1.0 / std::sqrt(static_cast<double>(deg[r]) * static_cast<double>(deg[c]));
      }
    }
  });
  return a;
}

void synthetic_features(int64_t n, int64_t d_in, uint64_t seed, float* out) {
  const uint64_t s0 = hash_combine(seed, 0xfea7);
  const int64_t total = n * d_in;
  if (total <= 0) return;
  const int64_t need = (total + 1) / 2;  // accepted attempts needed
  // attempt a uses draws 2a, 2a+1 (0-based): u = 2*unit-1, v = 2*unit-1
  auto attempt = [s0](int64_t a, double& u, double& v, double& q) {
    const uint64_t x0 = stream_draw(s0, static_cast<uint64_t>(2 * a));
    const uint64_t x1 = stream_draw(s0, static_cast<uint64_t>(2 * a + 1));
    u = 2.0 * (static_cast<double>(x0 >> 11) * 0x1.0p-53) - 1.0;
    v = 2.0 * (static_cast<double>(x1 >> 11) * 0x1.0p-53) - 1.0;
    q = u * u + v * v;
    return q < 1.0 && q != 0.0;
  };
  // acceptance rate pi/4: size the attempt range with slack, extend if short
  int64_t attempts = static_cast<int64_t>(static_cast<double>(need) / 0.78) + 4096;
  for (;;) {
    const int T = workers();
    const int64_t chunk = ceil_div(attempts, T);
    std::vector<int64_t> acc(static_cast<size_t>(T) + 1, 0);
    {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          const int64_t lo = t * chunk, hi = std::min(attempts, lo + chunk);
          int64_t c = 0;
          double u, v, q;
          for (int64_t a = lo; a < hi; ++a) c += attempt(a, u, v, q);
          acc[t + 1] = c;
        });
      for (auto& x : th) x.join();
    }
    for (int t = 0; t < T; ++t) acc[t + 1] += acc[t];
    if (acc[T] < need) {
      attempts = attempts * 2;
      continue;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
      th.emplace_back([&, t] {
        const int64_t lo = t * chunk, hi = std::min(attempts, lo + chunk);
        int64_t k = acc[t];
        double u, v, q;
        for (int64_t a = lo; a < hi && k < need; ++a) {
          if (!attempt(a, u, v, q)) continue;
          const double f = std::sqrt(-2.0 * std::log(q) / q);
          if (2 * k < total) out[2 * k] = static_cast<float>(u * f);
          if (2 * k + 1 < total) out[2 * k + 1] = static_cast<float>(v * f);
          ++k;
        }
      });
    for (auto& x : th) x.join();
    return;
  }
}

void degree_labels(int64_t n, const int64_t* row_ptr, int64_t n_classes, int32_t* labels) {
  int64_t maxd = 0;
  for (int64_t v = 0; v < n; ++v) maxd = std::max(maxd, row_ptr[v + 1] - row_ptr[v] - 1);
  std::vector<int64_t> cnt(static_cast<size_t>(maxd) + 2, 0);
  for (int64_t v = 0; v < n; ++v) ++cnt[row_ptr[v + 1] - row_ptr[v] - 1 + 1];
  for (int64_t d = 0; d <= maxd; ++d) cnt[d + 1] += cnt[d];
  for (int64_t v = 0; v < n; ++v) {
    const int64_t pos = cnt[row_ptr[v + 1] - row_ptr[v] - 1]++;
    labels[v] = static_cast<int32_t>((pos * n_classes) / n);
  }
}

void split_tags(int64_t n, uint64_t seed, uint8_t* split) {
  const uint64_t key = hash_combine(seed, 0x5b11);
  parallel_for(n, [&](int64_t lo, int64_t hi) {
    for (int64_t v = lo; v < hi; ++v) {
      const double u = element_unit(key, static_cast<uint64_t>(v), 0);
      split[v] = u < 0.6 ? 0 : (u < 0.8 ? 1 : 2);
    }
  });
}

HostDataset generate_synthetic(int64_t n, double avg_degree, int64_t d_in, int64_t n_classes,
                               uint64_t seed) {
  require(n >= 1, "generate_synthetic: n must be >= 1");
  require(avg_degree >= 0, "generate_synthetic: avg_degree must be >= 0");
  const auto uv = synthetic_edges(n, avg_degree, seed);
  return dataset_from_edges(n, uv.data(), static_cast<int64_t>(uv.size() / 2), d_in, n_classes, seed);
}

HostDataset dataset_from_edges(int64_t n, const int64_t* uv, int64_t m, int64_t d_in, int64_t n_classes,
                               uint64_t seed) {
  require(n >= 1, "generate_synthetic: n must be >= 1");
  require(n_classes >= 2, "generate_synthetic: n_classes must be >= 2");
  require(n_classes <= n, "generate_synthetic: n_classes > n");
  HostDataset ds;
  ds.adj = normalize_adjacency(uv, m, n);
  ds.n = n;
  ds.d_in = d_in;
  ds.n_classes = n_classes;
  ds.features.resize(static_cast<size_t>(n * d_in));
  synthetic_features(n, d_in, seed, ds.features.data());
  ds.labels.resize(static_cast<size_t>(n));
  degree_labels(n, ds.adj.row_ptr.data(), n_classes, ds.labels.data());
  ds.split.resize(static_cast<size_t>(n));
  split_tags(n, seed, ds.split.data());
  return ds;
}

}  // namespace ggb
