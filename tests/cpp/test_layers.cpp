// The C++ layer drop-in (cpp/gridgnn/pmm.hpp, tensor.hpp, shardsample.hpp)
// called with the reference's names and argument lists, checked against the
// reference's own operators (oracle/_ref through its neutral C shim — test
// infrastructure only) and against known answers of the reference's unit
// tests (test_pmm.cpp, test_shardsample.cpp). One PASS/FAIL line per check.
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "../../paper_2604_02651_b200/cpp/gridgnn/pmm.hpp"
#include "../../paper_2604_02651_b200/cpp/gridgnn/shardsample.hpp"

extern "C" {  // oracle/ref_shim.cpp
int ref_contract(std::int64_t m, std::int64_t k, std::int64_t n, const float* a, const float* b, int prec, float* c);
int ref_spmm(std::int64_t rows, std::int64_t cols, const std::int64_t* rp, const std::int64_t* col, const double* val,
             const float* f, std::int64_t n, int prec, float* h);
int ref_rmsnorm(std::int64_t m, std::int64_t n, const float* x, const float* gamma, float eps, const float* dy,
                float* y, float* rms, float* dx, float* dgamma);
int ref_fused(std::int64_t m, std::int64_t n, const float* x, const float* h_prev, double rate, std::uint64_t key,
              int training, const float* dy, float* out, float* scale, float* dx);
int ref_cross_entropy(std::int64_t m, std::int64_t n, const float* logits, const std::int32_t* labels, float* loss,
                      float* grad);
}

using namespace gridgnn;

static int g_fail = 0;
static void report(const char* name, bool ok, const std::string& detail = "") {
  std::printf("%-52s %s  %s\n", name, ok ? "PASS" : "FAIL", detail.c_str());
  if (!ok) ++g_fail;
}

static std::vector<float> randn(std::size_t n, unsigned seed, float scale = 1.f) {
  std::mt19937 g(seed);
  std::normal_distribution<float> d(0.f, scale);
  std::vector<float> v(n);
  for (auto& x : v) x = d(g);
  return v;
}

static float max_abs(const std::vector<float>& a) {
  float m = 0.f;
  for (float x : a) m = std::max(m, std::fabs(x));
  return m;
}

static float max_diff(const std::vector<float>& a, const std::vector<float>& b) {
  float m = 0.f;
  for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a[i] - b[i]));
  return m;
}

template <class F>
static bool throws_contract(F&& f) {
  try {
    f();
  } catch (const CommContract&) {
    return true;
  } catch (...) {
  }
  return false;
}

int main() {
  DeviceGrid grid(1, 1, 1, 1);
  RankComm rc(grid, 0);
  const Coord4 me = rc.coord();
  auto full = [&](Layout lay, index_t r, index_t c, const std::vector<float>& v) {
    Dense<float> d(r, c);
    d.v = v;
    return shard_from_global(grid, me, lay, d, {0, r}, {0, c});
  };

  {  // contract (pmm.hpp:97-130) vs the reference operator; test_pmm.cpp:129-152 KAT
    const index_t m = 700, k = 256, n = 47;
    auto a = full({Axis::X, Axis::Y}, m, k, randn(m * k, 1)), b = full({Axis::Y, Axis::Z}, k, n, randn(k * n, 2, 0.1f));
    auto c = contract(rc, a, b);
    std::vector<float> want(m * n);
    ref_contract(m, k, n, a.local.v.data(), b.local.v.data(), 0, want.data());
    const float d = max_diff(c.local.v, want);
    report("contract == reference (700x256x47)", d <= 1e-5f * std::max(1.f, max_abs(want)), std::to_string(d));
    auto ka = full({Axis::X, Axis::Y}, 2, 2, {1, 2, 3, 4}), kb = full({Axis::Y, Axis::Z}, 2, 1, {1, 2});
    auto kc = contract(rc, ka, kb);
    report("contract KAT [[1,2],[3,4]].[1,2] = [5,11]", kc.local.v == std::vector<float>({5, 11}));
    report("contract: inner axes differ -> CommContract",
           throws_contract([&] { contract(rc, ka, full({Axis::Z, Axis::X}, 2, 1, {1, 2})); }));
  }
  {  // spmm (pmm.hpp:134-167)
    const index_t rows = 500, cols = 800, n = 256;
    std::mt19937 g(3);
    ShardedSparse a;
    a.layout = {Axis::Z, Axis::X};
    a.g_rows = rows;
    a.g_cols = cols;
    a.row_off = {0, rows};
    a.col_off = {0, cols};
    a.r1 = rows;
    a.c1 = cols;
    a.local.n_rows = rows;
    a.local.n_cols = cols;
    for (index_t r = 0; r < rows; ++r) {
      for (index_t c = 0; c < cols; ++c)
        if (g() % 40 == 0) {
          a.local.col_idx.push_back(c);
          a.local.values.push_back(std::uniform_real_distribution<double>(0, 1)(g));
        }
      a.local.row_ptr.push_back(static_cast<index_t>(a.local.col_idx.size()));
    }
    auto f = full({Axis::X, Axis::Y}, cols, n, randn(cols * n, 4));
    auto h = spmm(rc, a, f);
    std::vector<float> want(rows * n);
    ref_spmm(rows, cols, a.local.row_ptr.data(), a.local.col_idx.data(), a.local.values.data(), f.local.v.data(), n, 0,
             want.data());
    const float d = max_diff(h.local.v, want);
    report("spmm == reference (500x800, H 256)", d <= 1e-5f * std::max(1.f, max_abs(want)), std::to_string(d));
  }
  {  // parallel_rmsnorm_fwd / _bwd (pmm.hpp:214-287); test_pmm.cpp:306-390 KAT
    const index_t m = 300, n = 256;
    auto x = full({Axis::X, Axis::Y}, m, n, randn(m * n, 5));
    auto dy = full({Axis::X, Axis::Y}, m, n, randn(m * n, 6));
    std::vector<float> gamma = randn(n, 7, 0.1f);
    for (auto& v : gamma) v += 1.f;
    auto r = parallel_rmsnorm_fwd<float>(rc, x, gamma, 1e-6f);
    auto gr = parallel_rmsnorm_bwd<float>(rc, x, gamma, r.rms, dy);
    std::vector<float> y(m * n), rms(m), dx(m * n), dg(n);
    ref_rmsnorm(m, n, x.local.v.data(), gamma.data(), 1e-6f, dy.local.v.data(), y.data(), rms.data(), dx.data(),
                dg.data());
    const float d = std::max({max_diff(r.y.local.v, y) / std::max(1.f, max_abs(y)), max_diff(r.rms, rms),
                              max_diff(gr.dx.local.v, dx) / std::max(1.f, max_abs(dx)),
                              max_diff(gr.dgamma, dg) / std::max(1.f, max_abs(dg))});
    report("parallel_rmsnorm_fwd/bwd == reference", d <= 1e-5f, std::to_string(d));
    auto k = parallel_rmsnorm_fwd<float>(rc, full({Axis::X, Axis::Y}, 1, 2, {3, 4}), std::vector<float>{1, 1}, 0.f);
    report("rmsnorm KAT [3,4] -> rms sqrt(12.5), y [0.848528, 1.131371]",
           std::fabs(k.rms[0] - std::sqrt(12.5f)) < 1e-6f && std::fabs(k.y.local.v[0] - 0.848528f) < 1e-6f &&
               std::fabs(k.y.local.v[1] - 1.131371f) < 1e-6f);
  }
  {  // fused_elementwise_fwd / _bwd (pmm.hpp:299-341); test_pmm.cpp:395-434 KAT
    const index_t m = 400, n = 256;
    auto x = full({Axis::X, Axis::Y}, m, n, randn(m * n, 8));
    auto hp = full({Axis::X, Axis::Y}, m, n, randn(m * n, 9));
    auto dy = full({Axis::X, Axis::Y}, m, n, randn(m * n, 10));
    auto r = fused_elementwise_fwd<float>(x, &hp, 0.3, 0xabcdef, true);
    auto dx = fused_elementwise_bwd(dy, r.scale);
    std::vector<float> out(m * n), scale(m * n), rdx(m * n);
    ref_fused(m, n, x.local.v.data(), hp.local.v.data(), 0.3, 0xabcdef, 1, dy.local.v.data(), out.data(),
              scale.data(), rdx.data());
    report("fused_elementwise scale (dropout mask) == reference", r.scale.v == scale);
    report("fused_elementwise_bwd == reference", dx.local.v == rdx);
    report("fused_elementwise_fwd == reference (one rounding)",
           max_diff(r.out.local.v, out) <= 1e-6f * std::max(1.f, max_abs(out)));
    auto kx = full({Axis::X, Axis::Y}, 1, 4, {0, 2, -3, 4}), kh = full({Axis::X, Axis::Y}, 1, 4, {10, 20, 30, 36});
    auto k = fused_elementwise_fwd<float>(kx, &kh, 0.0, 1, true);
    report("fused KAT rate 0: relu + residual", k.out.local.v == std::vector<float>({10, 22, 30, 40}));
    bool threw = false;
    try {
      fused_elementwise_fwd<float>(kx, nullptr, 1.0, 1, true);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    report("fused: rate 1 -> std::invalid_argument", threw);
  }
  {  // parallel_cross_entropy (pmm.hpp:352-401); test_pmm.cpp:462-520 KAT
    const index_t m = 600, n = 47;
    auto lg = full({Axis::X, Axis::Z}, m, n, randn(m * n, 11, 3.f));
    std::vector<std::int32_t> labels(m);
    for (index_t i = 0; i < m; ++i) labels[i] = static_cast<std::int32_t>((i * 7) % n);
    auto r = parallel_cross_entropy(rc, lg, labels);
    float loss = 0.f;
    std::vector<float> grad(m * n);
    ref_cross_entropy(m, n, lg.local.v.data(), labels.data(), &loss, grad.data());
    report("parallel_cross_entropy == reference",
           std::fabs(r.loss - loss) <= 1e-5f * loss && max_diff(r.grad_logits.local.v, grad) <= 1e-6f,
           std::to_string(r.loss) + " vs " + std::to_string(loss));
    auto k = parallel_cross_entropy(rc, full({Axis::X, Axis::Z}, 1, 2, {0, 0}), std::vector<std::int32_t>{0});
    report("cross-entropy KAT [0,0] -> ln 2, grad -0.5 / +0.5",
           std::fabs(k.loss - std::log(2.f)) < 1e-6f && std::fabs(k.grad_logits.local.v[0] + 0.5f) < 1e-6f &&
               std::fabs(k.grad_logits.local.v[1] - 0.5f) < 1e-6f);
  }
  {  // transposed / gather_full / reshard (pmm.hpp:76-204) on one rank
    auto a = full({Axis::X, Axis::Y}, 30, 17, randn(30 * 17, 12));
    auto t = transposed(a);
    bool ok = t.layout == Layout{Axis::Y, Axis::X} && t.local.rows == 17 && t.local.at(3, 5) == a.local.at(5, 3);
    auto g = gather_full(rc, a);
    auto r = reshard(rc, a, Layout{Axis::Z, Axis::X}, {0, 30}, {0, 17});
    report("transposed / gather_full / reshard (data movement)", ok && g.v == a.local.v && r.local.v == a.local.v);
  }
  {  // shardsample index functions: test_shardsample.cpp:34-39, 233-240 KATs
    SampleSet s;
    s.vertices = {1, 3, 6, 8};
    s.batch_size = 4;
    const bool bp = block_partition(10, 3) == std::vector<index_t>({0, 4, 7, 10}) &&
                    block_partition(2, 3) == std::vector<index_t>({0, 1, 2, 2});
    const bool sp = sample_partition(s, {0, 2, 4, 10}) == std::vector<index_t>({0, 1, 2, 4});
    const LocalRanges lr = locate_ranges(s, 2, 7, 0, 4);
    report("block_partition / sample_partition / locate_ranges KATs",
           bp && sp && lr.row_lo == 1 && lr.row_hi == 3 && lr.col_lo == 0 && lr.col_hi == 2);
  }
  std::printf("%d failure(s)\n", g_fail);
  return g_fail;
}
