// gridgnn/pmm.hpp drop-in (reference: include/gridgnn/pmm.hpp:31-401): the
// 3D-PMM layer operators with the reference's names, argument lists, result
// structs and exceptions, computed on the B200 through the layer-level C ABI
// (include/ggb.h ggb_contract ... ggb_cross_entropy). Each call stages the
// ShardedTensor blocks through HBM and returns host results, like the
// reference's by-value API ("parity mode"); the training step itself keeps
// everything resident (ggb.hpp train_step). Real = float: the device path
// computes in fp32 (the reference's fp64 instantiation is its gradient-check
// mode, model.hpp:752-786).
#pragma once

#include <cstring>
#include <limits>
#include <span>
#include <type_traits>

#include "tensor.hpp"

namespace gridgnn {

// ---- layout schedule (pmm.hpp:31-63) --------------------------------------------
inline Layout adjacency_layout(int layer) {
  static const Layout cycle[3] = {{Axis::Z, Axis::X}, {Axis::Y, Axis::Z}, {Axis::X, Axis::Y}};
  return cycle[(layer - 1) % 3];
}
inline Layout feature_layout(int layer) {
  static const Layout cycle[3] = {{Axis::X, Axis::Y}, {Axis::Z, Axis::X}, {Axis::Y, Axis::Z}};
  return cycle[(layer - 1) % 3];
}
inline Layout hagg_layout(int layer) { return {adjacency_layout(layer).row, feature_layout(layer).col}; }
inline Layout weight_layout_for(Layout h) { return {h.col, third_axis(h)}; }
inline Layout weight_layout(int layer) { return weight_layout_for(hagg_layout(layer)); }
inline constexpr Layout kInputFeatureLayout{Axis::X, Axis::Z};

template <class Real>
struct RmsNormResult {
  ShardedTensor<Real> y;
  std::vector<Real> rms;
};
template <class Real>
struct RmsNormGrads {
  ShardedTensor<Real> dx;
  std::vector<Real> dgamma;
};
template <class Real>
struct FusedResult {
  ShardedTensor<Real> out;
  Dense<Real> scale;
};
template <class Real>
struct CrossEntropyResult {
  Real loss{};
  ShardedTensor<Real> grad_logits;
};

namespace detail {

template <class Real>
constexpr void fp32_only() {
  static_assert(std::is_same_v<Real, float>, "the B200 layer operators compute in fp32");
}

inline void need(bool ok, const char* msg) {
  if (!ok) throw CommContract(msg);
}

/// Device bytes owned for the duration of one operator call.
class DeviceBuffer {
 public:
  DeviceBuffer(ggb_ctx_t ctx, std::size_t bytes) : ctx_(ctx) { check(ggb_device_alloc(ctx, bytes, &p_)); }
  ~DeviceBuffer() {
    if (p_) ggb_device_free(ctx_, p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p_);
  }
  void upload(const void* src, std::size_t bytes) { check(ggb_memcpy_h2d(ctx_, p_, src, bytes)); }
  void download(void* dst, std::size_t bytes) const { check(ggb_memcpy_d2h(ctx_, dst, p_, bytes)); }

 private:
  ggb_ctx_t ctx_;
  void* p_ = nullptr;
};

/// A ShardedTensor's block in HBM + its ggb_block descriptor.
struct Staged {
  DeviceBuffer buf;
  ggb_block blk{};
  Staged(RankComm& rc, const ShardedTensor<float>& t, bool upload)
      : buf(rc.handle(), static_cast<std::size_t>(t.local.rows * t.local.cols) * sizeof(float)) {
    blk.row_axis = static_cast<std::int32_t>(t.layout.row);
    blk.col_axis = static_cast<std::int32_t>(t.layout.col);
    blk.g_rows = t.g_rows;
    blk.g_cols = t.g_cols;
    blk.row_off = t.row_off.data();
    blk.col_off = t.col_off.data();
    blk.data = buf.as<float>();
    blk.ld = std::max<index_t>(t.local.cols, 1);
    if (upload) buf.upload(t.local.v.data(), t.local.v.size() * sizeof(float));
  }
  void fetch(ShardedTensor<float>& t) const { buf.download(t.local.v.data(), t.local.v.size() * sizeof(float)); }
};

inline ShardedTensor<float> like(RankComm& rc, Layout lay, index_t g_rows, index_t g_cols,
                                 const std::vector<index_t>& row_off, const std::vector<index_t>& col_off) {
  return make_sharded<float>(rc.grid(), rc.coord(), lay, g_rows, g_cols, row_off, col_off);
}

/// The element-wise operators have no RankComm in the reference's signature:
/// they run on the calling thread's most recent context (one per GPU).
inline RankComm& elementwise_context() {
  thread_local std::unique_ptr<RankComm> own;
  if (!own) own = std::make_unique<RankComm>(DeviceGrid(1, 1, 1, 1), 0);
  return *own;
}

}  // namespace detail

/// Materialized local transpose (pmm.hpp:76-92): layout, partitions and block swapped.
template <class Real>
ShardedTensor<Real> transposed(const ShardedTensor<Real>& t) {
  ShardedTensor<Real> out;
  out.layout = {t.layout.col, t.layout.row};
  out.g_rows = t.g_cols;
  out.g_cols = t.g_rows;
  out.row_off = t.col_off;
  out.col_off = t.row_off;
  out.r0 = t.c0;
  out.r1 = t.c1;
  out.c0 = t.r0;
  out.c1 = t.r1;
  out.local = Dense<Real>(t.local.cols, t.local.rows);
  for (index_t i = 0; i < t.local.rows; ++i)
    for (index_t j = 0; j < t.local.cols; ++j) out.local.at(j, i) = t.local.at(i, j);
  return out;
}

/// C = A . B, all-reduce along A's column axis (pmm.hpp:97-130).
template <class Real>
ShardedTensor<Real> contract(RankComm& rc, const ShardedTensor<Real>& a, const ShardedTensor<Real>& b,
                             Precision prec = Precision::kFp32) {
  detail::fp32_only<Real>();
  detail::need(a.layout.col == b.layout.row, "contract: inner axes differ");
  detail::need(a.g_cols == b.g_rows, "contract: inner dimensions differ");
  detail::need(a.col_off == b.row_off, "contract: inner partitions differ");
  detail::need(a.layout.row != b.layout.col, "contract: output axes collide");
  detail::need(a.local_cols() == b.local_rows(), "contract: local inner blocks differ");
  ShardedTensor<Real> c = detail::like(rc, {a.layout.row, b.layout.col}, a.g_rows, b.g_cols, a.row_off, b.col_off);
  detail::Staged sa(rc, a, true), sb(rc, b, true), sc(rc, c, false);
  detail::check(ggb_contract(rc.handle(), &sa.blk, &sb.blk, &sc.blk, static_cast<std::int32_t>(prec)));
  sc.fetch(c);
  return c;
}

/// H = A . F with a sparse A, all-reduce along A's column axis (pmm.hpp:134-167).
template <class Real>
ShardedTensor<Real> spmm(RankComm& rc, const ShardedSparse& a, const ShardedTensor<Real>& f,
                         Precision prec = Precision::kFp32) {
  detail::fp32_only<Real>();
  detail::need(a.layout.col == f.layout.row, "spmm: inner axes differ");
  detail::need(a.g_cols == f.g_rows, "spmm: inner dimensions differ");
  detail::need(a.col_off == f.row_off, "spmm: inner partitions differ");
  detail::need(a.r1 - a.r0 == a.local.n_rows && a.c1 - a.c0 == a.local.n_cols, "spmm: sparse block shape mismatch");
  detail::need(f.local_rows() == a.local.n_cols, "spmm: local inner blocks differ");
  ShardedTensor<Real> h = detail::like(rc, {a.layout.row, f.layout.col}, a.g_rows, f.g_cols, a.row_off, f.col_off);
  const index_t rows = a.local.n_rows, nnz = a.local.nnz();
  std::vector<std::int32_t> col(static_cast<std::size_t>(nnz));
  std::vector<float> val(static_cast<std::size_t>(nnz));
  for (index_t e = 0; e < nnz; ++e) {
    col[static_cast<std::size_t>(e)] = static_cast<std::int32_t>(a.local.col_idx[static_cast<std::size_t>(e)]);
    val[static_cast<std::size_t>(e)] = static_cast<float>(a.local.values[static_cast<std::size_t>(e)]);  // pmm.hpp:160
  }
  detail::DeviceBuffer rp(rc.handle(), static_cast<std::size_t>(rows + 1) * 8),
      cb(rc.handle(), static_cast<std::size_t>(nnz) * 4 + 4), vb(rc.handle(), static_cast<std::size_t>(nnz) * 4 + 4);
  rp.upload(a.local.row_ptr.data(), static_cast<std::size_t>(rows + 1) * 8);
  cb.upload(col.data(), col.size() * 4);
  vb.upload(val.data(), val.size() * 4);
  ggb_csr_block ab{};
  ab.row_axis = static_cast<std::int32_t>(a.layout.row);
  ab.col_axis = static_cast<std::int32_t>(a.layout.col);
  ab.g_rows = a.g_rows;
  ab.g_cols = a.g_cols;
  ab.row_off = a.row_off.data();
  ab.col_off = a.col_off.data();
  ab.row_ptr = rp.as<std::int64_t>();
  ab.col = cb.as<std::int32_t>();
  ab.val = vb.as<float>();
  detail::Staged sf(rc, f, true), sh(rc, h, false);
  detail::check(ggb_spmm(rc.handle(), &ab, &sf.blk, &sh.blk, static_cast<std::int32_t>(prec)));
  sh.fetch(h);
  return h;
}

/// The full matrix on every rank (pmm.hpp:171-195).
template <class Real>
Dense<Real> gather_full(RankComm& rc, const ShardedTensor<Real>& t) {
  detail::fp32_only<Real>();
  Dense<Real> out(t.g_rows, t.g_cols);
  detail::Staged st(rc, t, true);
  detail::DeviceBuffer full(rc.handle(), out.v.size() * sizeof(float));
  detail::check(ggb_gather_full(rc.handle(), &st.blk, full.as<float>(), std::max<index_t>(t.g_cols, 1)));
  full.download(out.v.data(), out.v.size() * sizeof(float));
  return out;
}

/// A new layout / partition (pmm.hpp:197-204), by block permutation.
template <class Real>
ShardedTensor<Real> reshard(RankComm& rc, const ShardedTensor<Real>& t, Layout layout, std::vector<index_t> row_off,
                            std::vector<index_t> col_off) {
  detail::fp32_only<Real>();
  if (layout == t.layout && row_off == t.row_off && col_off == t.col_off) return t;
  ShardedTensor<Real> out = detail::like(rc, layout, t.g_rows, t.g_cols, row_off, col_off);
  detail::Staged ss(rc, t, true), sd(rc, out, false);
  detail::check(ggb_reshard(rc.handle(), &ss.blk, &sd.blk));
  sd.fetch(out);
  return out;
}

/// y = gamma . x / rms(x) over the full feature dimension (pmm.hpp:214-243).
template <class Real>
RmsNormResult<Real> parallel_rmsnorm_fwd(RankComm& rc, const ShardedTensor<Real>& x, std::span<const Real> gamma,
                                         Real eps) {
  detail::fp32_only<Real>();
  detail::need(static_cast<index_t>(gamma.size()) == x.local_cols(),
               "rmsnorm: gamma slice does not match the column block");
  RmsNormResult<Real> r;
  r.y = x;
  r.rms.assign(static_cast<std::size_t>(x.local_rows()), 0.f);
  detail::Staged sx(rc, x, true), sy(rc, r.y, false);
  detail::DeviceBuffer g(rc.handle(), gamma.size() * 4 + 4), rms(rc.handle(), r.rms.size() * 4 + 4);
  g.upload(gamma.data(), gamma.size() * 4);
  detail::check(ggb_rmsnorm_fwd(rc.handle(), &sx.blk, g.as<float>(), eps, &sy.blk, rms.as<float>()));
  sy.fetch(r.y);
  rms.download(r.rms.data(), r.rms.size() * 4);
  return r;
}

/// dx and dgamma (pmm.hpp:251-287).
template <class Real>
RmsNormGrads<Real> parallel_rmsnorm_bwd(RankComm& rc, const ShardedTensor<Real>& x, std::span<const Real> gamma,
                                        const std::vector<Real>& rms, const ShardedTensor<Real>& dy) {
  detail::fp32_only<Real>();
  detail::need(static_cast<index_t>(rms.size()) == x.local_rows(), "rmsnorm_bwd: missing cache");
  detail::need(dy.layout == x.layout && dy.r0 == x.r0 && dy.c0 == x.c0, "rmsnorm_bwd: gradient layout mismatch");
  RmsNormGrads<Real> g;
  g.dx = x;
  g.dgamma.assign(static_cast<std::size_t>(x.local_cols()), 0.f);
  detail::Staged sx(rc, x, true), sdy(rc, dy, true), sdx(rc, g.dx, false);
  detail::DeviceBuffer gm(rc.handle(), gamma.size() * 4 + 4), rb(rc.handle(), rms.size() * 4 + 4),
      dg(rc.handle(), g.dgamma.size() * 4 + 4);
  gm.upload(gamma.data(), gamma.size() * 4);
  rb.upload(rms.data(), rms.size() * 4);
  detail::check(
      ggb_rmsnorm_bwd(rc.handle(), &sx.blk, gm.as<float>(), rb.as<float>(), &sdy.blk, &sdx.blk, dg.as<float>()));
  sdx.fetch(g.dx);
  dg.download(g.dgamma.data(), g.dgamma.size() * 4);
  return g;
}

/// out = dropout(relu(x)) + h_prev (pmm.hpp:299-328); scale is rebuilt from the keep bits.
template <class Real>
FusedResult<Real> fused_elementwise_fwd(const ShardedTensor<Real>& x,
                                        std::type_identity_t<const ShardedTensor<Real>*> h_prev, double rate,
                                        std::uint64_t mask_key, bool training) {
  detail::fp32_only<Real>();
  if (!(rate >= 0.0 && rate < 1.0)) throw std::invalid_argument("fused_elementwise: dropout rate must be in [0, 1)");
  if (h_prev)
    detail::need(h_prev->layout == x.layout && h_prev->r0 == x.r0 && h_prev->c0 == x.c0 && h_prev->r1 == x.r1 &&
                     h_prev->c1 == x.c1,
                 "fused_elementwise: residual layout mismatch");
  RankComm& rc = detail::elementwise_context();
  // the element-wise operator needs the block's global coordinates, not its
  // partition: stage it as a one-rank block whose offsets put it at (r0, c0)
  auto one_rank = [&](const ShardedTensor<Real>& t) {
    ShardedTensor<Real> v = t;
    v.row_off = {0, t.g_rows};
    v.col_off = {0, t.g_cols};
    return v;
  };
  FusedResult<Real> r;
  r.out = x;
  r.scale = Dense<Real>(x.local_rows(), x.local_cols());
  const index_t m = x.local_rows(), n = x.local_cols(), ldm = ggb_mask_words(n);
  // a full-height staging block with this block's rows at r0 .. r1
  ShardedTensor<Real> xs = one_rank(x), os = one_rank(x);
  xs.local = Dense<Real>(x.g_rows, x.g_cols);
  for (index_t i = 0; i < m; ++i) std::copy_n(&x.local.at(i, 0), n, &xs.local.at(x.r0 + i, x.c0));
  os.local = Dense<Real>(x.g_rows, x.g_cols);
  ShardedTensor<Real> hs;
  if (h_prev) {
    hs = one_rank(*h_prev);
    hs.local = Dense<Real>(x.g_rows, x.g_cols);
    for (index_t i = 0; i < m; ++i) std::copy_n(&h_prev->local.at(i, 0), n, &hs.local.at(x.r0 + i, x.c0));
  }
  const index_t ldm_full = ggb_mask_words(x.g_cols);
  detail::Staged sx(rc, xs, true), so(rc, os, false);
  std::unique_ptr<detail::Staged> sh;
  if (h_prev) sh = std::make_unique<detail::Staged>(rc, hs, true);
  detail::DeviceBuffer bits(rc.handle(), static_cast<std::size_t>(x.g_rows * ldm_full) * 4 + 4);
  detail::check(ggb_fused_elementwise_fwd(rc.handle(), &sx.blk, h_prev ? &sh->blk : nullptr, rate, mask_key,
                                          training ? 1 : 0, &so.blk, bits.as<std::uint32_t>()));
  so.fetch(os);
  std::vector<std::uint32_t> hb(static_cast<std::size_t>(x.g_rows * ldm_full));
  bits.download(hb.data(), hb.size() * 4);
  const float ks = training && rate > 0.0 ? static_cast<float>(1.0 / (1.0 - rate)) : 1.0f;
  for (index_t i = 0; i < m; ++i)
    for (index_t j = 0; j < n; ++j) {
      const index_t gi = x.r0 + i, gj = x.c0 + j;  // word 4(gj/128) + gj%4, bit (gj%128)/4
      const std::uint32_t w = hb[static_cast<std::size_t>(gi * ldm_full + 4 * (gj / 128) + gj % 4)];
      r.scale.at(i, j) = ((w >> ((gj % 128) / 4)) & 1u) ? ks : 0.f;
      r.out.local.at(i, j) = os.local.at(gi, gj);
    }
  (void)ldm;
  return r;
}

/// dx = dy . scale (pmm.hpp:331-341).
template <class Real>
ShardedTensor<Real> fused_elementwise_bwd(const ShardedTensor<Real>& dy, const Dense<Real>& scale) {
  detail::fp32_only<Real>();
  detail::need(scale.rows == dy.local_rows() && scale.cols == dy.local_cols(), "fused_elementwise_bwd: missing cache");
  RankComm& rc = detail::elementwise_context();
  const index_t m = dy.local_rows(), n = dy.local_cols(), ldm = ggb_mask_words(n);
  // the cache as keep bits + the kept value (the reference's scale is 0 or 1/(1-rate))
  std::vector<std::uint32_t> bits(static_cast<std::size_t>(std::max<index_t>(m * ldm, 1)), 0u);
  float ks = 1.f;
  for (index_t i = 0; i < m; ++i)
    for (index_t j = 0; j < n; ++j)
      if (scale.at(i, j) != 0.f) {
        ks = scale.at(i, j);
        bits[static_cast<std::size_t>(i * ldm + 4 * (j / 128) + j % 4)] |= 1u << ((j % 128) / 4);
      }
  ShardedTensor<Real> dys = dy, dx = dy;
  dys.row_off = {0, m};
  dys.col_off = {0, n};
  dys.g_rows = m;
  dys.g_cols = n;
  ShardedTensor<Real> dxs = dys;
  detail::Staged sdy(rc, dys, true), sdx(rc, dxs, false);
  detail::DeviceBuffer kb(rc.handle(), bits.size() * 4);
  kb.upload(bits.data(), bits.size() * 4);
  detail::check(ggb_fused_elementwise_bwd(rc.handle(), &sdy.blk, kb.as<std::uint32_t>(), ks, &sdx.blk));
  sdx.fetch(dx);
  return dx;
}

/// Mean softmax cross-entropy over class-sharded logits (pmm.hpp:352-401).
template <class Real>
CrossEntropyResult<Real> parallel_cross_entropy(RankComm& rc, const ShardedTensor<Real>& logits,
                                                const std::vector<std::int32_t>& labels) {
  detail::fp32_only<Real>();
  if (static_cast<index_t>(labels.size()) != logits.g_rows)
    throw std::invalid_argument("cross_entropy: one label per batch row required");
  for (auto y : labels)
    if (y < 0 || static_cast<index_t>(y) >= logits.g_cols) throw std::invalid_argument("cross_entropy: label out of range");
  CrossEntropyResult<Real> r;
  r.grad_logits = logits;
  detail::Staged sl(rc, logits, true), sg(rc, r.grad_logits, false);
  detail::DeviceBuffer lab(rc.handle(), labels.size() * 4 + 4), loss(rc.handle(), 4);
  lab.upload(labels.data(), labels.size() * 4);
  detail::check(ggb_cross_entropy(rc.handle(), &sl.blk, lab.as<std::int32_t>(), loss.as<float>(), &sg.blk));
  sg.fetch(r.grad_logits);
  loss.download(&r.loss, 4);
  return r;
}

}  // namespace gridgnn
