// Device training step: init_state (model.hpp:175-208), forward
// (model.hpp:335-376), parallel_cross_entropy (pmm.hpp:352-401), backward
// (model.hpp:378-420), dp_sync (model.hpp:423-433) and optimizer_step
// (model.hpp:435-456). Every contraction follows the reference's 3D-PMM
// rule (pmm.hpp:17-29): local product, then an all-reduce along the
// contraction axis (a no-op for singleton groups).
#include <cmath>

#include "comm.hpp"
#include "prof.hpp"
#include "rng.cuh"
#include "trainer.hpp"

namespace ggb {

Block make_block(const Ctx& ctx, Layout lay, int64_t g_rows, int64_t g_cols,
                 const std::vector<int64_t>& row_off, const std::vector<int64_t>& col_off) {
  Block b;
  b.lay = lay;
  b.g_rows = g_rows;
  b.g_cols = g_cols;
  const int cr = ctx.coord[lay.row], cc = ctx.coord[lay.col];
  b.r0 = row_off[cr];
  b.r1 = row_off[cr + 1];
  b.c0 = col_off[cc];
  b.c1 = col_off[cc + 1];
  return b;
}

namespace {

inline int64_t ld8(int64_t c) { return round_up(std::max<int64_t>(c, 1), 8); }

template <class T>
T* grow(DevBuf& b, int64_t n) {
  return b.reserve_n<T>(static_cast<size_t>(std::max<int64_t>(n, 1)));
}

std::vector<int64_t> hoff(const Ctx& ctx, int64_t d, int axis) { return block_partition(d, ctx.grid.dims[axis]); }

// ---- reshard (pmm.hpp:171-204) as a block permutation -----------------------------
// The reference all-gathers the full matrix along both source axes and slices
// the new block. Here every destination rank receives exactly the pieces of
// its new block, each from one provider: the rank holding that source block
// whose coordinate on the source layout's replica axis equals the receiver's
// (so replicas of a source block share the sending). Pure data movement, hence
// bit-exact; about g^2 times fewer bytes than the gather.
struct Span {
  int64_t lo, hi;
};
inline Span meet(int64_t a0, int64_t a1, int64_t b0, int64_t b1) { return {std::max(a0, b0), std::min(a1, b1)}; }

void reshard(Ctx& ctx, const Block& sb, const std::vector<int64_t>& s_roff, const std::vector<int64_t>& s_coff,
             const float* src, int64_t lds, const Block& db, const std::vector<int64_t>& d_roff,
             const std::vector<int64_t>& d_coff, float* dst, int64_t ldd) {
  const Grid& G = ctx.grid;
  const int me = ctx.rank;
  int mc[4];
  G.coord_of(me, mc);
  const Layout sl = sb.lay, dl = db.lay;
  const int s_rep = third_axis(sl);
  if (peer_ok(ctx, kPeerPmm, GGB_FP32)) {
    // through peer memory: stage the source block, pull the destination's
    // pieces — on the reshard stream, joined by the consumer (reshard_join)
    size_t reserve = 0;  // the group's largest source block (same offsets on every member)
    for (int i = 0; i + 1 < static_cast<int>(s_roff.size()); ++i)
      for (int j = 0; j + 1 < static_cast<int>(s_coff.size()); ++j)
        reserve = std::max(reserve, static_cast<size_t>((s_roff[i + 1] - s_roff[i]) * ld8(s_coff[j + 1] - s_coff[j])) * 4);
    const int psize = G.dims[1] * G.dims[2] * G.dims[3];
    std::vector<PeerPiece> pieces;
    for (int i = 0; i + 1 < static_cast<int>(s_roff.size()); ++i)
      for (int j = 0; j + 1 < static_cast<int>(s_coff.size()); ++j) {
        const Span r = meet(s_roff[i], s_roff[i + 1], db.r0, db.r1), c = meet(s_coff[j], s_coff[j + 1], db.c0, db.c1);
        if (r.lo >= r.hi || c.lo >= c.hi) continue;
        int pc[4] = {mc[0], mc[1], mc[2], mc[3]};
        pc[sl.row] = i;
        pc[sl.col] = j;
        pc[s_rep] = mc[s_rep];
        const int64_t ldp = ld8(s_coff[j + 1] - s_coff[j]);
        pieces.push_back({G.rank_of(pc) % psize, (r.lo - s_roff[i]) * ldp + (c.lo - s_coff[j]), ldp,
                          dst + (r.lo - db.r0) * ldd + (c.lo - db.c0), ldd, r.hi - r.lo, c.hi - c.lo});
      }
    reshard_async(ctx, [&] {
      peer_stage(ctx, src, lds, sb.rows(), sb.cols(), ld8(sb.cols()), reserve);
      peer_pull(ctx, pieces);
    });
    return;
  }
  std::vector<BlockXfer> sends, recvs;
  // receives: pieces of my destination block
  for (int i = 0; i + 1 < static_cast<int>(s_roff.size()); ++i)
    for (int j = 0; j + 1 < static_cast<int>(s_coff.size()); ++j) {
      const Span r = meet(s_roff[i], s_roff[i + 1], db.r0, db.r1), c = meet(s_coff[j], s_coff[j + 1], db.c0, db.c1);
      if (r.lo >= r.hi || c.lo >= c.hi) continue;
      int pc[4] = {mc[0], mc[1], mc[2], mc[3]};
      pc[sl.row] = i;
      pc[sl.col] = j;
      pc[s_rep] = mc[s_rep];
      const int p = G.rank_of(pc);
      float* out = dst + (r.lo - db.r0) * ldd + (c.lo - db.c0);
      if (p == me) {  // local piece
        GGB_CUDA(cudaMemcpy2DAsync(out, ldd * 4, src + (r.lo - sb.r0) * lds + (c.lo - sb.c0), lds * 4,
                                   (c.hi - c.lo) * 4, r.hi - r.lo, cudaMemcpyDeviceToDevice, ctx.stream));
      } else {
        recvs.push_back({p, out, ldd, r.hi - r.lo, c.hi - c.lo});
      }
    }
  // sends: for every rank q of my DP group that takes its piece from me
  for (int q = 0; q < G.total(); ++q) {
    if (q == me) continue;
    int qc[4];
    G.coord_of(q, qc);
    if (qc[0] != mc[0] || qc[s_rep] != mc[s_rep]) continue;  // other DP group / other provider
    const int64_t q_r0 = d_roff[qc[dl.row]], q_r1 = d_roff[qc[dl.row] + 1];
    const int64_t q_c0 = d_coff[qc[dl.col]], q_c1 = d_coff[qc[dl.col] + 1];
    const Span r = meet(sb.r0, sb.r1, q_r0, q_r1), c = meet(sb.c0, sb.c1, q_c0, q_c1);
    if (r.lo >= r.hi || c.lo >= c.hi) continue;
    sends.push_back({q, const_cast<float*>(src) + (r.lo - sb.r0) * lds + (c.lo - sb.c0), lds, r.hi - r.lo,
                     c.hi - c.lo});
  }
  exchange_blocks(ctx, sends, recvs);
}

// reshard's accounting (pmm.hpp:171-204): a layout change runs gather_full,
// an all-gather of the column strip (g_rows x local cols) along the row axis,
// then of the whole matrix along the column axis; an unchanged layout is free
void charge_reshard(Ctx& ctx, const Block& t, Layout to) {
  if (t.lay == to) return;
  charge_all_gather(ctx, t.lay.row, static_cast<uint64_t>(t.g_rows) * t.cols() * 4);
  charge_all_gather(ctx, t.lay.col, static_cast<uint64_t>(t.g_rows) * t.g_cols * 4);
}

inline int wire_bytes(int wire) { return wire == GGB_FP32 ? 4 : 2; }  // RankComm::elem_bytes (comm.hpp:266-270)

bool pmm_trivial(const Ctx& ctx) { return ctx.grid.dims[1] == 1 && ctx.grid.dims[2] == 1 && ctx.grid.dims[3] == 1; }

}  // namespace

void reshard_block(Ctx& ctx, const Block& sb, const std::vector<int64_t>& s_roff, const std::vector<int64_t>& s_coff,
                   const float* src, int64_t lds, const Block& db, const std::vector<int64_t>& d_roff,
                   const std::vector<int64_t>& d_coff, float* dst, int64_t ldd) {
  reshard(ctx, sb, s_roff, s_coff, src, lds, db, d_roff, d_coff, dst, ldd);
  reshard_join(ctx);
}

// ---- init_state (model.hpp:175-208) -------------------------------------------------
void state_init(Ctx& ctx, State& st, const ggb_model_config& cfg, uint64_t seed) {
  require(cfg.layers >= 1, "ModelConfig: layers must be >= 1");
  require(cfg.d_in >= 1 && cfg.d_h >= 1 && cfg.d_out >= 1, "ModelConfig: dims must be >= 1");
  require(cfg.dropout_rate >= 0.0 && cfg.dropout_rate < 1.0, "ModelConfig: dropout rate must be in [0, 1)");
  st.ctx = &ctx;
  st.cfg = cfg;
  st.seed = seed;
  st.params.clear();
  st.wl.clear();
  st.gamma.clear();
  int64_t off = 0;
  auto add_mat = [&](Layout lay, int64_t rows, int64_t cols) {
    ParamSlot p;
    p.blk = make_block(ctx, lay, rows, cols, hoff(ctx, rows, lay.row), hoff(ctx, cols, lay.col));
    p.off = off;
    p.n = p.blk.rows() * p.blk.cols();
    p.ldb = ld8(p.blk.cols());
    p.ldt = ld8(p.blk.rows());
    off += round_up(std::max<int64_t>(p.n, 1), 64);
    st.params.push_back(std::move(p));
    return static_cast<int>(st.params.size() - 1);
  };
  st.win = add_mat(weight_layout_for(kInputFeatureLayout), cfg.d_in, cfg.d_h);
  for (int l = 1; l <= cfg.layers; ++l) {
    st.wl.push_back(add_mat(weight_layout(l), cfg.d_h, cfg.d_h));
    if (cfg.use_rmsnorm) {
      const Layout out = feature_layout(l + 1);
      ParamSlot p;
      p.is_vec = true;
      p.row_axis = out.row;
      p.col_axis = out.col;
      const auto o = hoff(ctx, cfg.d_h, out.col);
      p.blk.lay = out;
      p.blk.g_rows = 1;
      p.blk.g_cols = cfg.d_h;
      p.blk.r0 = 0;
      p.blk.r1 = 1;
      p.blk.c0 = o[ctx.coord[out.col]];
      p.blk.c1 = o[ctx.coord[out.col] + 1];
      p.off = off;
      p.n = p.blk.cols();
      off += round_up(std::max<int64_t>(p.n, 1), 64);
      st.params.push_back(std::move(p));
      st.gamma.push_back(static_cast<int>(st.params.size() - 1));
    }
  }
  st.wout = add_mat(weight_layout_for(feature_layout(cfg.layers + 1)), cfg.d_h, cfg.d_out);
  st.total = off;
  float* W = st.W.reserve_n<float>(off);
  float* G = st.G.reserve_n<float>(off);
  float* M = st.M.reserve_n<float>(off);
  float* V = st.V.reserve_n<float>(off);
  GGB_CUDA(cudaMemsetAsync(W, 0, off * 4, ctx.stream));
  GGB_CUDA(cudaMemsetAsync(G, 0, off * 4, ctx.stream));
  GGB_CUDA(cudaMemsetAsync(M, 0, off * 4, ctx.stream));
  GGB_CUDA(cudaMemsetAsync(V, 0, off * 4, ctx.stream));
  auto init_mat = [&](int idx, uint64_t key) {
    ParamSlot& p = st.params[idx];
    init_weight(ctx, W + p.off, p.blk.rows(), p.blk.cols(), p.blk.g_rows, p.blk.g_cols, p.blk.r0, p.blk.c0, key);
  };
  init_mat(st.win, hash_combine(seed, 101));
  for (int l = 1; l <= cfg.layers; ++l) init_mat(st.wl[l - 1], hash_combine(seed, 200 + static_cast<uint64_t>(l)));
  for (int gi : st.gamma) fill(ctx, W + st.params[gi].off, st.params[gi].n, 1.0f);
  init_mat(st.wout, hash_combine(seed, 102));
  st.opt_step = 0;
  st.have_forward = false;
  for (auto& p : st.params)
    if (!p.is_vec) {
      p.wb.reserve_n<bf16>(std::max<int64_t>(p.blk.rows(), 1) * p.ldb);
      p.wt.reserve_n<bf16>(std::max<int64_t>(p.blk.cols(), 1) * p.ldt);
      p.wtl.reserve_n<bf16>(std::max<int64_t>(p.blk.cols(), 1) * p.ldt);
      GGB_CUDA(cudaMemsetAsync(p.wb.p, 0, p.wb.bytes, ctx.stream));
      GGB_CUDA(cudaMemsetAsync(p.wt.p, 0, p.wt.bytes, ctx.stream));
      GGB_CUDA(cudaMemsetAsync(p.wtl.p, 0, p.wtl.bytes, ctx.stream));
    }
  refresh_bf16(st);
}

void refresh_bf16(State& st) {
  Ctx& ctx = *st.ctx;
  for (auto& p : st.params)
    if (!p.is_vec)
      weight_bf16(ctx, st.W.as<float>() + p.off, p.blk.rows(), p.blk.cols(), p.wb.as<bf16>(), p.ldb,
                  p.wt.as<bf16>(), p.wtl.as<bf16>(), p.ldt);
}

namespace {

// Algorithmic traffic of one SpMM launch (SURVEY §8d gather model): the CSR
// (int32 col + fp32 val per nonzero, int64 row pointers), one e_in-byte
// feature row per nonzero, and the output rows (e_out bytes per element).
double spmm_bytes(int64_t rows, int64_t nnz, int64_t cols, int e_in, int e_out) {
  return static_cast<double>(nnz) * 8.0 + static_cast<double>(rows + 1) * 8.0 +
         static_cast<double>(nnz) * cols * e_in + static_cast<double>(rows) * cols * e_out;
}

double gemm_bytes(int64_t m, int64_t n, int64_t k, int ea, int eb, int ec) {
  return static_cast<double>(m) * k * ea + static_cast<double>(n) * k * eb + static_cast<double>(m) * n * ec;
}

// A producer's partial block for peer_all_reduce (comm.hpp): fp32, or bf16
// under the bf16 wire (the reference rounds every contribution to bf16 before
// summing, so the producer's RNE output is exactly that contribution and half
// the bytes cross NVLink).
struct PeerPart {
  void* p = nullptr;
  bool b16 = false;
  int64_t ld = 0;
  ptrdiff_t mirror = 0;  // push mode: byte distance to the peer's copy of the area (MirrorScope)
  float* f(int64_t r0 = 0) const { return b16 ? nullptr : static_cast<float*>(p) + r0 * ld; }
  bf16* h(int64_t r0 = 0) const { return b16 ? static_cast<bf16*>(p) + r0 * ld : nullptr; }
};
// push: the producer mirrors its output stores into the peer's slot
// (2-member groups), so the reduction reads only local HBM. Used for the
// SpMM producers, whose gather-bound runtime hides the NVLink stores (C2
// 1x2x2x1: SpMM +5%, reduction -40%); a GEMM producer is too short to hide
// them (its TMA stores to the peer run at NVLink speed: GEMM 0.07 -> 0.25 ms
// per launch), so GEMM sites pull unless GGB_PEER_PUSH_GEMM=1.
bool push_gemm() {
  static const bool on = [] {
    const char* e = std::getenv("GGB_PEER_PUSH_GEMM");
    return e && e[0] == '1';
  }();
  return on;
}
PeerPart peer_part(Ctx& ctx, int axis, int wire, int64_t rows, int64_t cols, bool push = false) {
  PeerPart pp;
  pp.b16 = wire == GGB_BF16_WIRE;
  pp.ld = ld8(cols);
  const size_t bytes = static_cast<size_t>(rows * pp.ld) * (pp.b16 ? 2 : 4);
  if (push) {
    const PeerSlot sl = peer_slot_push(ctx, axis, bytes, pp.b16);
    pp.p = sl.local;
    if (sl.mirror) pp.mirror = static_cast<char*>(sl.mirror) - static_cast<char*>(sl.local);
  } else {
    pp.p = peer_slot(ctx, axis, bytes);
  }
  return pp;
}

// C = A . W (forward contract): split-bf16 in the accurate mode, bf16 otherwise.
void fwd_gemm(State& st, int64_t m, int64_t n, int64_t k, const Tensor& a, const ParamSlot& w, float* c,
              int64_t ldc, bf16* cb, int64_t ldcb, bf16* cl = nullptr) {
  const int e = st.compute == kAccurate ? 4 : 2;
  // algorithmic flops 2mnk: the split form's 3 MMAs reproduce ONE fp32 product
  ProfScope ps(*st.ctx, kProfGemmFwd, gemm_bytes(m, n, k, e, e, (c ? 4 : 0) + (cb ? 2 : 0) + (cl ? 2 : 0)),
               2.0 * m * n * k);
  if (st.compute == kAccurate)
    gemm_split(*st.ctx, m, n, k, a.b, a.lo, a.ldb, w.wt.as<bf16>(), w.wtl.as<bf16>(), w.ldt, c, ldc, cb, ldcb, cl);
  else
    gemm_bf16(*st.ctx, m, n, k, a.b, a.ldb, w.wt.as<bf16>(), w.ldt, c, ldc, cb, ldcb);
}

}  // namespace

bool preagg_enabled() {
  const char* e = std::getenv("GGB_PREAGG");
  return !(e && e[0] == '0');
}

// GGB_GATHER24=1: the fused row kernel also writes a 24-bit copy of each
// layer's activations and the next forward SpMM gathers it (3 instead of 4
// bytes per element, 2^-16 relative like the split-bf16 GEMMs). Measured at
// C2: forward SpMM 2.75 -> 2.24 ms/step, but the step only 10.73 -> 10.60 ms
// (the sampling stream's batch build is the critical chain) and e2e 11.43 ->
// 11.66 ms (the extra write traffic lands on the build), so it is off.
bool gather24_enabled() {
  const char* e = std::getenv("GGB_GATHER24");
  return e && e[0] == '1';
}

bool preagg_in_prefetch() {
  const char* e = std::getenv("GGB_PREAGG_PF");
  return !(e && e[0] == '0');
}

// ---- forward (model.hpp:335-376) ----------------------------------------------------
void forward(State& st, const Batch& bt, int precision, bool training, uint64_t run_seed, uint64_t global_step,
             double eps) {
  Ctx& ctx = *st.ctx;
  const auto& cfg = st.cfg;
  require(precision >= GGB_FP32 && precision <= GGB_BF16_SUM, "forward: unknown precision");
  const int wire = precision;  // ggb_precision: the all-reduce wire mode
  const int64_t H = cfg.d_h;
  const int dp = ctx.coord[0];
  if (prof_of(ctx).on) settle_totals(bt);  // the kernel-class byte counts need the block sizes
  contract(bt.planes == std::min(cfg.layers, 3), "forward: batch planes do not match the model layers");
  float* W = st.W.as<float>();

  // X0 = x_in (X,Z) . W_in (Z,Y) -> (X,Y), all-reduce Z
  {
    const ParamSlot& w = st.params[st.win];
    Block ob = make_block(ctx, feature_layout(1), bt.b, H, bt.batch_off[feature_layout(1).row],
                          hoff(ctx, H, feature_layout(1).col));
    contract(ob.rows() == bt.x_r1 - bt.x_r0 && w.blk.rows() == bt.x_c1 - bt.x_c0,
             "contract: local inner blocks differ");
    st.x0.blk = ob;
    st.x0.ldf = ld8(ob.cols());
    st.x0.ldb = ld8(ob.cols());
    st.x0.f = grow<float>(st.x0_f, ob.rows() * st.x0.ldf);
    st.x0.p = nullptr;
    st.x0.b = grow<bf16>(st.x0_b, ob.rows() * st.x0.ldb);
    // accurate: X0 stays fp32 (the next SpMM gathers fp32); fast: + bf16 operand copy
    const bool want_b = st.compute != kAccurate;
    const bool ar = reduces(ctx, kInputFeatureLayout.col, wire);
    charge_all_reduce(ctx, kInputFeatureLayout.col, ob.rows() * ob.cols(), wire_bytes(wire));
    Tensor xin;
    xin.b = bt.x_in.as<bf16>();
    xin.lo = bt.x_in_lo.as<bf16>();
    xin.ldb = bt.x_ld;
    if (ar && peer_ok(ctx, kInputFeatureLayout.col, wire)) {
      // partial into the peer slot; the ordered sum lands in X0 (+ its bf16 copy)
      const int ax = kInputFeatureLayout.col;
      const PeerPart pp = peer_part(ctx, ax, wire, ob.rows(), ob.cols(), push_gemm());
      peer_pipelined(
          ctx, ob.rows(), 128,
          [&](int64_t r0, int64_t r1) {
            MirrorScope mirror(ctx, pp.mirror);
            Tensor sub = xin;
            sub.b = xin.b + r0 * xin.ldb;
            sub.lo = xin.lo ? xin.lo + r0 * xin.ldb : nullptr;
            fwd_gemm(st, r1 - r0, ob.cols(), w.blk.rows(), sub, w, pp.f(r0), pp.ld, pp.h(r0), pp.ld);
          },
          [&](int64_t r0, int64_t r1) {
            peer_all_reduce(ctx, ax, r1 - r0, ob.cols(), pp.ld, pp.b16, wire, st.x0.f + r0 * st.x0.ldf, st.x0.ldf,
                            want_b ? st.x0.b + r0 * st.x0.ldb : nullptr, nullptr, st.x0.ldb, nullptr, 0, r0);
          });
    } else {
    fwd_gemm(st, ob.rows(), ob.cols(), w.blk.rows(), xin, w, st.x0.f, st.x0.ldf, (ar || !want_b) ? nullptr : st.x0.b,
             st.x0.ldb);
    if (ar) {
      all_reduce_sum(ctx, kInputFeatureLayout.col, st.x0.f, ob.rows() * st.x0.ldf, wire);
      if (want_b) cast_bf16(ctx, st.x0.f, ob.rows(), ob.cols(), st.x0.ldf, st.x0.b, st.x0.ldb);
    }
    }
  }
  const bool accurate = st.compute == kAccurate;
  if (st.layers.size() < static_cast<size_t>(cfg.layers)) st.layers.resize(cfg.layers);
  const double rate = cfg.use_dropout ? cfg.dropout_rate : 0.0;
  const bool drop = training && rate > 0.0;
  st.fwd_drop = drop;
  st.fwd_keep_scale = drop ? static_cast<float>(1.0 / (1.0 - rate)) : 1.0f;
  const uint64_t thresh = drop ? static_cast<uint64_t>(std::ceil(rate * 0x1.0p53)) : 0;

  // layer 1 as (A_0 . x_in) . W_in: same product, d_in-wide instead of H-wide gathers
  // (not under a bf16 wire: it would skip the rounded X0 and hagg_1 intermediates)
  st.preagg = preagg_enabled() && preagg_eligible(ctx, bt) && wire == GGB_FP32;
  const Tensor* prev = &st.x0;
  for (int l = 1; l <= cfg.layers; ++l) {
    LayerBufs& L = st.layers[l - 1];
    const int p = (l - 1) % 3;
    const BatchCsr& A = bt.csrs[bt.csr_of[p]];
    const Layout alay = adjacency_layout(l);
    const Block& F = prev->blk;
    contract(alay.col == F.lay.row && A.c0 == F.r0 && A.c1 == F.r1, "spmm: inner partitions differ");
    // residual: X_{l-1} resharded to feature_layout(l+1); issued first so a
    // peer-memory reshard runs beside this layer's SpMM and GEMM (joined
    // before the fused row kernel reads it)
    const Layout out = feature_layout(l + 1);
    const float* res = nullptr;
    const uint8_t* resp = nullptr;  // X_{l-1} kept only as 24-bit rows
    int64_t ldres = 0;
    Block rb;
    if (cfg.use_residual) {
      rb = make_block(ctx, out, bt.b, H, bt.batch_off[out.row], hoff(ctx, H, out.col));
      charge_reshard(ctx, F, out);
      if (pmm_trivial(ctx)) {
        res = prev->f;
        ldres = prev->ldf;
        if (!res) resp = prev->p;
      } else {
        float* r = grow<float>(st.dres, rb.rows() * ld8(rb.cols()));
        reshard(ctx, F, bt.batch_off[F.lay.row], hoff(ctx, H, F.lay.col), prev->f, prev->ldf, rb,
                bt.batch_off[out.row], hoff(ctx, H, out.col), r, ld8(rb.cols()));
        res = r;
        ldres = ld8(rb.cols());
      }
    }
    // hagg = A . F -> (A.row, F.col), all-reduce A.col
    Block hb;
    hb.lay = {alay.row, F.lay.col};
    hb.g_rows = bt.b;
    hb.g_cols = H;
    hb.r0 = A.r0;
    hb.r1 = A.r1;
    hb.c0 = F.c0;
    hb.c1 = F.c1;
    L.hagg.blk = hb;
    L.hagg.ldb = ld8(hb.cols());
    L.hagg.b = grow<bf16>(L.hagg_b, hb.rows() * L.hagg.ldb);
    L.hagg.lo = accurate ? grow<bf16>(L.hagg_lo, hb.rows() * L.hagg.ldb) : nullptr;
    const bool ar_h = reduces(ctx, alay.col, wire);
    charge_all_reduce(ctx, alay.col, hb.rows() * hb.cols(), wire_bytes(wire));  // spmm (pmm.hpp:165)
    const int64_t* arp = A.row_ptr.as<int64_t>();
    LongRowsScope lrs(ctx, A.long_rows);
    if (l == 1 && st.preagg) {
      // hagg_1 = P . W_in with P = A_0 . x_in (built with the batch); X and Z
      // unsplit, so neither product needs an all-reduce
      if (!bt.p_ready) preaggregate(ctx, bt);
      const ParamSlot& wi = st.params[st.win];
      contract(wi.blk.c0 == hb.c0 && wi.blk.c1 == hb.c1 && wi.blk.rows() == bt.x_c1 - bt.x_c0,
               "contract: inner partitions differ");
      Tensor pt;
      pt.b = bt.p_in.as<bf16>();
      pt.lo = bt.p_in_lo.as<bf16>();
      pt.ldb = bt.x_ld;
      fwd_gemm(st, A.n_rows, hb.cols(), wi.blk.rows(), pt, wi, nullptr, 0, L.hagg.b, L.hagg.ldb, L.hagg.lo);
    } else {
    const int32_t* acol = A.col.as<int32_t>();
    const float* aval = A.val.as<float>();
    if (ar_h && peer_ok(ctx, alay.col, wire)) {
      // partial sums over A's column blocks into the peer slot; the ordered
      // sum is written as hagg's bf16 operand copies (no fp32 hagg, no cast pass)
      const PeerPart pp = peer_part(ctx, alay.col, wire, A.n_rows, hb.cols(), true);
      peer_pipelined(
          ctx, A.n_rows, 128,
          [&](int64_t r0, int64_t r1) {
            MirrorScope mirror(ctx, pp.mirror);
            const double frac = static_cast<double>(r1 - r0) / std::max<int64_t>(A.n_rows, 1);
            ProfScope ps(ctx, kProfSpmmFwd, frac * spmm_bytes(A.n_rows, A.nnz, F.cols(), accurate ? 4 : 2, pp.b16 ? 2 : 4),
                         frac * 2.0 * A.nnz * F.cols());
            if (accurate)
              spmm_csr_f32(ctx, r1 - r0, arp + r0, acol, aval, prev->f, prev->ldf, F.cols(), pp.f(r0), pp.ld, pp.h(r0),
                           nullptr, pp.ld, 0);
            else
              spmm_csr(ctx, r1 - r0, arp + r0, acol, aval, prev->b, prev->ldb, F.cols(), pp.f(r0), pp.ld, pp.h(r0),
                       pp.ld, 0);
          },
          [&](int64_t r0, int64_t r1) {
            peer_all_reduce(ctx, alay.col, r1 - r0, hb.cols(), pp.ld, pp.b16, wire, nullptr, 0,
                            L.hagg.b + r0 * L.hagg.ldb, L.hagg.lo ? L.hagg.lo + r0 * L.hagg.ldb : nullptr, L.hagg.ldb,
                            nullptr, 0, r0);
          });
    } else if (ar_h) {
      // partial sums over A's column blocks: row chunks of the SpMM pipelined
      // with their all-reduce (and the bf16 split of the reduced rows)
      L.hagg.ldf = ld8(hb.cols());
      L.hagg.f = grow<float>(L.hagg_f, hb.rows() * L.hagg.ldf);
      const int64_t ldf = L.hagg.ldf, ldb = L.hagg.ldb;
      pipelined_all_reduce(
          ctx, alay.col, A.n_rows, 128, L.hagg.f, ldf, wire,
          [&](int64_t r0, int64_t r1) {
            const double frac = static_cast<double>(r1 - r0) / std::max<int64_t>(A.n_rows, 1);
            ProfScope ps(ctx, kProfSpmmFwd, frac * spmm_bytes(A.n_rows, A.nnz, F.cols(), accurate ? 4 : 2, 4),
                         frac * 2.0 * A.nnz * F.cols());
            if (accurate)
              spmm_csr_f32(ctx, r1 - r0, arp + r0, acol, aval, prev->f, prev->ldf, F.cols(), L.hagg.f + r0 * ldf,
                           ldf, nullptr, nullptr, 0, 0);
            else
              spmm_csr(ctx, r1 - r0, arp + r0, acol, aval, prev->b, prev->ldb, F.cols(), L.hagg.f + r0 * ldf, ldf,
                       nullptr, 0, 0);
          },
          [&](int64_t r0, int64_t r1) {
            if (accurate)
              cast_split(ctx, L.hagg.f + r0 * ldf, r1 - r0, hb.cols(), ldf, L.hagg.b + r0 * ldb, L.hagg.lo + r0 * ldb,
                         ldb);
            else
              cast_bf16(ctx, L.hagg.f + r0 * ldf, r1 - r0, hb.cols(), ldf, L.hagg.b + r0 * ldb, ldb);
          });
    } else {
    // accurate: the gathered rows are the previous layer's 24-bit copies when
    // it wrote them (3 bytes per element instead of 4)
    const bool p24 = accurate && prev->p != nullptr;
    ProfScope ps(ctx, kProfSpmmFwd, spmm_bytes(A.n_rows, A.nnz, F.cols(), p24 ? 3 : (accurate ? 4 : 2), accurate ? 4 : 2),
                 2.0 * A.nnz * F.cols());
    if (accurate) {
      if (!(p24 && spmm_pipe_p24(ctx, A.n_rows, arp, acol, aval, prev->p, prev->ldp, F.cols(), L.hagg.b, L.hagg.lo,
                                 L.hagg.ldb)))
        spmm_csr_f32(ctx, A.n_rows, arp, acol, aval, prev->f, prev->ldf, F.cols(), nullptr, 0, L.hagg.b, L.hagg.lo,
                     L.hagg.ldb, 0);
    } else {
      spmm_csr(ctx, A.n_rows, arp, acol, aval, prev->b, prev->ldb, F.cols(), nullptr, 0, L.hagg.b, L.hagg.ldb, 0);
    }
    }
    }
    // xw = hagg . W_l -> (A.row, third), all-reduce F.col
    const ParamSlot& w = st.params[st.wl[l - 1]];
    contract(w.blk.lay.row == hb.lay.col && w.blk.r0 == hb.c0 && w.blk.r1 == hb.c1,
             "contract: inner partitions differ");
    Block xb;
    xb.lay = {hb.lay.row, w.blk.lay.col};
    xb.g_rows = bt.b;
    xb.g_cols = H;
    xb.r0 = hb.r0;
    xb.r1 = hb.r1;
    xb.c0 = w.blk.c0;
    xb.c1 = w.blk.c1;
    L.xw_t.blk = xb;
    L.xw_t.ldf = ld8(xb.cols());
    L.xw_t.f = grow<float>(L.xw, xb.rows() * L.xw_t.ldf);
    charge_all_reduce(ctx, hb.lay.col, xb.rows() * xb.cols(), wire_bytes(wire));  // contract (pmm.hpp:128)
    if (reduces(ctx, hb.lay.col, wire) && peer_ok(ctx, hb.lay.col, wire)) {
      const PeerPart pp = peer_part(ctx, hb.lay.col, wire, xb.rows(), xb.cols(), push_gemm());
      peer_pipelined(
          ctx, xb.rows(), 128,
          [&](int64_t r0, int64_t r1) {
            MirrorScope mirror(ctx, pp.mirror);
            Tensor sub = L.hagg;
            sub.b = L.hagg.b + r0 * L.hagg.ldb;
            sub.lo = L.hagg.lo ? L.hagg.lo + r0 * L.hagg.ldb : nullptr;
            fwd_gemm(st, r1 - r0, xb.cols(), hb.cols(), sub, w, pp.f(r0), pp.ld, pp.h(r0), pp.ld);
          },
          [&](int64_t r0, int64_t r1) {
            peer_all_reduce(ctx, hb.lay.col, r1 - r0, xb.cols(), pp.ld, pp.b16, wire, L.xw_t.f + r0 * L.xw_t.ldf,
                            L.xw_t.ldf, nullptr, nullptr, 0, nullptr, 0, r0);
          });
    } else {
    pipelined_all_reduce(ctx, hb.lay.col, xb.rows(), 128, L.xw_t.f, L.xw_t.ldf, wire, [&](int64_t r0, int64_t r1) {
      Tensor sub = L.hagg;
      sub.b = L.hagg.b + r0 * L.hagg.ldb;
      sub.lo = L.hagg.lo ? L.hagg.lo + r0 * L.hagg.ldb : nullptr;
      fwd_gemm(st, r1 - r0, xb.cols(), hb.cols(), sub, w, L.xw_t.f + r0 * L.xw_t.ldf, L.xw_t.ldf, nullptr, 0);
    });
    }
    // RMSNorm statistics: row sum of squares, all-reduce along the column axis (fp32)
    float* ss = nullptr;
    float* rms = nullptr;
    const float* gam = nullptr;
    const bool row_local = trivial(ctx, xb.lay.col);  // whole feature row on this rank
    if (cfg.use_rmsnorm) {
      ss = grow<float>(L.ss, xb.rows());
      rms = grow<float>(L.rms, xb.rows());
      charge_all_reduce(ctx, xb.lay.col, xb.rows(), 4);  // pmm.hpp:229
      if (!row_local) {  // partial sums of squares, all-reduced along the column axis
        ProfScope ps(ctx, kProfElementwise, 4.0 * xb.rows() * xb.cols());
        rowsumsq(ctx, L.xw_t.f, L.xw_t.ldf, xb.rows(), xb.cols(), ss);
        all_reduce_sum(ctx, xb.lay.col, ss, xb.rows(), false);
      }
      const ParamSlot& gp = st.params[st.gamma[l - 1]];
      contract(gp.blk.c0 == xb.c0 && gp.blk.c1 == xb.c1, "rmsnorm: gamma slice does not match the column block");
      gam = W + gp.off;
    }
    // residual X_{l-1} (resharded to feature_layout(l+1) at the top of the layer)
    if (cfg.use_residual)
      contract(rb.r0 == xb.r0 && rb.r1 == xb.r1 && rb.c0 == xb.c0 && rb.c1 == xb.c1,
               "fused_elementwise: residual layout mismatch");
    // fused RMSNorm apply + ReLU + dropout + residual -> X_l
    L.x.blk = xb;
    L.x.ldf = ld8(xb.cols());
    L.x.ldb = ld8(xb.cols());
    // bf16 copy: next SpMM operand (fast) and, for the last layer, the
    // out-head operand (hi + lo in the accurate mode) and dW_out operand; the
    // last layer's fp32 rows have no reader (no next SpMM, no residual), so
    // they are not written
    const bool last = l == cfg.layers;
    L.x.f = last ? nullptr : grow<float>(L.x_f, xb.rows() * L.x.ldf);
    L.x.b = (!accurate || last) ? grow<bf16>(L.x_b, xb.rows() * L.x.ldb) : nullptr;
    L.x.lo = (accurate && last) ? grow<bf16>(L.x_lo, xb.rows() * L.x.ldb) : nullptr;
    L.ldm = mask_words(std::max<int64_t>(xb.cols(), 1));
    FwdApply fa{};
    fa.fuse_ss = row_local ? 1 : 0;
    fa.rows = xb.rows();
    fa.cols = xb.cols();
    fa.x = L.xw_t.f;
    fa.ldx = L.xw_t.ldf;
    fa.ss = ss;
    fa.gamma = gam;
    fa.d = static_cast<float>(H);
    fa.eps = static_cast<float>(eps);
    fa.rms = rms;
    fa.res = res;
    fa.ldres = ldres;
    fa.resp = resp;
    fa.ldresp = resp ? prev->ldp : 0;
    fa.reshoff = resp ? prev->hoff : 0;
    fa.mask_key = dropout_key(run_seed, dp, global_step, l);
    fa.row_g0 = xb.r0;
    fa.col_g0 = xb.c0;
    fa.drop = drop;
    fa.thresh = thresh;
    fa.keep_scale = st.fwd_keep_scale;
    fa.out = L.x.f;  // null when only the 24-bit rows are kept (set below, before the launch)
    fa.ldo = L.x.ldf;
    fa.outb = L.x.b;
    fa.outlo = L.x.lo;
    fa.ldob = L.x.ldb;
    fa.mask = grow<uint32_t>(L.mask, xb.rows() * L.ldm);
    // 24-bit copy of X_l for the next layer's forward SpMM (its gathers are
    // the step's largest traffic) when that SpMM runs whole on this rank
    L.x.p = nullptr;
    if (accurate && !last && gather24_enabled() && xb.cols() <= 256 && !reduces(ctx, adjacency_layout(l + 1).col, wire) &&
        !ctx.side_stream) {
      const int64_t c16 = round_up(xb.cols(), 8);
      L.x.hoff = 2 * c16;
      L.x.ldp = round_up(3 * c16, 16);
      L.x.p = grow<uint8_t>(L.x_p, xb.rows() * L.x.ldp);
      // the 24-bit rows also serve as the next layer's residual when it is
      // not resharded: the fp32 copy of X_l then has no reader
      if (pmm_trivial(ctx) || !cfg.use_residual) L.x.f = nullptr;
    }
    fa.out = L.x.f;
    fa.outp = L.x.p;
    fa.ldp = L.x.ldp;
    fa.hoff = L.x.hoff;
    fa.ldm = L.ldm;
    fa.keep = nullptr;  // keep-bits precomputed by the prefetcher for exactly this block?
    if (drop && bt.masks.size() >= static_cast<size_t>(l)) {
      const DropMask& dm = bt.masks[l - 1];
      if (dm.key == fa.mask_key && dm.thresh == thresh && dm.r0 == xb.r0 && dm.c0 == xb.c0 &&
          dm.rows == xb.rows() && dm.cols == xb.cols() && dm.ldm == L.ldm)
        fa.keep = dm.bits.as<uint32_t>();
    }
    {
      const double e = static_cast<double>(xb.rows()) * xb.cols();
      ProfScope ps(ctx, kProfFwdRow,
                   e * (4 + (res ? 4 : resp ? 3 : 0) + (L.x.f ? 4 : 0) + (L.x.b ? 2 : 0) + (L.x.lo ? 2 : 0) +
                        (L.x.p ? 3 : 0)) + e / 8);
      reshard_join(ctx);
      fwd_apply(ctx, fa);
    }
    prev = &L.x;
  }
  // logits = X_L . W_out, all-reduce X_L.col
  {
    const ParamSlot& w = st.params[st.wout];
    const Block& F = prev->blk;
    contract(w.blk.lay.row == F.lay.col && w.blk.r0 == F.c0 && w.blk.r1 == F.c1, "contract: inner partitions differ");
    Block lb;
    lb.lay = {F.lay.row, w.blk.lay.col};
    lb.g_rows = bt.b;
    lb.g_cols = cfg.d_out;
    lb.r0 = F.r0;
    lb.r1 = F.r1;
    lb.c0 = w.blk.c0;
    lb.c1 = w.blk.c1;
    st.logits_blk = lb;
    float* lg = grow<float>(st.logits, lb.rows() * lb.cols());
    fwd_gemm(st, lb.rows(), lb.cols(), F.cols(), *prev, w, lg, lb.cols(), nullptr, 0);
    charge_all_reduce(ctx, F.lay.col, lb.rows() * lb.cols(), wire_bytes(wire));
    all_reduce_sum(ctx, F.lay.col, lg, lb.rows() * lb.cols(), wire);
  }
  st.have_forward = true;
}

// ---- parallel_cross_entropy (pmm.hpp:352-401) ---------------------------------------
void cross_entropy(State& st, const Batch& bt) {
  Ctx& ctx = *st.ctx;
  const Block& lb = st.logits_blk;
  CeArgs c{};
  c.rows = lb.rows();
  c.cols = lb.cols();
  c.logits = st.logits.as<float>();
  c.ld = lb.cols();
  c.labels = bt.labels.as<int32_t>();
  c.row_g0 = lb.r0;
  c.c0 = lb.c0;
  c.mx = grow<float>(st.ce_mx, c.rows);
  c.zt = grow<float>(st.ce_zt, 2 * c.rows);
  c.invb = 1.0f / static_cast<float>(lb.g_rows);
  c.dlogb = grow<bf16>(st.dlog_b, c.rows * ld8(c.cols));
  c.lddlogb = ld8(c.cols);
  c.loss_part = grow<float>(st.ce_part, ce_grad_blocks(c.rows) + 1);
  c.loss_acc = grow<float>(st.loss_acc, 1);
  charge_all_reduce(ctx, lb.lay.col, c.rows, 4);      // row max (pmm.hpp:368)
  charge_all_reduce(ctx, lb.lay.col, 2 * c.rows, 4);  // [sum exp, label logit] (pmm.hpp:381)
  charge_all_reduce(ctx, lb.lay.row, 1, 4);           // loss (pmm.hpp:398)
  if (trivial(ctx, lb.lay.col)) {  // class block complete here: one pass per row
    ProfScope ps(ctx, kProfCe, static_cast<double>(c.rows) * c.cols * (4 + 2));
    ce_fused(ctx, c);
  } else {
    ProfScope ps(ctx, kProfCe, static_cast<double>(c.rows) * c.cols * (3 * 4 + 2));
    ce_rowmax(ctx, c);
    all_reduce_max(ctx, lb.lay.col, c.mx, c.rows);
    ce_rowsum(ctx, c);
    all_reduce_sum(ctx, lb.lay.col, c.zt, 2 * c.rows, false);
    ce_grad(ctx, c);
  }
  all_reduce_sum(ctx, lb.lay.row, c.loss_acc, 1, false);
  scale_scalar(ctx, c.loss_acc, c.invb, grow<float>(st.loss, 1));
}

// ---- backward (model.hpp:378-420) ---------------------------------------------------
void backward(State& st, const Batch& bt, int precision) {
  Ctx& ctx = *st.ctx;
  const auto& cfg = st.cfg;
  contract(st.have_forward && st.layers.size() >= static_cast<size_t>(cfg.layers),
           "backward: cache does not match the model");
  const int wire = precision;  // ggb_precision: the all-reduce wire mode
  const int64_t H = cfg.d_h;
  float* W = st.W.as<float>();
  float* G = st.G.as<float>();
  GGB_CUDA(cudaMemsetAsync(G, 0, st.total * 4, ctx.stream));  // zero_grads (model.hpp:98-104)
  const Block& lb = st.logits_blk;
  const int64_t lddlog = ld8(lb.cols());
  const Tensor& XL = st.layers[cfg.layers - 1].x;

  // dW_out = X_L^T . dlogits, all-reduce X_L.row
  {
    const ParamSlot& w = st.params[st.wout];
    {
      ProfScope ps(ctx, kProfGemmWgrad, gemm_bytes(XL.blk.cols(), lb.cols(), lb.rows(), 2, 2, 4),
                   2.0 * lb.rows() * XL.blk.cols() * lb.cols());
      gemm_wgrad_bf16(ctx, lb.rows(), XL.blk.cols(), lb.cols(), XL.b, XL.ldb, st.dlog_b.as<bf16>(), lddlog,
                      G + w.off, w.blk.cols(), st.ws_wgrad);
    }
    charge_all_reduce(ctx, XL.blk.lay.row, w.n, wire_bytes(wire));
    all_reduce_sum_async(ctx, XL.blk.lay.row, G + w.off, w.n, wire);
  }
  // dxh = dlogits . W_out^T -> (X_L.row, X_L.col), all-reduce logits.col
  Block db = XL.blk;
  float* dxh = grow<float>(st.dxh, db.rows() * ld8(db.cols()));
  bool dxh_b_ready = false;  // bf16 copy of the final dxh already written
  {
    const ParamSlot& w = st.params[st.wout];
    ProfScope ps(ctx, kProfGemmDx, gemm_bytes(db.rows(), db.cols(), lb.cols(), 2, 2, 4),
                 2.0 * db.rows() * db.cols() * lb.cols());
    charge_all_reduce(ctx, lb.lay.col, db.rows() * db.cols(), wire_bytes(wire));
    if (reduces(ctx, lb.lay.col, wire) && peer_ok(ctx, lb.lay.col, wire)) {
      ps.end();
      const PeerPart pp = peer_part(ctx, lb.lay.col, wire, db.rows(), db.cols(), push_gemm());
      const int64_t ldd = ld8(db.cols());
      peer_pipelined(
          ctx, db.rows(), 128,
          [&](int64_t r0, int64_t r1) {
            MirrorScope mirror(ctx, pp.mirror);
            ProfScope pc(ctx, kProfGemmDx, gemm_bytes(r1 - r0, db.cols(), lb.cols(), 2, 2, pp.b16 ? 2 : 4),
                         2.0 * (r1 - r0) * db.cols() * lb.cols());
            gemm_bf16(ctx, r1 - r0, db.cols(), lb.cols(), st.dlog_b.as<bf16>() + r0 * lddlog, lddlog, w.wb.as<bf16>(),
                      w.ldb, pp.f(r0), pp.ld, pp.h(r0), pp.ld);
          },
          [&](int64_t r0, int64_t r1) {
            peer_all_reduce(ctx, lb.lay.col, r1 - r0, db.cols(), pp.ld, pp.b16, wire, dxh + r0 * ldd, ldd, nullptr,
                            nullptr, 0, nullptr, 0, r0);
          });
    } else {
    gemm_bf16(ctx, db.rows(), db.cols(), lb.cols(), st.dlog_b.as<bf16>(), lddlog, w.wb.as<bf16>(), w.ldb, dxh,
              ld8(db.cols()), nullptr, 0);
    ps.end();
    all_reduce_sum(ctx, lb.lay.col, dxh, db.rows() * ld8(db.cols()), wire);
    }
  }
  const bf16* pre_dhb = nullptr;  // layer 1 under pre-aggregation: dhagg_1 (bf16) and the residual gradient
  int64_t pre_ldhb = 0;
  const float* pre_dres = nullptr;
  for (int l = cfg.layers; l >= 1; --l) {
    LayerBufs& L = st.layers[l - 1];
    const Block& xb = L.xw_t.blk;  // == db
    contract(xb.lay == db.lay && xb.r0 == db.r0 && xb.c0 == db.c0, "backward: gradient layout mismatch");
    const int64_t rows = xb.rows(), cols = xb.cols();
    // residual gradient dres = reshard(dxh -> feature_layout(l))
    const Block& F = (l == 1) ? st.x0.blk : st.layers[l - 2].x.blk;
    float* dres = nullptr;
    if (cfg.use_residual) {
      charge_reshard(ctx, db, F.lay);
      if (pmm_trivial(ctx)) {
        dres = dxh;  // identical block; the SpMM below accumulates into it
      } else {
        dres = grow<float>(st.dres, F.rows() * ld8(F.cols()));
        reshard(ctx, db, bt.batch_off[db.lay.row], hoff(ctx, H, db.lay.col), dxh, ld8(db.cols()), F,
                bt.batch_off[F.lay.row], hoff(ctx, H, F.lay.col), dres, ld8(F.cols()));
      }
    }
    // fused element-wise backward + RMSNorm backward -> dxw (bf16), dgamma
    BwdApply ba{};
    ba.rows = rows;
    ba.cols = cols;
    ba.dy = dxh;
    ba.lddy = ld8(db.cols());
    ba.mask = L.mask.as<uint32_t>();
    ba.ldm = L.ldm;
    const bool row_local = trivial(ctx, xb.lay.col);
    ba.fuse_s = row_local ? 1 : 0;
    ba.keep_scale = st.fwd_keep_scale;
    ba.x = L.xw_t.f;
    ba.ldx = L.xw_t.ldf;
    ba.d = static_cast<float>(H);
    const int64_t lddxw = ld8(cols);
    ba.dxb = grow<bf16>(st.dxw_b, rows * lddxw);
    ba.lddxb = lddxw;
    {
    // reads dy + xw (once more for the row statistics when the row is split),
    // the keep bits, writes dxw bf16
    ProfScope ps(ctx, kProfBwdRow,
                 static_cast<double>(rows) * cols * ((row_local ? 8 : 16) + 2) + static_cast<double>(rows) * cols / 8.0);
    if (cfg.use_rmsnorm) {
      const ParamSlot& gp = st.params[st.gamma[l - 1]];
      ba.gamma = W + gp.off;
      ba.rms = L.rms.as<float>();
      ba.s = grow<float>(st.s_row, rows);
      charge_all_reduce(ctx, xb.lay.col, rows, 4);  // pmm.hpp:268
      charge_all_reduce(ctx, xb.lay.row, cols, 4);  // dgamma (pmm.hpp:285)
      if (!row_local) {
        bwd_stats(ctx, ba);
        all_reduce_sum(ctx, xb.lay.col, ba.s, rows, false);
      }
      const int blocks = bwd_apply_blocks(ctx, rows, cols);
      ba.dgamma_part = grow<float>(st.dg_part, static_cast<int64_t>(blocks) * cols);
      bwd_apply(ctx, ba, blocks);
      reduce_rows(ctx, ba.dgamma_part, blocks, cols, G + gp.off);
      all_reduce_sum_async(ctx, xb.lay.row, G + gp.off, cols, false);
    } else {
      bwd_apply(ctx, ba, bwd_apply_blocks(ctx, rows, cols));
    }
    }
    // dW_l = hagg^T . dxw, all-reduce hagg.row
    const ParamSlot& w = st.params[st.wl[l - 1]];
    const Tensor& hg = L.hagg;
    {
      ProfScope ps(ctx, kProfGemmWgrad, gemm_bytes(hg.blk.cols(), cols, rows, 2, 2, 4),
                   2.0 * rows * hg.blk.cols() * cols);
      gemm_wgrad_bf16(ctx, rows, hg.blk.cols(), cols, hg.b, hg.ldb, ba.dxb, lddxw, G + w.off, w.blk.cols(),
                      st.ws_wgrad);
    }
    charge_all_reduce(ctx, hg.blk.lay.row, w.n, wire_bytes(wire));
    all_reduce_sum_async(ctx, hg.blk.lay.row, G + w.off, w.n, wire);
    // dhagg = dxw . W_l^T -> (xw.row, hagg.col), all-reduce xw.col
    const int64_t hc = hg.blk.cols();
    const bool ar_d = reduces(ctx, xb.lay.col, wire);
    charge_all_reduce(ctx, xb.lay.col, rows * hc, wire_bytes(wire));
    const int64_t ldhb = ld8(hc);
    bf16* dhb = grow<bf16>(st.dhagg_b, rows * ldhb);
    {
    ProfScope ps(ctx, kProfGemmDx, gemm_bytes(rows, hc, cols, 2, 2, ar_d ? 4 : 2), 2.0 * rows * hc * cols);
    if (ar_d && peer_ok(ctx, xb.lay.col, wire)) {
      ps.end();
      const PeerPart pp = peer_part(ctx, xb.lay.col, wire, rows, hc, push_gemm());
      peer_pipelined(
          ctx, rows, 128,
          [&](int64_t r0, int64_t r1) {
            MirrorScope mirror(ctx, pp.mirror);
            ProfScope pc(ctx, kProfGemmDx, gemm_bytes(r1 - r0, hc, cols, 2, 2, pp.b16 ? 2 : 4), 2.0 * (r1 - r0) * hc * cols);
            gemm_bf16(ctx, r1 - r0, hc, cols, ba.dxb + r0 * lddxw, lddxw, w.wb.as<bf16>(), w.ldb, pp.f(r0), pp.ld,
                      pp.h(r0), pp.ld);
          },
          [&](int64_t r0, int64_t r1) {
            peer_all_reduce(ctx, xb.lay.col, r1 - r0, hc, pp.ld, pp.b16, wire, nullptr, 0, dhb + r0 * ldhb, nullptr,
                            ldhb, nullptr, 0, r0);
          });
    } else if (ar_d) {
      ps.end();
      float* dhf = grow<float>(st.dhagg_f, rows * hc);
      pipelined_all_reduce(
          ctx, xb.lay.col, rows, 128, dhf, hc, wire,
          [&](int64_t r0, int64_t r1) {
            ProfScope pc(ctx, kProfGemmDx, gemm_bytes(r1 - r0, hc, cols, 2, 2, 4), 2.0 * (r1 - r0) * hc * cols);
            gemm_bf16(ctx, r1 - r0, hc, cols, ba.dxb + r0 * lddxw, lddxw, w.wb.as<bf16>(), w.ldb, dhf + r0 * hc, hc,
                      nullptr, 0);
          },
          [&](int64_t r0, int64_t r1) { cast_bf16(ctx, dhf + r0 * hc, r1 - r0, hc, hc, dhb + r0 * ldhb, ldhb); });
    } else {
      gemm_bf16(ctx, rows, hc, cols, ba.dxb, lddxw, w.wb.as<bf16>(), w.ldb, nullptr, 0, dhb, ldhb);
    }
    }
    reshard_join(ctx);  // dres (its peer-memory reshard ran beside the element-wise backward and the GEMMs)
    // dxh = spmm(A_t, dhagg) (pmm.hpp:165), charged also when pre-aggregation folds it into dW_in
    charge_all_reduce(ctx, adjacency_layout(l).row, bt.csrs[bt.csrt_of[(l - 1) % 3]].n_rows * hc, wire_bytes(wire));
    if (l == 1 && st.preagg) {
      // layer 1 was (A_0 . x_in) . W_in: dX_0 is not formed; dW_in takes
      // P^T . dhagg_1 plus the residual term x_in^T . dres (below)
      pre_dhb = dhb;
      pre_ldhb = ldhb;
      pre_dres = dres;
      db = F;
      break;
    }
    // dxh = A_t . dhagg (+ dres) -> (A.col, hagg.col) = F's layout, all-reduce A.row
    const int p = (l - 1) % 3;
    const BatchCsr& At = bt.csrs[bt.csrt_of[p]];
    const Layout alay = adjacency_layout(l);
    contract(At.c0 == hg.blk.r0 && At.c1 == hg.blk.r1, "spmm: inner partitions differ");
    LongRowsScope lrs(ctx, At.long_rows);
    const bool inplace = pmm_trivial(ctx) && cfg.use_residual && wire == GGB_FP32;
    ProfScope ps(ctx, kProfSpmmBwd, spmm_bytes(At.n_rows, At.nnz, hc, 2, inplace ? 8 : 4), 2.0 * At.nnz * hc);
    if (inplace) {
      // dxh (== dres) += A_t . dhagg; the first layer also emits the bf16
      // copy that feeds dW_in (no separate cast pass)
      // (under pre-aggregation layer 2 emits it: its dX_1 is layer 1's residual gradient)
      const bool emit_b = st.preagg ? l == 2 : l == 1;
      bf16* outb = emit_b ? grow<bf16>(st.dxh_b, F.rows() * ld8(F.cols())) : nullptr;
      spmm_csr(ctx, At.n_rows, At.row_ptr.as<int64_t>(), At.col.as<int32_t>(), At.val.as<float>(), dhb, ldhb, hc,
               dxh, ld8(F.cols()), outb, ld8(F.cols()), 1);
      dxh_b_ready = emit_b;
    } else if (peer_ok(ctx, alay.row, wire) && reduces(ctx, alay.row, wire)) {
      // partial into the peer slot; ordered sum + residual gradient in one pass
      float* nd = grow<float>(st.dxh2, F.rows() * ld8(F.cols()));
      const int64_t ldn = ld8(F.cols());
      ps.end();
      const PeerPart pp = peer_part(ctx, alay.row, wire, At.n_rows, F.cols(), true);
      const int64_t* trp = At.row_ptr.as<int64_t>();
      peer_pipelined(
          ctx, At.n_rows, 128,
          [&](int64_t r0, int64_t r1) {
            MirrorScope mirror(ctx, pp.mirror);
            const double frac = static_cast<double>(r1 - r0) / std::max<int64_t>(At.n_rows, 1);
            ProfScope pc(ctx, kProfSpmmBwd, frac * spmm_bytes(At.n_rows, At.nnz, hc, 2, pp.b16 ? 2 : 4),
                         frac * 2.0 * At.nnz * hc);
            spmm_csr(ctx, r1 - r0, trp + r0, At.col.as<int32_t>(), At.val.as<float>(), dhb, ldhb, hc, pp.f(r0), pp.ld,
                     pp.h(r0), pp.ld, 0);
          },
          [&](int64_t r0, int64_t r1) {
            peer_all_reduce(ctx, alay.row, r1 - r0, F.cols(), pp.ld, pp.b16, wire, nd + r0 * ldn, ldn, nullptr, nullptr,
                            0, dres ? dres + r0 * ldn : nullptr, ldn, r0);
          });
      std::swap(st.dxh, st.dxh2);
      dxh = nd;
    } else {
      ps.end();
      float* nd = grow<float>(st.dxh2, F.rows() * ld8(F.cols()));
      const int64_t ldn = ld8(F.cols());
      const int64_t* trp = At.row_ptr.as<int64_t>();
      // row chunks of the SpMM pipelined with their all-reduce along A.row and the residual add
      pipelined_all_reduce(
          ctx, alay.row, At.n_rows, 128, nd, ldn, wire,
          [&](int64_t r0, int64_t r1) {
            const double frac = static_cast<double>(r1 - r0) / std::max<int64_t>(At.n_rows, 1);
            ProfScope pc(ctx, kProfSpmmBwd, frac * spmm_bytes(At.n_rows, At.nnz, hc, 2, 4), frac * 2.0 * At.nnz * hc);
            spmm_csr(ctx, r1 - r0, trp + r0, At.col.as<int32_t>(), At.val.as<float>(), dhb, ldhb, hc, nd + r0 * ldn,
                     ldn, nullptr, 0, 0);
          },
          [&](int64_t r0, int64_t r1) {
            if (dres) add_inplace(ctx, nd + r0 * ldn, ldn, dres + r0 * ldn, ldn, r1 - r0, F.cols());
          });
      std::swap(st.dxh, st.dxh2);
      dxh = nd;
    }
    db = F;
  }
  if (st.preagg) {
    // dW_in = x_in^T . dres + P^T . dhagg_1 (= x_in^T . (dres + A_0^T . dhagg_1)); X, Z unsplit
    const ParamSlot& w = st.params[st.win];
    const int64_t rows = db.rows(), cols = db.cols();
    const int64_t kin = bt.x_c1 - bt.x_c0;
    const BatchCsr& A0 = bt.csrs[bt.csr_of[0]];
    contract(rows == bt.x_r1 - bt.x_r0 && A0.n_rows == rows, "backward: first-layer blocks differ");
    ProfScope ps(ctx, kProfGemmWgrad, gemm_bytes(kin, cols, rows, 2, 2, 4) * (pre_dres ? 2 : 1),
                 2.0 * rows * kin * cols * (pre_dres ? 2 : 1));
    if (pre_dres) {
      const int64_t ldb = ld8(cols);
      bf16* drb = grow<bf16>(st.dxh_b, rows * ldb);
      if (!(dxh_b_ready && pre_dres == dxh)) cast_bf16(ctx, pre_dres, rows, cols, ld8(cols), drb, ldb);
      gemm_wgrad_bf16(ctx, rows, kin, cols, bt.x_in.as<bf16>(), bt.x_ld, drb, ldb, G + w.off, w.blk.cols(),
                      st.ws_wgrad, 0);
    }
    gemm_wgrad_bf16(ctx, rows, kin, cols, bt.p_in.as<bf16>(), bt.x_ld, pre_dhb, pre_ldhb, G + w.off, w.blk.cols(),
                    st.ws_wgrad, pre_dres ? 1 : 0);
    charge_all_reduce(ctx, kInputFeatureLayout.row, w.n, wire_bytes(wire));
    all_reduce_sum_async(ctx, kInputFeatureLayout.row, G + w.off, w.n, wire);
    reshard_join(ctx);
    join_async(ctx);  // every gradient reduced before dp_sync / the optimizer read G
    return;
  }
  // dW_in = x_in^T . dxh, all-reduce x_in.row (X)
  {
    const ParamSlot& w = st.params[st.win];
    const int64_t rows = db.rows(), cols = db.cols();
    const int64_t ldb = ld8(cols);
    bf16* dxb = grow<bf16>(st.dxh_b, rows * ldb);
    if (!dxh_b_ready) {
      ProfScope ps(ctx, kProfElementwise, static_cast<double>(rows) * cols * 6);
      cast_bf16(ctx, dxh, rows, cols, ld8(cols), dxb, ldb);
    }
    const int64_t kin = bt.x_c1 - bt.x_c0;
    ProfScope ps(ctx, kProfGemmWgrad, gemm_bytes(kin, cols, rows, 2, 2, 4), 2.0 * rows * kin * cols);
    gemm_wgrad_bf16(ctx, rows, kin, cols, bt.x_in.as<bf16>(), bt.x_ld, dxb, ldb, G + w.off, w.blk.cols(),
                    st.ws_wgrad);
    charge_all_reduce(ctx, kInputFeatureLayout.row, w.n, wire_bytes(wire));
    all_reduce_sum_async(ctx, kInputFeatureLayout.row, G + w.off, w.n, wire);
  }
  reshard_join(ctx);
  join_async(ctx);  // every gradient reduced before dp_sync / the optimizer read G
}

// ---- dp_sync (model.hpp:423-433) ------------------------------------------------------
void dp_sync(State& st) {
  Ctx& ctx = *st.ctx;
  const int gd = ctx.grid.dims[0];
  PhaseScope ps(ctx, kPhaseDpSync);
  for (const ParamSlot& p : st.params) charge_all_reduce(ctx, kD, p.n, 4);  // one all-reduce per view (model.hpp:428-429)
  all_reduce_sum(ctx, kD, st.G.as<float>(), st.total, false);
  if (gd > 1) scale(ctx, st.G.as<float>(), st.total, 1.0f / static_cast<float>(gd));
}

// ---- optimizer_step (model.hpp:435-456) -----------------------------------------------
void optimizer_step(State& st, int optimizer, double lr) {
  Ctx& ctx = *st.ctx;
  st.opt_step += 1;
  ProfScope ps(ctx, kProfOptimizer, static_cast<double>(st.total) * 4 * 7);
  if (optimizer == GGB_SGD) {
    sgd(ctx, st.W.as<float>(), st.G.as<float>(), st.total, static_cast<float>(lr));
  } else {
    const double bc1 = 1.0 - std::pow(0.9, static_cast<double>(st.opt_step));
    const double bc2 = 1.0 - std::pow(0.999, static_cast<double>(st.opt_step));
    adam(ctx, st.W.as<float>(), st.G.as<float>(), st.M.as<float>(), st.V.as<float>(), st.total, lr, bc1, bc2);
  }
  refresh_bf16(st);
}

}  // namespace ggb
