// The reference's GCN layer operators (include/gridgnn/pmm.hpp:76-401) as C-ABI
// entry points over device blocks: contract, spmm, transposed, gather_full,
// reshard, parallel_rmsnorm_fwd/bwd, fused_elementwise_fwd/bwd,
// parallel_cross_entropy. A ggb_block carries a ShardedTensor's metadata
// (tensor.hpp:75-86: ordered layout, global shape, explicit row / column
// partition offsets) with this rank's block in HBM; each operator runs the same
// kernels and collectives as the fused training step (trainer.cu), with the
// reference's contract checks (CommContract -> GGB_ECONTRACT) and input checks
// (std::invalid_argument -> GGB_EINVAL).
#include <cmath>

#include "comm.hpp"
#include "layers.hpp"
#include "ops.hpp"
#include "trainer.hpp"

namespace ggb {
namespace {

struct View {
  Block blk;
  std::vector<int64_t> roff, coff;
};

View view(const Ctx& ctx, const ggb_block& t, const char* what) {
  require(t.row_axis >= kX && t.row_axis <= kZ && t.col_axis >= kX && t.col_axis <= kZ && t.row_axis != t.col_axis,
          "Layout: axes must be distinct PMM axes");
  require(t.row_off && t.col_off, (std::string(what) + ": null partition offsets").c_str());
  View v;
  const int gr = ctx.grid.dims[t.row_axis], gc = ctx.grid.dims[t.col_axis];
  v.roff.assign(t.row_off, t.row_off + gr + 1);
  v.coff.assign(t.col_off, t.col_off + gc + 1);
  require(v.roff.front() == 0 && v.roff.back() == t.g_rows, "ShardedTensor: bad row partition offsets");
  require(v.coff.front() == 0 && v.coff.back() == t.g_cols, "ShardedTensor: bad col partition offsets");
  for (int i = 0; i < gr; ++i) require(v.roff[i] <= v.roff[i + 1], "ShardedTensor: bad row partition offsets");
  for (int i = 0; i < gc; ++i) require(v.coff[i] <= v.coff[i + 1], "ShardedTensor: bad col partition offsets");
  v.blk = make_block(ctx, {t.row_axis, t.col_axis}, t.g_rows, t.g_cols, v.roff, v.coff);
  require(t.ld >= v.blk.cols(), (std::string(what) + ": leading dimension below the block width").c_str());
  return v;
}

View view_csr(const Ctx& ctx, const ggb_csr_block& a) {
  ggb_block t{};
  t.row_axis = a.row_axis;
  t.col_axis = a.col_axis;
  t.g_rows = a.g_rows;
  t.g_cols = a.g_cols;
  t.row_off = a.row_off;
  t.col_off = a.col_off;
  t.ld = a.g_cols;
  return view(ctx, t, "spmm");
}

bool same_meta(const View& a, const View& b) {
  return a.blk.lay == b.blk.lay && a.blk.g_rows == b.blk.g_rows && a.blk.g_cols == b.blk.g_cols && a.roff == b.roff &&
         a.coff == b.coff;
}

inline int64_t ld8(int64_t c) { return round_up(std::max<int64_t>(c, 1), 8); }
inline int wire_bytes(int wire) { return wire == GGB_FP32 ? 4 : 2; }

// B (k x n, ldb) -> its transpose as a split-bf16 pair [n][ldt] (hi = bf16(b), lo = bf16(b - hi))
__global__ void k_transpose_split(const float* __restrict__ b, int64_t k, int64_t n, int64_t ldb, bf16* __restrict__ hi,
                                  bf16* __restrict__ lo, int64_t ldt) {
  __shared__ float tile[32][33];
  const int64_t k0 = static_cast<int64_t>(blockIdx.y) * 32, n0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t kk = k0 + i, nn = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (kk < k && nn < n) ? b[kk * ldb + nn] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t nn = n0 + i, kk = k0 + threadIdx.x;
    if (nn < n && kk < ldt) {
      const float x = tile[threadIdx.x][i];
      const bf16 h = __float2bfloat16_rn(x);
      hi[nn * ldt + kk] = h;
      lo[nn * ldt + kk] = __float2bfloat16_rn(x - __bfloat162float(h));
    }
  }
}

// out (n x k, ldo) = B^T, fp32 (transposed)
__global__ void k_transpose_f32(const float* __restrict__ b, int64_t k, int64_t n, int64_t ldb, float* __restrict__ out,
                                int64_t ldo) {
  __shared__ float tile[32][33];
  const int64_t k0 = static_cast<int64_t>(blockIdx.y) * 32, n0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t kk = k0 + i, nn = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (kk < k && nn < n) ? b[kk * ldb + nn] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t nn = n0 + i, kk = k0 + threadIdx.x;
    if (nn < n && kk < k) out[nn * ldo + kk] = tile[threadIdx.x][i];
  }
}

// dx = dy * (keep ? keep_scale : 0) is k_bwd_row without RMSNorm; a tiny
// kernel keeps the layer API independent of the row kernels' width limits
__global__ void k_masked_scale(const float* __restrict__ dy, int64_t lddy, const uint32_t* __restrict__ mask,
                               int64_t ldm, int64_t rows, int64_t cols, float keep_scale, float* __restrict__ dx,
                               int64_t lddx) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= rows * cols) return;
  const int64_t r = t / cols, c = t % cols;
  // row-kernel mask layout: word 4j+i, bit l <-> column 128j + 4l + i
  const int64_t j = c / kRowChunk, l = (c % kRowChunk) / 4, i = c % 4;
  const bool keep = (mask[r * ldm + 4 * j + i] >> l) & 1u;
  dx[r * lddx + c] = keep ? dy[r * lddy + c] * keep_scale : 0.f;
}

// fp32 rows padded to 16-byte multiples (what the row / SpMM kernels read),
// or the caller's buffer when it already is
struct Staged {
  DevBuf buf;
  float* p = nullptr;
  int64_t ld = 0;
};
void stage_in(Ctx& ctx, const float* src, int64_t ld, int64_t rows, int64_t cols, Staged& s) {
  if (ld % 8 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    s.p = const_cast<float*>(src);
    s.ld = ld;
    return;
  }
  s.ld = ld8(cols);
  s.p = s.buf.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(rows, 1) * s.ld));
  GGB_CUDA(cudaMemsetAsync(s.p, 0, static_cast<size_t>(std::max<int64_t>(rows, 1) * s.ld) * 4, ctx.stream));
  if (rows > 0 && cols > 0)
    GGB_CUDA(cudaMemcpy2DAsync(s.p, s.ld * 4, src, ld * 4, cols * 4, rows, cudaMemcpyDeviceToDevice, ctx.stream));
}
void copy_out(Ctx& ctx, const float* src, int64_t lds, float* dst, int64_t ldd, int64_t rows, int64_t cols) {
  if (src == dst || rows <= 0 || cols <= 0) return;
  GGB_CUDA(cudaMemcpy2DAsync(dst, ldd * 4, src, lds * 4, cols * 4, rows, cudaMemcpyDeviceToDevice, ctx.stream));
}

}  // namespace

// contract (pmm.hpp:97-130): C = A . B, all-reduce along A's column axis.
void layer_contract(Ctx& ctx, const ggb_block& a, const ggb_block& b, const ggb_block& c, int wire) {
  const View A = view(ctx, a, "contract"), B = view(ctx, b, "contract"), Cv = view(ctx, c, "contract");
  contract(a.col_axis == b.row_axis, "contract: inner axes differ");
  contract(a.g_cols == b.g_rows, "contract: inner dimensions differ");
  contract(A.coff == B.roff, "contract: inner partitions differ");
  contract(a.row_axis != b.col_axis, "contract: output axes collide");
  contract(A.blk.cols() == B.blk.rows(), "contract: local inner blocks differ");
  contract(c.row_axis == a.row_axis && c.col_axis == b.col_axis && c.g_rows == a.g_rows && c.g_cols == b.g_cols &&
               Cv.roff == A.roff && Cv.coff == B.coff,
           "contract: output block does not match (A.row, B.col)");
  const int64_t m = A.blk.rows(), k = A.blk.cols(), n = B.blk.cols(), ldk = ld8(k), ldn = ld8(n);
  DevBuf ah, al, bh, bl, cc;
  bf16* a_hi = ah.reserve_n<bf16>(static_cast<size_t>(std::max<int64_t>(m, 1) * ldk));
  bf16* a_lo = al.reserve_n<bf16>(static_cast<size_t>(std::max<int64_t>(m, 1) * ldk));
  bf16* b_hi = bh.reserve_n<bf16>(static_cast<size_t>(std::max<int64_t>(n, 1) * ldk));
  bf16* b_lo = bl.reserve_n<bf16>(static_cast<size_t>(std::max<int64_t>(n, 1) * ldk));
  float* cbuf = cc.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(m, 1) * ldn));
  GGB_CUDA(cudaMemsetAsync(cbuf, 0, static_cast<size_t>(std::max<int64_t>(m, 1) * ldn) * 4, ctx.stream));
  if (m > 0 && n > 0 && k > 0) {
    GGB_CUDA(cudaMemsetAsync(a_hi, 0, static_cast<size_t>(m * ldk) * 2, ctx.stream));
    GGB_CUDA(cudaMemsetAsync(a_lo, 0, static_cast<size_t>(m * ldk) * 2, ctx.stream));
    cast_split(ctx, a.data, m, k, a.ld, a_hi, a_lo, ldk);
    const dim3 grid(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(ldk, 32)));
    k_transpose_split<<<grid, dim3(32, 8), 0, ctx.stream>>>(b.data, k, n, b.ld, b_hi, b_lo, ldk);
    GGB_LAUNCH_CHECK();
    ctx.launches += 1;
    // split-bf16 on tcgen05: fp32-accurate to ~2^-16 (3 MMAs per k-step)
    gemm_split(ctx, m, n, k, a_hi, a_lo, ldk, b_hi, b_lo, ldk, cbuf, ldn, nullptr, 0);
  }
  charge_all_reduce(ctx, a.col_axis, m * n, wire_bytes(wire));
  all_reduce_sum(ctx, a.col_axis, cbuf, m * ldn, wire);
  copy_out(ctx, cbuf, ldn, c.data, c.ld, m, n);
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));  // before the temporaries are released
}

// spmm (pmm.hpp:134-167): H = A . F (A's fp32 values), all-reduce along A's column axis.
void layer_spmm(Ctx& ctx, const ggb_csr_block& a, const ggb_block& f, const ggb_block& h, int wire) {
  const View A = view_csr(ctx, a), F = view(ctx, f, "spmm"), Hv = view(ctx, h, "spmm");
  contract(a.col_axis == f.row_axis, "spmm: inner axes differ");
  contract(a.g_cols == f.g_rows, "spmm: inner dimensions differ");
  contract(A.coff == F.roff, "spmm: inner partitions differ");
  contract(h.row_axis == a.row_axis && h.col_axis == f.col_axis && h.g_rows == a.g_rows && h.g_cols == f.g_cols &&
               Hv.roff == A.roff && Hv.coff == F.coff,
           "spmm: output block does not match (A.row, F.col)");
  const int64_t m = A.blk.rows(), n = F.blk.cols();
  Staged fs;
  stage_in(ctx, f.data, f.ld, F.blk.rows(), n, fs);
  DevBuf hb;
  const int64_t ldn = ld8(n);
  float* hbuf = hb.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(m, 1) * ldn));
  GGB_CUDA(cudaMemsetAsync(hbuf, 0, static_cast<size_t>(std::max<int64_t>(m, 1) * ldn) * 4, ctx.stream));
  if (m > 0 && n > 0) {
    LongRowsScope lrs(ctx, true);  // any row-length profile
    spmm_csr_f32(ctx, m, a.row_ptr, a.col, a.val, fs.p, fs.ld, n, hbuf, ldn, nullptr, nullptr, 0, 0);
  }
  charge_all_reduce(ctx, a.col_axis, m * n, wire_bytes(wire));
  all_reduce_sum(ctx, a.col_axis, hbuf, m * ldn, wire);
  copy_out(ctx, hbuf, ldn, h.data, h.ld, m, n);
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
}

// reshard (pmm.hpp:197-204) as a block permutation; an unchanged layout copies.
void layer_reshard(Ctx& ctx, const ggb_block& src, const ggb_block& dst) {
  const View S = view(ctx, src, "reshard"), D = view(ctx, dst, "reshard");
  contract(src.g_rows == dst.g_rows && src.g_cols == dst.g_cols, "reshard: global shapes differ");
  if (same_meta(S, D)) {
    copy_out(ctx, src.data, src.ld, dst.data, dst.ld, S.blk.rows(), S.blk.cols());
    return;
  }
  reshard_block(ctx, S.blk, S.roff, S.coff, src.data, src.ld, D.blk, D.roff, D.coff, dst.data, dst.ld);
}

// gather_full (pmm.hpp:171-195): the global matrix on every rank of the group,
// each block sent once per replica set (as reshard's pieces)
void layer_gather_full(Ctx& ctx, const ggb_block& src, float* full, int64_t ldf) {
  const View S = view(ctx, src, "gather_full");
  const Grid& G = ctx.grid;
  int mc[4];
  G.coord_of(ctx.rank, mc);
  const Layout sl = S.blk.lay;
  const int rep = third_axis(sl);
  std::vector<BlockXfer> sends, recvs;
  for (int i = 0; i + 1 < static_cast<int>(S.roff.size()); ++i)
    for (int j = 0; j + 1 < static_cast<int>(S.coff.size()); ++j) {
      const int64_t r0 = S.roff[i], r1 = S.roff[i + 1], c0 = S.coff[j], c1 = S.coff[j + 1];
      if (r0 >= r1 || c0 >= c1) continue;
      int pc[4] = {mc[0], mc[1], mc[2], mc[3]};
      pc[sl.row] = i;
      pc[sl.col] = j;
      const int p = G.rank_of(pc);
      float* out = full + r0 * ldf + c0;
      if (p == ctx.rank)
        copy_out(ctx, src.data, src.ld, out, ldf, r1 - r0, c1 - c0);
      else
        recvs.push_back({p, out, ldf, r1 - r0, c1 - c0});
    }
  if (S.blk.rows() > 0 && S.blk.cols() > 0)
    for (int q = 0; q < G.total(); ++q) {
      int qc[4];
      G.coord_of(q, qc);
      if (q == ctx.rank || qc[0] != mc[0] || qc[rep] != mc[rep]) continue;
      sends.push_back({q, src.data, src.ld, S.blk.rows(), S.blk.cols()});
    }
  charge_all_gather(ctx, sl.row, static_cast<uint64_t>(S.blk.g_rows) * S.blk.cols() * 4);
  charge_all_gather(ctx, sl.col, static_cast<uint64_t>(S.blk.g_rows) * S.blk.g_cols * 4);
  exchange_blocks(ctx, sends, recvs);
}

// transposed (pmm.hpp:76-92): the transposed shard's local block (fp32).
void layer_transposed(Ctx& ctx, const ggb_block& t, const ggb_block& out) {
  const View T = view(ctx, t, "transposed"), O = view(ctx, out, "transposed");
  contract(out.row_axis == t.col_axis && out.col_axis == t.row_axis && out.g_rows == t.g_cols &&
               out.g_cols == t.g_rows && O.roff == T.coff && O.coff == T.roff,
           "transposed: output block is not the transposed shard");
  const int64_t k = T.blk.rows(), n = T.blk.cols();
  if (k <= 0 || n <= 0) return;
  const dim3 grid(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(k, 32)));
  k_transpose_f32<<<grid, dim3(32, 8), 0, ctx.stream>>>(t.data, k, n, t.ld, out.data, out.ld);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

// parallel_rmsnorm_fwd (pmm.hpp:214-243)
void layer_rmsnorm_fwd(Ctx& ctx, const ggb_block& x, const float* gamma, double eps, const ggb_block& y, float* rms) {
  const View X = view(ctx, x, "rmsnorm"), Y = view(ctx, y, "rmsnorm");
  contract(same_meta(X, Y), "rmsnorm: output block differs from the input block");
  const int64_t m = X.blk.rows(), n = X.blk.cols();
  if (m <= 0) return;
  require(n <= 512, "rmsnorm: at most 512 local columns");
  Staged xs;
  stage_in(ctx, x.data, x.ld, m, n, xs);
  Staged ys;
  stage_in(ctx, y.data, y.ld, m, n, ys);
  DevBuf ssb;
  float* ss = ssb.reserve_n<float>(static_cast<size_t>(m));
  const bool row_local = trivial(ctx, x.col_axis);
  charge_all_reduce(ctx, x.col_axis, m, 4);
  if (!row_local) {
    rowsumsq(ctx, xs.p, xs.ld, m, n, ss);
    all_reduce_sum(ctx, x.col_axis, ss, m, GGB_FP32);
  }
  FwdApply p{};
  p.rows = m;
  p.cols = n;
  p.x = xs.p;
  p.ldx = xs.ld;
  p.ss = ss;
  p.fuse_ss = row_local ? 1 : 0;
  p.gamma = gamma;
  p.d = static_cast<float>(x.g_cols);
  p.eps = static_cast<float>(eps);
  p.rms = rms;
  p.no_relu = 1;
  p.keep_scale = 1.f;
  p.out = ys.p;
  p.ldo = ys.ld;
  p.ldm = mask_words(n);
  fwd_apply(ctx, p);
  copy_out(ctx, ys.p, ys.ld, y.data, y.ld, m, n);
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
}

// parallel_rmsnorm_bwd (pmm.hpp:251-287)
void layer_rmsnorm_bwd(Ctx& ctx, const ggb_block& x, const float* gamma, const float* rms, const ggb_block& dy,
                       const ggb_block& dx, float* dgamma) {
  const View X = view(ctx, x, "rmsnorm_bwd"), DY = view(ctx, dy, "rmsnorm_bwd"), DX = view(ctx, dx, "rmsnorm_bwd");
  contract(DY.blk.lay == X.blk.lay && DY.blk.r0 == X.blk.r0 && DY.blk.c0 == X.blk.c0 && same_meta(X, DX),
           "rmsnorm_bwd: gradient layout mismatch");
  const int64_t m = X.blk.rows(), n = X.blk.cols();
  require(n <= 512, "rmsnorm: at most 512 local columns");
  Staged xs, dys, dxs;
  stage_in(ctx, x.data, x.ld, m, n, xs);
  stage_in(ctx, dy.data, dy.ld, m, n, dys);
  stage_in(ctx, dx.data, dx.ld, m, n, dxs);
  const bool row_local = trivial(ctx, x.col_axis);
  DevBuf sb, part;
  BwdApply p{};
  p.rows = m;
  p.cols = n;
  p.dy = dys.p;
  p.lddy = dys.ld;
  p.fuse_s = row_local ? 1 : 0;
  p.keep_scale = 1.f;
  p.x = xs.p;
  p.ldx = xs.ld;
  p.gamma = gamma;
  p.rms = rms;
  p.s = sb.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(m, 1)));
  p.d = static_cast<float>(x.g_cols);
  p.dxf = dxs.p;
  p.lddxf = dxs.ld;
  charge_all_reduce(ctx, x.col_axis, m, 4);
  charge_all_reduce(ctx, x.row_axis, n, 4);
  GGB_CUDA(cudaMemsetAsync(dgamma, 0, static_cast<size_t>(std::max<int64_t>(n, 0)) * 4, ctx.stream));
  if (m > 0) {
    if (!row_local) {
      bwd_stats(ctx, p);
      all_reduce_sum(ctx, x.col_axis, p.s, m, GGB_FP32);
    }
    const int blocks = bwd_apply_blocks(ctx, m, n);
    p.dgamma_part = part.reserve_n<float>(static_cast<size_t>(blocks) * n);
    bwd_apply(ctx, p, blocks);
    reduce_rows(ctx, p.dgamma_part, blocks, n, dgamma);
  }
  all_reduce_sum(ctx, x.row_axis, dgamma, n, GGB_FP32);
  copy_out(ctx, dxs.p, dxs.ld, dx.data, dx.ld, m, n);
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
}

// fused_elementwise_fwd (pmm.hpp:299-328): out = x * scale + h_prev with scale
// = (x > 0) * (training && rate > 0 ? keep(key, row, col) / (1 - rate) : 1); the
// keep bits of scale != 0 are written in the row-kernel layout (mask_words)
void layer_fused_fwd(Ctx& ctx, const ggb_block& x, const ggb_block* h_prev, double rate, uint64_t key, int training,
                     const ggb_block& out, uint32_t* keep_bits) {
  require(rate >= 0.0 && rate < 1.0, "fused_elementwise: dropout rate must be in [0, 1)");
  const View X = view(ctx, x, "fused_elementwise"), O = view(ctx, out, "fused_elementwise");
  contract(same_meta(X, O), "fused_elementwise: output block differs from the input block");
  const int64_t m = X.blk.rows(), n = X.blk.cols();
  Staged rs;
  if (h_prev) {
    const View R = view(ctx, *h_prev, "fused_elementwise");
    contract(R.blk.lay == X.blk.lay && R.blk.r0 == X.blk.r0 && R.blk.c0 == X.blk.c0 && R.blk.r1 == X.blk.r1 &&
                 R.blk.c1 == X.blk.c1,
             "fused_elementwise: residual layout mismatch");
    stage_in(ctx, h_prev->data, h_prev->ld, m, n, rs);
  }
  if (m <= 0) return;
  require(n <= 512, "fused_elementwise: at most 512 local columns");
  Staged xs, os;
  stage_in(ctx, x.data, x.ld, m, n, xs);
  stage_in(ctx, out.data, out.ld, m, n, os);
  const bool drop = training && rate > 0.0;
  FwdApply p{};
  p.rows = m;
  p.cols = n;
  p.x = xs.p;
  p.ldx = xs.ld;
  p.fuse_ss = 1;
  p.res = h_prev ? rs.p : nullptr;
  p.ldres = rs.ld;
  p.mask_key = key;
  p.row_g0 = X.blk.r0;
  p.col_g0 = X.blk.c0;
  p.drop = drop;
  p.thresh = drop ? static_cast<uint64_t>(std::ceil(rate * 0x1.0p53)) : 0;
  p.keep_scale = drop ? static_cast<float>(1.0 / (1.0 - rate)) : 1.0f;
  p.out = os.p;
  p.ldo = os.ld;
  p.mask = keep_bits;
  p.ldm = mask_words(n);
  fwd_apply(ctx, p);
  copy_out(ctx, os.p, os.ld, out.data, out.ld, m, n);
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
}

// fused_elementwise_bwd (pmm.hpp:331-341): dx = dy * scale from the keep bits
void layer_fused_bwd(Ctx& ctx, const ggb_block& dy, const uint32_t* keep_bits, float keep_scale,
                     const ggb_block& dx) {
  const View DY = view(ctx, dy, "fused_elementwise_bwd"), DX = view(ctx, dx, "fused_elementwise_bwd");
  contract(same_meta(DY, DX), "fused_elementwise_bwd: missing cache");
  const int64_t m = DY.blk.rows(), n = DY.blk.cols();
  if (m <= 0 || n <= 0) return;
  const float ks = keep_scale;
  k_masked_scale<<<static_cast<unsigned>(ceil_div(m * n, 256)), 256, 0, ctx.stream>>>(
      dy.data, dy.ld, keep_bits, mask_words(n), m, n, ks, dx.data, dx.ld);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

// parallel_cross_entropy (pmm.hpp:352-401): loss (device scalar, replicated)
// and grad_logits = (softmax - onehot) / B
void layer_cross_entropy(Ctx& ctx, const ggb_block& logits, const int32_t* labels, float* loss,
                         const ggb_block& grad) {
  const View L = view(ctx, logits, "cross_entropy"), G = view(ctx, grad, "cross_entropy");
  contract(same_meta(L, G), "cross_entropy: gradient block differs from the logits block");
  const int64_t m = L.blk.rows(), n = L.blk.cols();
  DevBuf mx, zt, part, acc;
  CeArgs c{};
  c.rows = m;
  c.cols = n;
  c.logits = logits.data;
  c.ld = logits.ld;
  c.labels = labels;
  c.row_g0 = L.blk.r0;
  c.c0 = L.blk.c0;
  c.mx = mx.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(m, 1)));
  c.zt = zt.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(2 * m, 1)));
  c.invb = 1.0f / static_cast<float>(logits.g_rows);
  c.dlog = grad.data;
  c.lddlog = grad.ld;
  c.loss_part = part.reserve_n<float>(static_cast<size_t>(ce_grad_blocks(std::max<int64_t>(m, 1)) + 1));
  c.loss_acc = acc.reserve_n<float>(1);
  GGB_CUDA(cudaMemsetAsync(c.loss_acc, 0, 4, ctx.stream));
  charge_all_reduce(ctx, logits.col_axis, m, 4);
  charge_all_reduce(ctx, logits.col_axis, 2 * m, 4);
  charge_all_reduce(ctx, logits.row_axis, 1, 4);
  if (m > 0) {
    if (trivial(ctx, logits.col_axis) && n <= 512) {
      ce_fused(ctx, c);
    } else {
      ce_rowmax(ctx, c);
      all_reduce_max(ctx, logits.col_axis, c.mx, m);
      ce_rowsum(ctx, c);
      all_reduce_sum(ctx, logits.col_axis, c.zt, 2 * m, GGB_FP32);
      ce_grad(ctx, c);
    }
  }
  all_reduce_sum(ctx, logits.row_axis, c.loss_acc, 1, GGB_FP32);
  scale_scalar(ctx, c.loss_acc, c.invb, loss);
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));  // the temporaries above are freed on return
}

}  // namespace ggb
