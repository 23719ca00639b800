// Kernel launchers (ops.cu, gemm.cu, spmm.cu) used by the trainer.
#pragma once

#include "runtime.hpp"

namespace ggb {

struct FwdApply {
  int64_t rows, cols;
  const float* x;  // xw (GEMM output), fp32 [rows][ldx]
  int64_t ldx;
  const float* ss;  // row sums of squares over the FULL feature dim (after all-reduce) or null
  const float* gamma;
  float d, eps;
  float* rms;        // out: per-row rms (nullable)
  const float* res;  // residual (nullable)
  int64_t ldres;
  const uint8_t* resp;  // or the residual as 24-bit rows (outp layout; nullable)
  int64_t ldresp, reshoff;
  uint64_t mask_key;
  int64_t row_g0, col_g0;  // global batch coordinates of this block
  int drop;
  uint64_t thresh;  // ceil(rate * 2^53)
  float keep_scale;
  float* out;  // fp32 output (nullable)
  int64_t ldo;
  bf16* outb;  // bf16 copy (nullable) = hi part of the split pair
  bf16* outlo; // bf16 lo part (nullable): out == hi + lo to ~2^-16
  int64_t ldob;
  uint8_t* outp;  // 24-bit copy for the next SpMM's gather (nullable): per row [hi16 x C16][lo8 x C16]
  int64_t ldp;    // its row stride in bytes
  int64_t hoff;   // byte offset of the lo8 plane (2 * C16)
  const uint32_t* keep;  // precomputed dropout keep-bits (same layout) or null: hash in-kernel
  uint32_t* mask;  // [rows][ldm] keep bits, row-kernel layout (see kRowChunk)
  int64_t ldm;     // words per row = mask_words(cols)
  int fuse_ss;     // 1: the row is complete here, compute ss in-kernel (ss ignored)
  int no_relu;     // 1: no ReLU (y passes; the layer API's RMSNorm alone)
};

// Row kernels: lane l of a warp owns columns c = 128*j + 4*l + i (i < 4) of
// its row (one float4 per chunk j); the keep mask of chunk j is 4 ballot
// words, word i holding bit l for column 128*j + 4*l + i.
constexpr int kRowChunk = 128;
inline int64_t mask_words(int64_t cols) { return 4 * ((cols + kRowChunk - 1) / kRowChunk); }

struct BwdApply {
  int64_t rows, cols;
  const float* dy;  // upstream gradient fp32
  int64_t lddy;
  const uint32_t* mask;  // keep bits; null: every element kept (RMSNorm backward alone)
  int64_t ldm;
  int fuse_s;  // 1: the row is complete here, compute s in-kernel
  float keep_scale;  // scale value of a kept element (1 without dropout)
  const float* x;    // xw
  int64_t ldx;
  const float* gamma;
  const float* rms;  // null: no rmsnorm
  float* s;          // row dot products (stats out / apply in)
  float d;
  bf16* dxb;  // out: dxw bf16 (nullable)
  int64_t lddxb;
  float* dxf;  // out: dxw fp32 (nullable; the layer API's parallel_rmsnorm_bwd)
  int64_t lddxf;
  float* dgamma_part;  // [blocks][cols] or null
};

struct CeArgs {
  int64_t rows, cols;
  const float* logits;
  int64_t ld;
  const int32_t* labels;  // full batch labels
  int64_t row_g0, c0;
  float* mx;         // [rows]
  float* zt;         // [2 rows]
  float invb;
  float* dlog;       // nullable fp32 grad
  int64_t lddlog;
  bf16* dlogb;       // nullable bf16 grad
  int64_t lddlogb;
  float* loss_part;  // [blocks]
  float* loss_acc;   // [1]
};

void init_weight(Ctx& ctx, float* w, int64_t rows, int64_t cols, int64_t g_rows, int64_t g_cols,
                 int64_t r0, int64_t c0, uint64_t key);
void fill(Ctx& ctx, float* x, int64_t n, float v);
void weight_bf16(Ctx& ctx, const float* w, int64_t rows, int64_t cols, bf16* wb, int64_t ldb, bf16* wt,
                 bf16* wt_lo, int64_t ldt);
void cast_bf16(Ctx& ctx, const float* x, int64_t rows, int64_t cols, int64_t ldx, bf16* y, int64_t ldy);
// y_hi = bf16(x), y_lo = bf16(x - y_hi)
void cast_split(Ctx& ctx, const float* x, int64_t rows, int64_t cols, int64_t ldx, bf16* hi, bf16* lo, int64_t ldy);
void add_inplace(Ctx& ctx, float* a, int64_t lda, const float* b, int64_t ldb, int64_t rows, int64_t cols);
void rowsumsq(Ctx& ctx, const float* x, int64_t ldx, int64_t rows, int64_t cols, float* ss);
void fwd_apply(Ctx& ctx, const FwdApply& p);
void bwd_stats(Ctx& ctx, const BwdApply& p);
int bwd_apply_blocks(Ctx& ctx, int64_t rows, int64_t cols);
void bwd_apply(Ctx& ctx, const BwdApply& p, int blocks);
void reduce_rows(Ctx& ctx, const float* part, int parts, int64_t cols, float* out);
void ce_rowmax(Ctx& ctx, const CeArgs& p);
void ce_rowsum(Ctx& ctx, const CeArgs& p);
int ce_grad_blocks(int64_t rows);
void ce_grad(Ctx& ctx, const CeArgs& p);
// all three cross-entropy passes in one warp-per-row kernel (row fully local)
void ce_fused(Ctx& ctx, const CeArgs& p);
// keep-bits of a rows x cols block at global (row_g0, col_g0), row-kernel layout
void dropout_keep(Ctx& ctx, uint64_t key, int64_t rows, int64_t cols, int64_t row_g0, int64_t col_g0,
                  uint64_t thresh, uint32_t* out, int64_t ldm);
void scale_scalar(Ctx& ctx, const float* in, float s, float* out);
void adam(Ctx& ctx, float* w, const float* g, float* m, float* v, int64_t n, double lr, double bc1,
          double bc2);
void sgd(Ctx& ctx, float* w, const float* g, int64_t n, float lr);
void scale(Ctx& ctx, float* x, int64_t n, float s);

// gemm.cu
void gemm_bf16(Ctx& ctx, int64_t m, int64_t n, int64_t k, const bf16* a, int64_t lda, const bf16* bt,
               int64_t ldb, float* c, int64_t ldc, bf16* cb, int64_t ldcb);
// split-bf16: fp32 operands carried as (hi, lo) bf16 pairs; 3 tcgen05 MMAs per k-step
void gemm_split(Ctx& ctx, int64_t m, int64_t n, int64_t k, const bf16* a_hi, const bf16* a_lo, int64_t lda,
                const bf16* bt_hi, const bf16* bt_lo, int64_t ldb, float* c, int64_t ldc, bf16* cb, int64_t ldcb,
                bf16* cl = nullptr);
void gemm_wgrad_bf16(Ctx& ctx, int64_t m, int64_t kw, int64_t nw, const bf16* x, int64_t ldx,
                     const bf16* dy, int64_t lddy, float* dw, int64_t lddw, DevBuf& ws, int accumulate = 0);
// spmm.cu
void spmm_csr(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
              const bf16* f, int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* outb,
              int64_t ldob, int accumulate);
// fp32 feature operand; optional split-bf16 (hi, lo) outputs
/// Forward SpMM over 24-bit rows (spmm_pipe.cu P24): out = A . F to the split
/// bf16 pair; false when the pipelined kernel does not apply (caller falls back).
bool spmm_pipe_p24(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
                   const uint8_t* f, int64_t ld_bytes, int64_t fcols, bf16* out_hi, bf16* out_lo, int64_t ldob);
void spmm_csr_f32(Ctx& ctx, int64_t rows, const int64_t* rp, const int32_t* col, const float* val,
                  const float* f, int64_t ldf, int64_t fcols, float* out, int64_t ldo, bf16* out_hi,
                  bf16* out_lo, int64_t ldob, int accumulate);

}  // namespace ggb
