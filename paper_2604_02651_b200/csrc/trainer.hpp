// ModelState and the training step (model.hpp:60-478) on the device.
#pragma once

#include "ops.hpp"

namespace ggb {

/// One rank's block of a 2D-sharded matrix (ShardedTensor metadata,
/// tensor.hpp:75-86).
struct Block {
  Layout lay{kX, kY};
  int64_t g_rows = 0, g_cols = 0, r0 = 0, r1 = 0, c0 = 0, c1 = 0;
  int64_t rows() const { return r1 - r0; }
  int64_t cols() const { return c1 - c0; }
};

Block make_block(const Ctx& ctx, Layout lay, int64_t g_rows, int64_t g_cols,
                 const std::vector<int64_t>& row_off, const std::vector<int64_t>& col_off);

struct ParamSlot {
  bool is_vec = false;
  Block blk;       // matrices: layout + ranges; vectors: c0/c1 (rows = 1)
  int row_axis = 0, col_axis = 0;  // vectors: VecParam axes (model.hpp:70-76)
  int64_t off = 0, n = 0;          // into the flat W/G/M/V arrays
  int64_t ldb = 0, ldt = 0;        // bf16 copies: wb [rows][ldb], wt (+ lo) [cols][ldt]
  DevBuf wb, wt, wtl;
};

struct Tensor {  // device activation block: fp32 and/or bf16 copy (+ lo of the split pair)
  Block blk;
  float* f = nullptr;
  int64_t ldf = 0;
  bf16* b = nullptr;
  bf16* lo = nullptr;
  int64_t ldb = 0;
  uint8_t* p = nullptr;  // 24-bit gather copy (spmm_pipe.cu P24): row stride ldp bytes, lo plane at hoff
  int64_t ldp = 0, hoff = 0;
};

/// Compute precision of the forward pass. kAccurate (default): fp32
/// activations, fp32 SpMM gathers and split-bf16 (hi+lo, 3 MMAs) tensor-core
/// GEMMs, so ReLU / dropout decisions match the fp32 reference; the backward
/// pass runs on bf16 operands either way. kFast: bf16 operands throughout.
enum Compute : int { kAccurate = 0, kFast = 1 };

struct LayerBufs {
  DevBuf hagg_f, hagg_b, hagg_lo, xw, ss, rms, mask, x_f, x_b, x_lo, x_p;
  Tensor hagg, xw_t, x;  // x = layer output X_l
  int64_t ldm = 0;
};

struct State {
  Ctx* ctx = nullptr;
  ggb_model_config cfg{};
  uint64_t seed = 0;
  int compute = kAccurate;
  std::vector<ParamSlot> params;  // param_views order
  int win = 0, wout = 0;
  std::vector<int> wl, gamma;
  int64_t total = 0;
  DevBuf W, G, M, V;  // flat fp32
  int64_t opt_step = 0;
  // activations (grow-only)
  DevBuf x0_f, x0_b, logits, dlog_b, ce_mx, ce_zt, ce_part, loss_acc, loss;
  DevBuf dxh, dxh_b, dxh2, dxw_b, dhagg_f, dhagg_b, s_row, dg_part, ws_wgrad, dres, tmp;
  std::vector<LayerBufs> layers;
  Tensor x0;
  Block logits_blk;
  bool fwd_drop = false;
  float fwd_keep_scale = 1.f;
  bool have_forward = false;
  bool preagg = false;  // the last forward computed layer 1 as (A_0 . x_in) . W_in
};

/// First-layer pre-aggregation switch (GGB_PREAGG=0 turns it off); applied
/// where preagg_eligible() holds.
bool preagg_enabled();
/// ... computed by the prefetcher with the batch (GGB_PREAGG_PF=0: lazily by forward)
bool preagg_in_prefetch();

/// reshard (pmm.hpp:197-204) as a block permutation: this rank's block of src
/// (layout sb, offsets s_roff / s_coff) to its block of the new layout db.
void reshard_block(Ctx& ctx, const Block& sb, const std::vector<int64_t>& s_roff, const std::vector<int64_t>& s_coff,
                   const float* src, int64_t lds, const Block& db, const std::vector<int64_t>& d_roff,
                   const std::vector<int64_t>& d_coff, float* dst, int64_t ldd);
void state_init(Ctx& ctx, State& st, const ggb_model_config& cfg, uint64_t seed);
void refresh_bf16(State& st);
void forward(State& st, const Batch& bt, int precision, bool training, uint64_t run_seed,
             uint64_t global_step, double eps);
void cross_entropy(State& st, const Batch& bt);
void backward(State& st, const Batch& bt, int precision);
void dp_sync(State& st);
void optimizer_step(State& st, int optimizer, double lr);
// evaluate_full_graph (model.hpp:493-537); counts = {correct train/val/test, total train/val/test}
void evaluate_full_graph(State& st, const Batch& eval, const Graph& g, int precision, double eps,
                         uint64_t counts[6]);

}  // namespace ggb
