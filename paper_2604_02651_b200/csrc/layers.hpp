// Layer operators of the C ABI (layers.cu; pmm.hpp:76-401).
#pragma once

#include "runtime.hpp"

namespace ggb {

void layer_contract(Ctx& ctx, const ggb_block& a, const ggb_block& b, const ggb_block& c, int wire);
void layer_spmm(Ctx& ctx, const ggb_csr_block& a, const ggb_block& f, const ggb_block& h, int wire);
void layer_transposed(Ctx& ctx, const ggb_block& t, const ggb_block& out);
void layer_gather_full(Ctx& ctx, const ggb_block& t, float* full, int64_t ldf);
void layer_reshard(Ctx& ctx, const ggb_block& src, const ggb_block& dst);
void layer_rmsnorm_fwd(Ctx& ctx, const ggb_block& x, const float* gamma, double eps, const ggb_block& y, float* rms);
void layer_rmsnorm_bwd(Ctx& ctx, const ggb_block& x, const float* gamma, const float* rms, const ggb_block& dy,
                       const ggb_block& dx, float* dgamma);
void layer_fused_fwd(Ctx& ctx, const ggb_block& x, const ggb_block* h_prev, double rate, uint64_t key, int training,
                     const ggb_block& out, uint32_t* keep_bits);
void layer_fused_bwd(Ctx& ctx, const ggb_block& dy, const uint32_t* keep_bits, float keep_scale,
                     const ggb_block& dx);
void layer_cross_entropy(Ctx& ctx, const ggb_block& logits, const int32_t* labels, float* loss, const ggb_block& grad);

}  // namespace ggb
