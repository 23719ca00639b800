#include "comm.hpp"
#include "prof.hpp"

#include <nccl.h>

#include <cstring>

namespace ggb {
namespace {

#define GGB_NCCL(call)                                                                          \
  do {                                                                                          \
    ncclResult_t r_ = (call);                                                                   \
    if (r_ != ncclSuccess)                                                                      \
      ::ggb::fail(GGB_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_) + " at " +      \
                                 __FILE__ + ":" + std::to_string(__LINE__));                    \
  } while (0)

__global__ void k_to_bf16(const float* __restrict__ in, int64_t n, bf16* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __float2bfloat16_rn(in[i]);
}

// out[i] = 0 + c_0[i] + c_1[i] + ... in ascending member order (comm.hpp:282-295)
__global__ void k_ordered_sum_bf16(const bf16* __restrict__ parts, int g, int64_t n, float* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int k = 0; k < g; ++k) s += __bfloat162float(parts[k * n + i]);
  out[i] = s;
}

ncclComm_t as_nccl(void* p) { return static_cast<ncclComm_t>(p); }

void need(const Ctx& ctx, int axis) {
  if (!ctx.comm || !ctx.comm->axis[axis])
    fail(GGB_ECONTRACT, "collective over a multi-rank group on a context without communicators");
}

}  // namespace

Comm::~Comm() {
  for (auto& a : axis)
    if (a) ncclCommDestroy(as_nccl(a));
  if (world) ncclCommDestroy(as_nccl(world));
}

int comm_get_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  GGB_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
  return 0;
}

std::unique_ptr<Comm> comm_create(const Grid& grid, int rank, const uint8_t* uid) {
  auto c = std::make_unique<Comm>();
  ncclUniqueId id;
  std::memcpy(&id, uid, 128);
  ncclComm_t world;
  GGB_NCCL(ncclCommInitRank(&world, grid.total(), id, rank));
  c->world = world;
  int co[4];
  grid.coord_of(rank, co);
  for (int a = 0; a < 4; ++a) {
    c->size[a] = grid.dims[a];
    c->pos[a] = co[a];
    // every rank takes part in every split (ncclCommSplit is collective on world)
    ncclComm_t sub = nullptr;
    const int colour = grid.dims[a] > 1 ? grid.group_id(a, rank) : NCCL_SPLIT_NOCOLOR;
    GGB_NCCL(ncclCommSplit(world, colour, co[a], &sub, nullptr));
    if (grid.dims[a] > 1) c->axis[a] = sub;
  }
  // NCCL connects point-to-point peers lazily, on their first send/recv; the
  // reshard's block permutation meets new peer pairs in later steps, so one
  // tiny exchange with every peer here keeps that setup (tens of ms) out of
  // the training steps
  const int n = grid.total();
  if (n > 1) {
    float* buf = nullptr;
    GGB_CUDA(cudaMalloc(&buf, sizeof(float) * 2 * n));
    GGB_CUDA(cudaMemset(buf, 0, sizeof(float) * 2 * n));
    GGB_NCCL(ncclGroupStart());
    for (int p = 0; p < n; ++p) {
      if (p == rank) continue;
      GGB_NCCL(ncclSend(buf + p, 1, ncclFloat32, p, world, nullptr));
      GGB_NCCL(ncclRecv(buf + n + p, 1, ncclFloat32, p, world, nullptr));
    }
    GGB_NCCL(ncclGroupEnd());
    GGB_CUDA(cudaDeviceSynchronize());
    GGB_CUDA(cudaFree(buf));
  }
  return c;
}

void all_reduce_sum(Ctx& ctx, int axis, float* buf, int64_t count, bool bf16_wire) {
  if (trivial(ctx, axis) || count <= 0) return;
  need(ctx, axis);
  Comm& c = *ctx.comm;
  const int gg = c.size[axis];
  // bytes one rank sends: ring all-reduce 2(g-1)/g of the fp32 buffer; bf16 wire: its bf16 contribution to g-1 peers
  ProfScope ps(ctx, kProfComm, bf16_wire ? 2.0 * count * (gg - 1) : 2.0 * (gg - 1) / gg * count * 4);
  if (!bf16_wire) {
    GGB_NCCL(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclFloat32, ncclSum,
                           as_nccl(c.axis[axis]), ctx.stream));
    return;
  }
  const int g = c.size[axis];
  bf16* mine = c.wire.reserve_n<bf16>(static_cast<size_t>(count));
  bf16* all = c.gather.reserve_n<bf16>(static_cast<size_t>(count) * g);
  const unsigned blocks = static_cast<unsigned>(ceil_div(count, 256));
  k_to_bf16<<<blocks, 256, 0, ctx.stream>>>(buf, count, mine);
  GGB_NCCL(ncclAllGather(mine, all, static_cast<size_t>(count), ncclBfloat16, as_nccl(c.axis[axis]),
                         ctx.stream));
  k_ordered_sum_bf16<<<blocks, 256, 0, ctx.stream>>>(all, g, count, buf);
  GGB_LAUNCH_CHECK();
  ctx.launches += 2;
}

void all_reduce_max(Ctx& ctx, int axis, float* buf, int64_t count) {
  if (trivial(ctx, axis) || count <= 0) return;
  need(ctx, axis);
  GGB_NCCL(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclFloat32, ncclMax,
                         as_nccl(ctx.comm->axis[axis]), ctx.stream));
}

void all_reduce_u64(Ctx& ctx, int axis, uint64_t* buf, int64_t count) {
  if (trivial(ctx, axis) || count <= 0) return;
  need(ctx, axis);
  GGB_NCCL(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclUint64, ncclSum,
                         as_nccl(ctx.comm->axis[axis]), ctx.stream));
}

void all_gather(Ctx& ctx, int axis, const float* in, int64_t count, float* out) {
  if (trivial(ctx, axis)) {
    if (count > 0)
      GGB_CUDA(cudaMemcpyAsync(out, in, count * 4, cudaMemcpyDeviceToDevice, ctx.stream));
    return;
  }
  need(ctx, axis);
  GGB_NCCL(ncclAllGather(in, out, static_cast<size_t>(count), ncclFloat32,
                         as_nccl(ctx.comm->axis[axis]), ctx.stream));
}

void exchange_blocks(Ctx& ctx, const std::vector<BlockXfer>& sends, const std::vector<BlockXfer>& recvs) {
  if (sends.empty() && recvs.empty()) return;
  if (!ctx.comm) fail(GGB_ECONTRACT, "block exchange on a context without communicators");
  Comm& c = *ctx.comm;
  int64_t ns = 0, nr = 0;
  for (const auto& x : sends) ns += x.rows * x.cols;
  for (const auto& x : recvs) nr += x.rows * x.cols;
  ProfScope ps(ctx, kProfComm, 4.0 * ns);
  float* sbuf = c.wire.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(ns, 1)));
  float* rbuf = c.gather.reserve_n<float>(static_cast<size_t>(std::max<int64_t>(nr, 1)));
  int64_t off = 0;
  for (const auto& x : sends) {
    if (x.rows * x.cols == 0) continue;
    GGB_CUDA(cudaMemcpy2DAsync(sbuf + off, x.cols * 4, x.ptr, x.ld * 4, x.cols * 4, x.rows,
                               cudaMemcpyDeviceToDevice, ctx.stream));
    off += x.rows * x.cols;
  }
  GGB_NCCL(ncclGroupStart());
  off = 0;
  for (const auto& x : sends) {
    const int64_t n = x.rows * x.cols;
    if (n == 0) continue;
    GGB_NCCL(ncclSend(sbuf + off, static_cast<size_t>(n), ncclFloat32, x.peer, as_nccl(c.world), ctx.stream));
    off += n;
  }
  off = 0;
  for (const auto& x : recvs) {
    const int64_t n = x.rows * x.cols;
    if (n == 0) continue;
    GGB_NCCL(ncclRecv(rbuf + off, static_cast<size_t>(n), ncclFloat32, x.peer, as_nccl(c.world), ctx.stream));
    off += n;
  }
  GGB_NCCL(ncclGroupEnd());
  off = 0;
  for (const auto& x : recvs) {
    if (x.rows * x.cols == 0) continue;
    GGB_CUDA(cudaMemcpy2DAsync(x.ptr, x.ld * 4, rbuf + off, x.cols * 4, x.cols * 4, x.rows,
                               cudaMemcpyDeviceToDevice, ctx.stream));
    off += x.rows * x.cols;
  }
}

void barrier(Ctx& ctx) {
  if (ctx.grid.total() == 1) return;
  if (!ctx.comm) fail(GGB_ECONTRACT, "barrier on a context without communicators");
  float* one = ctx.comm->gather.reserve_n<float>(1);
  GGB_NCCL(ncclAllReduce(one, one, 1, ncclFloat32, ncclSum, as_nccl(ctx.comm->world), ctx.stream));
  GGB_CUDA(cudaStreamSynchronize(ctx.stream));
}

}  // namespace ggb
