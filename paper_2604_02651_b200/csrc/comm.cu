#include "comm.hpp"
#include "prof.hpp"

#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <thread>

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
__global__ void k_from_bf16(const bf16* __restrict__ in, int64_t n, float* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __bfloat162float(in[i]);
}

// bf16_round (comm.hpp:29-39) as integer arithmetic: RNE to 8 exponent + 7
// fraction bits; Inf/NaN truncated, NaN keeps a payload bit
__device__ __forceinline__ float bf16_round_ref(float x) {
  const uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) == 0x7f800000u) {
    uint32_t r = u & 0xffff0000u;
    if ((u & 0x007fffffu) != 0 && (r & 0x007f0000u) == 0) r |= 0x00400000u;
    return __uint_as_float(r);
  }
  return __uint_as_float((u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u);
}

// a one-member group's kBf16Roundtrip all-reduce: out = 0 + bf16_round(x)
// (Channel::rendezvous runs the same compute for size 1, comm.hpp:135-145)
__global__ void k_round_bf16_inplace(float* __restrict__ buf, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = 0.0f + bf16_round_ref(buf[i]);
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

// CTAs of an axis collective = SMs the persistent kernels leave it while overlapped
int comm_ctas() {
  static int v = [] {
    const char* e = std::getenv("GGB_COMM_CTAS");
    const int c = e ? std::atoi(e) : 16;
    return c >= 1 && c <= 64 ? c : 16;
  }();
  return v;
}

int comm_chunks() {
  static int v = [] {
    const char* e = std::getenv("GGB_COMM_CHUNKS");
    const int c = e ? std::atoi(e) : 1;
    return c >= 1 && c <= 16 ? c : 1;
  }();
  return v;
}

void need(const Ctx& ctx, int axis) {
  if (ctx.comm && ctx.comm->aborted)
    fail(GGB_ETIMEOUT, "communicators were aborted after a collective timed out or failed");
  if (!ctx.comm || !ctx.comm->axis[axis])
    fail(GGB_ECONTRACT, "collective over a multi-rank group on a context without communicators");
}

}  // namespace

Comm::~Comm() {
  if (pstream) cudaStreamDestroy(pstream);
  for (auto& e : pev) cudaEventDestroy(e);
  if (rstream) cudaStreamDestroy(rstream);
  if (rfork) cudaEventDestroy(rfork);
  if (rjoin) cudaEventDestroy(rjoin);
  if (gstream) cudaStreamDestroy(gstream);
  if (gfork) cudaEventDestroy(gfork);
  if (gjoin) cudaEventDestroy(gjoin);
  for (auto& e : ev) cudaEventDestroy(e);
  if (cstream) cudaStreamDestroy(cstream);
  for (auto& a : axis)
    if (a) ncclCommDestroy(as_nccl(a));
  if (pmm) ncclCommDestroy(as_nccl(pmm));
  if (world) ncclCommDestroy(as_nccl(world));
}

namespace {
void abort_all(Comm& c) {
  for (auto& a : c.axis)
    if (a) {
      ncclCommAbort(as_nccl(a));
      a = nullptr;
    }
  if (c.pmm) {
    ncclCommAbort(as_nccl(c.pmm));
    c.pmm = nullptr;
  }
  if (c.world) {
    ncclCommAbort(as_nccl(c.world));
    c.world = nullptr;
  }
  c.aborted = true;
}
}  // namespace

void sync_stream(Ctx& ctx, cudaStream_t s) {
  if (!ctx.comm || ctx.comm->aborted) {
    GGB_CUDA(cudaStreamSynchronize(s));
    return;
  }
  Comm& c = *ctx.comm;
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(s);
    if (peer_timed_out(c)) {  // a peer-memory reduction gave up waiting for a member
      abort_all(c);
      fail(GGB_ETIMEOUT, "collective timed out: not all group members arrived");
    }
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) GGB_CUDA(q);
    void* comms[6] = {c.world, c.axis[0], c.axis[1], c.axis[2], c.axis[3], c.pmm};
    for (void* k : comms) {
      if (!k) continue;
      ncclResult_t st = ncclSuccess;
      if (ncclCommGetAsyncError(as_nccl(k), &st) == ncclSuccess && st != ncclSuccess && st != ncclInProgress) {
        const std::string why = ncclGetErrorString(st);
        abort_all(c);
        fail(GGB_ENCCL, "collective failed on a peer (" + why + "); communicators aborted");
      }
    }
    const auto ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    if (ms > c.timeout_ms) {
      abort_all(c);
      fail(GGB_ETIMEOUT, "collective timed out: not all group members arrived");
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(spin > 4096 ? 500 : 20));
  }
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
  if (const char* e = std::getenv("GGB_COMM_TIMEOUT_MS")) {
    const long long v = std::atoll(e);
    if (v > 0) c->timeout_ms = v;
  }
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
    // axis collectives run beside the persistent kernels (pipelined_all_reduce):
    // a bounded CTA count, matching the SMs those kernels leave free
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (comm_chunks() > 1) cfg.maxCTAs = comm_ctas();
    GGB_NCCL(ncclCommSplit(world, colour, co[a], &sub, &cfg));
    if (grid.dims[a] > 1) c->axis[a] = sub;
  }
  {  // the DP group's PMM grid (peer-memory reshards)
    const int p = grid.dims[1] * grid.dims[2] * grid.dims[3];
    ncclComm_t sub = nullptr;
    GGB_NCCL(ncclCommSplit(world, p > 1 ? co[0] : NCCL_SPLIT_NOCOLOR, rank % p, &sub, nullptr));
    if (p > 1) c->pmm = sub;
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
    // collectives connect their rings / trees on first use too, with a host
    // handshake between the members: one tiny all-reduce per communicator
    // here, so no step (and no collective watchdog wait) pays for it
    GGB_NCCL(ncclAllReduce(buf, buf, 1, ncclFloat32, ncclSum, world, nullptr));
    for (int a = 0; a < 4; ++a)
      if (c->axis[a]) GGB_NCCL(ncclAllReduce(buf, buf, 1, ncclFloat32, ncclSum, as_nccl(c->axis[a]), nullptr));
    if (c->pmm) GGB_NCCL(ncclAllReduce(buf, buf, 1, ncclFloat32, ncclSum, as_nccl(c->pmm), nullptr));
    GGB_CUDA(cudaDeviceSynchronize());
    GGB_CUDA(cudaFree(buf));
  }
  return c;
}

namespace {
void all_reduce_sum_on(Ctx& ctx, int axis, float* buf, int64_t count, int mode, cudaStream_t s, DevBuf& wire,
                       DevBuf& gather) {
  Comm& c = *ctx.comm;
  const int gg = c.size[axis];
  // bytes one rank sends: ring all-reduce 2(g-1)/g of the buffer (fp32 or bf16); exact bf16 wire: its bf16
  // contribution to g-1 peers
  const double sent = mode == 1 ? 2.0 * count * (gg - 1) : 2.0 * (gg - 1) / gg * count * (mode == 2 ? 2 : 4);
  ProfScope ps(ctx, kProfComm, sent, 0, s);
  if (mode == 0) {
    GGB_NCCL(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclFloat32, ncclSum, as_nccl(c.axis[axis]), s));
    return;
  }
  if (mode == 2) {
    bf16* w = wire.reserve_n<bf16>(static_cast<size_t>(count));
    const unsigned blocks = static_cast<unsigned>(ceil_div(count, 256));
    k_to_bf16<<<blocks, 256, 0, s>>>(buf, count, w);
    GGB_NCCL(ncclAllReduce(w, w, static_cast<size_t>(count), ncclBfloat16, ncclSum, as_nccl(c.axis[axis]), s));
    k_from_bf16<<<blocks, 256, 0, s>>>(w, count, buf);
    GGB_LAUNCH_CHECK();
    ctx.launches += 2;
    return;
  }
  bf16* mine = wire.reserve_n<bf16>(static_cast<size_t>(count));
  bf16* all = gather.reserve_n<bf16>(static_cast<size_t>(count) * gg);
  const unsigned blocks = static_cast<unsigned>(ceil_div(count, 256));
  k_to_bf16<<<blocks, 256, 0, s>>>(buf, count, mine);
  GGB_NCCL(ncclAllGather(mine, all, static_cast<size_t>(count), ncclBfloat16, as_nccl(c.axis[axis]), s));
  k_ordered_sum_bf16<<<blocks, 256, 0, s>>>(all, gg, count, buf);
  GGB_LAUNCH_CHECK();
  ctx.launches += 2;
}
}  // namespace

// GGB_PEER_SMALL=0: the in-place sums (row statistics, cross-entropy terms,
// logits, dp_sync) stay on NCCL while the contraction sums use peer memory
bool peer_small() {
  static const bool on = [] {
    const char* e = std::getenv("GGB_PEER_SMALL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void all_reduce_sum(Ctx& ctx, int axis, float* buf, int64_t count, int wire) {
  if (count <= 0) return;
  if (trivial(ctx, axis)) {  // one member: the bf16 wires still round its contribution
    if (wire != GGB_FP32) {
      k_round_bf16_inplace<<<static_cast<unsigned>(ceil_div(count, 256)), 256, 0, ctx.stream>>>(buf, count);
      GGB_LAUNCH_CHECK();
      ctx.launches += 1;
    }
    return;
  }
  need(ctx, axis);
  if (peer_small() && peer_inplace_ok(ctx, axis, wire, buf)) {
    peer_all_reduce_inplace(ctx, axis, buf, count, wire, false);
    return;
  }
  all_reduce_sum_on(ctx, axis, buf, count, wire, ctx.stream, ctx.comm->wire, ctx.comm->gather);
}

namespace {
bool async_grad() {
  static const bool on = [] {
    const char* e = std::getenv("GGB_ASYNC_GRAD");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace

void all_reduce_sum_async(Ctx& ctx, int axis, float* buf, int64_t count, int wire) {
  if (count <= 0) return;
  if (trivial(ctx, axis) || !async_grad()) {
    all_reduce_sum(ctx, axis, buf, count, wire);
    return;
  }
  need(ctx, axis);
  Comm& c = *ctx.comm;
  if (!c.gstream) {
    int lo = 0, hi = 0;
    GGB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GGB_CUDA(cudaStreamCreateWithPriority(&c.gstream, cudaStreamNonBlocking, hi));
    GGB_CUDA(cudaEventCreateWithFlags(&c.gfork, cudaEventDisableTiming));
    GGB_CUDA(cudaEventCreateWithFlags(&c.gjoin, cudaEventDisableTiming));
  }
  GGB_CUDA(cudaEventRecord(c.gfork, ctx.stream));
  GGB_CUDA(cudaStreamWaitEvent(c.gstream, c.gfork, 0));
  all_reduce_sum_on(ctx, axis, buf, count, wire, c.gstream, c.gwire, c.ggather);
  c.gpending = true;
}

void reshard_async(Ctx& ctx, const std::function<void()>& f) {
  static const bool on = [] {
    const char* e = std::getenv("GGB_ASYNC_RESHARD");
    return !(e && e[0] == '0');
  }();
  Comm& c = *ctx.comm;
  if (!on) {
    f();
    return;
  }
  if (!c.rstream) {
    int lo = 0, hi = 0;
    GGB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GGB_CUDA(cudaStreamCreateWithPriority(&c.rstream, cudaStreamNonBlocking, hi));
    GGB_CUDA(cudaEventCreateWithFlags(&c.rfork, cudaEventDisableTiming));
    GGB_CUDA(cudaEventCreateWithFlags(&c.rjoin, cudaEventDisableTiming));
  }
  reshard_join(ctx);  // one reshard in flight at a time
  GGB_CUDA(cudaEventRecord(c.rfork, ctx.stream));
  GGB_CUDA(cudaStreamWaitEvent(c.rstream, c.rfork, 0));
  cudaStream_t saved = ctx.stream;
  ctx.stream = c.rstream;
  try {
    f();
  } catch (...) {
    ctx.stream = saved;
    throw;
  }
  ctx.stream = saved;
  GGB_CUDA(cudaEventRecord(c.rjoin, c.rstream));
  c.rpending = true;
}

void reshard_join(Ctx& ctx) {
  if (!ctx.comm || !ctx.comm->rpending) return;
  GGB_CUDA(cudaStreamWaitEvent(ctx.stream, ctx.comm->rjoin, 0));
  ctx.comm->rpending = false;
}

void join_async(Ctx& ctx) {
  if (!ctx.comm || !ctx.comm->gpending) return;
  Comm& c = *ctx.comm;
  GGB_CUDA(cudaEventRecord(c.gjoin, c.gstream));
  GGB_CUDA(cudaStreamWaitEvent(ctx.stream, c.gjoin, 0));
  c.gpending = false;
}

void pipelined_all_reduce(Ctx& ctx, int axis, int64_t rows, int64_t quantum, float* buf, int64_t ld, int bf16_wire,
                          const std::function<void(int64_t, int64_t)>& produce,
                          const std::function<void(int64_t, int64_t)>& after) {
  const int K = comm_chunks();
  if (trivial(ctx, axis) || rows <= 0 || K <= 1 || rows < 2 * quantum) {
    produce(0, rows);
    all_reduce_sum(ctx, axis, buf, rows * ld, bf16_wire);
    if (after) after(0, rows);
    return;
  }
  need(ctx, axis);
  Comm& c = *ctx.comm;
  if (!c.cstream) {
    int lo = 0, hi = 0;
    GGB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GGB_CUDA(cudaStreamCreateWithPriority(&c.cstream, cudaStreamNonBlocking, hi));
  }
  while (static_cast<int>(c.ev.size()) < K + 1) {
    cudaEvent_t e;
    GGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.ev.push_back(e);
  }
  const int64_t per = round_up(ceil_div(rows, K), quantum);
  const int saved_reserve = ctx.sm_reserve;
  ctx.sm_reserve = std::max(saved_reserve, comm_ctas());
  int k = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += per, ++k) {
    const int64_t r1 = std::min(rows, r0 + per);
    produce(r0, r1);
    GGB_CUDA(cudaEventRecord(c.ev[k], ctx.stream));
    GGB_CUDA(cudaStreamWaitEvent(c.cstream, c.ev[k], 0));
    all_reduce_sum_on(ctx, axis, buf + r0 * ld, (r1 - r0) * ld, bf16_wire, c.cstream, c.wire2, c.gather2);
    if (after) {
      cudaStream_t saved = ctx.stream;  // the post-processing runs on the communication stream
      ctx.stream = c.cstream;
      after(r0, r1);
      ctx.stream = saved;
    }
  }
  ctx.sm_reserve = saved_reserve;
  GGB_CUDA(cudaEventRecord(c.ev[K], c.cstream));
  GGB_CUDA(cudaStreamWaitEvent(ctx.stream, c.ev[K], 0));
}

void all_reduce_max(Ctx& ctx, int axis, float* buf, int64_t count) {
  if (trivial(ctx, axis) || count <= 0) return;
  need(ctx, axis);
  if (peer_small() && peer_inplace_ok(ctx, axis, GGB_FP32, buf)) {
    peer_all_reduce_inplace(ctx, axis, buf, count, GGB_FP32, true);
    return;
  }
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
  if (ctx.comm->aborted) fail(GGB_ETIMEOUT, "communicators were aborted after a collective timed out or failed");
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
  if (ctx.comm->aborted) fail(GGB_ETIMEOUT, "communicators were aborted after a collective timed out or failed");
  float* one = ctx.comm->gather.reserve_n<float>(1);
  GGB_NCCL(ncclAllReduce(one, one, 1, ncclFloat32, ncclSum, as_nccl(ctx.comm->world), ctx.stream));
  sync_stream(ctx, ctx.stream);
}

}  // namespace ggb
