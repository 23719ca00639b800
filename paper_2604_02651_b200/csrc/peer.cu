// Peer-memory all-reduce of the contraction sums over NVLink (CUDA IPC).
//
// The reference's RankComm::all_reduce (comm.hpp:271-303) sums the members'
// contributions in ascending axis order from 0 (fp32, or each contribution
// rounded to bf16 first under kBf16Roundtrip). On one NVLink/NVSwitch box
// every member's HBM is addressable from every other member, so the sum is a
// kernel, not a message exchange:
//   * each member's producer (the SpMM / GEMM of pmm.hpp:128,165) writes its
//     partial block straight into a slot of an IPC-exported buffer;
//   * k_peer_wait (one CTA) signals arrival into every peer's flag word and
//     waits for theirs; k_peer_reduce then reads all g partials (its own from
//     HBM, the others over NVLink) in axis order: out = 0 + p_0 + p_1 + ... —
//     the reference's exact summation order for any g (NCCL's ring order is
//     not). Only the one-CTA wait kernel ever spins, so a waiting rank never
//     holds the SMs another stream's arrival kernel needs;
//   * the consumer's format is written directly: fp32, bf16 hi (+ lo) operand
//     copies for the next tcgen05 GEMM, or fp32 plus the residual gradient —
//     the cast / add passes that follow an NCCL all-reduce are fused away;
//   * push mode (2-member groups, bf16 partials of an SpMM): the producer's
//     epilogue also stores its partial into the peer's copy of the slot, so
//     the NVLink transfer rides under the gather-bound SpMM and the reduction
//     reads local HBM only;
//   * the reshard's block permutation pulls its pieces from the members'
//     staged source blocks on a stream of its own (peer_stage / peer_pull);
//   * in-place sums (row statistics, cross-entropy terms, logits) copy the
//     buffer into the slot and sum it back in axis order (k_peer_flat).
// Every slot holds one area per member; slots alternate per call (parity of
// the call count): a member writes slot c&1 for call c only after its call
// c-1 reduction saw every peer arrive, and a peer arrives at c-1 only after
// its call c-2 reduction (the last reader of slot c&1) finished, so no
// partial is overwritten while a peer reads it. Groups are probed once, at
// context creation (every member on this host, peer-accessible, in another
// process). A wait longer than the communicator timeout raises a mapped host
// flag that the host watchdog (sync_stream) turns into CommTimeout.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <unistd.h>

#include <nccl.h>

#include "comm.hpp"
#include "prof.hpp"

namespace ggb {
namespace {

constexpr int kMaxPeers = 8;
constexpr size_t kFlagBytes = 4096;  // flag words at the head of each member's buffer

struct ReduceArgs {
  const void* src[kMaxPeers];  // partial block of member q (axis order)
  int g, wire;
  int64_t rows, cols, ld;
  float* out;
  int64_t ldo;
  bf16* outb;
  bf16* outlo;
  int64_t ldb;
  const float* add;  // optional: out = sum + add (fp32 out only)
  int64_t ldadd;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// bf16_round (comm.hpp:29-39): RNE to bf16, Inf/NaN truncated (NaN keeps a payload bit)
__device__ __forceinline__ float bf16_round_ref(float x) {
  const uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) == 0x7f800000u) {
    uint32_t r = u & 0xffff0000u;
    if ((u & 0x007fffffu) != 0 && (r & 0x007f0000u) == 0) r |= 0x00400000u;
    return __uint_as_float(r);
  }
  return __uint_as_float((u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u);
}

// V consecutive elements of a member's partial as one 16-byte load: fp32
// partials (V = 4) or bf16 partials already rounded by their producer (V = 8).
template <class T>
struct Vec;
template <>
struct Vec<float> {
  static constexpr int V = 4;
  __device__ static void unpack(const uint4& x, float* v) {
    v[0] = __uint_as_float(x.x), v[1] = __uint_as_float(x.y), v[2] = __uint_as_float(x.z), v[3] = __uint_as_float(x.w);
  }
};
template <>
struct Vec<bf16> {
  static constexpr int V = 8;
  __device__ static void unpack(const uint4& x, float* v) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};

__device__ __forceinline__ void put_bf16x4(bf16* p, const float* v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}

// Arrival barrier of one peer collective: thread q < g posts this member's
// arrival into member q's flag word, then waits for every member's arrival
// in its own flag words (system-scope release / acquire; the partials
// written by earlier kernels are published by the fence before the flag).
// A wait beyond the deadline raises the mapped host error word and returns.
struct WaitArgs {
  unsigned long long* arrive[kMaxPeers];  // member q's flag word for this member
  const unsigned long long* mine;         // this member's flag words [g]
  int g, me;
  unsigned long long epoch, timeout_ns;
  int* err;
};
__global__ void __launch_bounds__(32) k_peer_wait(WaitArgs a) {
  const int q = threadIdx.x;
  if (q < a.g && q != a.me) {
    __threadfence_system();
    st_release_sys(a.arrive[q], a.epoch);
    // a member already timed out: the host raises CommTimeout at its next
    // wait; later barriers return at once instead of each spinning to the deadline
    if (*reinterpret_cast<volatile int*>(a.err)) return;
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(a.mine + q) < a.epoch) {
      if (globaltimer() - t0 > a.timeout_ns) {
        *reinterpret_cast<volatile int*>(a.err) = 1;
        break;
      }
      __nanosleep(128);
    }
  }
  __syncwarp();
}

// Grid-stride over the block's 16-byte units (row-major, so a warp reads
// 512 contiguous bytes of every member); each thread issues the loads of U
// units of every member before summing any, so enough NVLink reads are in
// flight to cover the remote latency.
template <class T, int G>
__global__ void __launch_bounds__(256) k_peer_reduce(ReduceArgs a) {
  constexpr int V = Vec<T>::V;
  constexpr int NG = G > 0 ? G : kMaxPeers;
  constexpr int U = G == 2 ? 4 : (G == 4 ? 2 : 1);
  const int n = G > 0 ? G : a.g;
  const uint32_t cv = static_cast<uint32_t>((a.cols + V - 1) / V);
  const uint32_t total = static_cast<uint32_t>(a.rows) * cv;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < total; base += U * stride) {
    uint4 x[U][NG];
    uint32_t row[U], col[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t t = base + u * stride;
      row[u] = t / cv;
      col[u] = (t - row[u] * cv) * V;
      if (t < total) {
        const int64_t off = static_cast<int64_t>(row[u]) * a.ld + col[u];
#pragma unroll
        for (int q = 0; q < NG; ++q)
          if (q < n) x[u][q] = *reinterpret_cast<const uint4*>(static_cast<const T*>(a.src[q]) + off);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (base + u * stride >= total) break;
      const int64_t r = row[u];
      float v[V];
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = 0.f;
#pragma unroll
      for (int q = 0; q < NG; ++q) {  // 0 + p_0 + p_1 + ... in axis order
        if (q >= n) break;
        float y[V];
        Vec<T>::unpack(x[u][q], y);
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] += (sizeof(T) == 4 && a.wire) ? bf16_round_ref(y[i]) : y[i];
      }
#pragma unroll
      for (int h = 0; h < V; h += 4) {
        const int64_t cc = col[u] + h;
        float* w = v + h;
        if (cc >= a.cols) break;
        if (a.add) {
          const float4 d = *reinterpret_cast<const float4*>(a.add + r * a.ldadd + cc);
          w[0] += d.x, w[1] += d.y, w[2] += d.z, w[3] += d.w;
        }
        if (cc + 4 > a.cols)  // padding columns of the row stay zero
          for (int i = 0; i < 4; ++i)
            if (cc + i >= a.cols) w[i] = 0.f;
        if (a.out) *reinterpret_cast<float4*>(a.out + r * a.ldo + cc) = make_float4(w[0], w[1], w[2], w[3]);
        if (a.outb) {
          put_bf16x4(a.outb + r * a.ldb + cc, w);
          if (a.outlo) {
            float lo[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) lo[i] = w[i] - __bfloat162float(__float2bfloat16_rn(w[i]));
            put_bf16x4(a.outlo + r * a.ldb + cc, lo);
          }
        }
      }
    }
  }
}

// GGB_PEER_PUSH: 1 always, 0 never; default: push bf16 partials only (an
// fp32 partial's NVLink stores outlast the SpMM that produces it: C2 1x2x2x1
// fp32 13.3 -> 13.8 ms/step with push, bf16 wire 12.2 -> 12.1)
int peer_push_mode() {
  static const int v = [] {
    const char* e = std::getenv("GGB_PEER_PUSH");
    return e ? (e[0] == '1' ? 1 : 0) : 2;
  }();
  return v;
}

bool peer_env_on() {
  static const bool on = [] {
    const char* e = std::getenv("GGB_PEER");
    return !(e && e[0] == '0');
  }();
  return on;
}

#define GGB_NCCL_P(call)                                                                       \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      ::ggb::fail(GGB_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_));              \
  } while (0)

// Member q's area of the current slot in member m's buffer: every slot holds
// one partial-sized area per member (pull mode fills only its own area of its
// own buffer; push mode mirrors it into the same area of the peers' buffers).
char* area(const PeerAxis& P, int m, int q) {
  return P.rbase[m] + kFlagBytes + (static_cast<size_t>(P.parity) * P.g + q) * P.cap;
}

// group index 0..3: a grid axis; kPeerPmm: the ranks of this rank's DP group
// (its X x Y x Z grid, contiguous world ranks)
int pmm_size(const Ctx& ctx) { return ctx.grid.dims[1] * ctx.grid.dims[2] * ctx.grid.dims[3]; }
void* group_comm(const Comm& c, int axis) { return axis == kPeerPmm ? c.pmm : c.axis[axis]; }
int group_size(const Ctx& ctx, int axis) { return axis == kPeerPmm ? pmm_size(ctx) : ctx.comm->size[axis]; }
int group_pos(const Ctx& ctx, int axis) { return axis == kPeerPmm ? ctx.rank % pmm_size(ctx) : ctx.comm->pos[axis]; }

void close_mappings(PeerAxis& P) {
  for (int q = 0; q < P.g; ++q)
    if (q != P.me && P.rbase[q]) {
      cudaIpcCloseMemHandle(P.rbase[q]);
      P.rbase[q] = nullptr;
    }
  if (P.base) cudaFree(P.base);
  P.base = nullptr;
  P.cap = 0;
}

// Collective on the axis group (every member calls it with the same bytes):
// (re)allocates this member's [flags | slot 0 | slot 1] buffer with room for
// `bytes` per slot and maps every peer's.
void grow(Ctx& ctx, int axis, PeerAxis& P, size_t bytes) {
  Comm& c = *ctx.comm;
  auto* nc = static_cast<ncclComm_t>(group_comm(c, axis));
  if (P.base) {  // every member done reading the old buffers
    float* one = P.stage.reserve_n<float>(1);
    GGB_NCCL_P(ncclAllReduce(one, one, 1, ncclFloat32, ncclSum, nc, ctx.stream));
    sync_stream(ctx, ctx.stream);
    close_mappings(P);
  }
  size_t want = bytes + bytes / 8;
  want = (want + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
  GGB_CUDA(cudaMalloc(&P.base, kFlagBytes + 2 * static_cast<size_t>(P.g) * want));
  GGB_CUDA(cudaMemsetAsync(P.base, 0, kFlagBytes, ctx.stream));
  P.cap = want;
  P.epoch = 0;
  P.calls = 0;
  cudaIpcMemHandle_t h;
  GGB_CUDA(cudaIpcGetMemHandle(&h, P.base));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  // staging of its own: grow may run on the reshard stream while the compute
  // stream uses the communicator's staging buffers
  uint8_t* d = P.stage.reserve_n<uint8_t>(64 * (P.g + 1));
  GGB_CUDA(cudaMemcpyAsync(d + 64 * P.g, &h, 64, cudaMemcpyHostToDevice, ctx.stream));
  GGB_NCCL_P(ncclAllGather(d + 64 * P.g, d, 64, ncclUint8, nc, ctx.stream));
  std::vector<uint8_t> all(64 * P.g);
  GGB_CUDA(cudaMemcpyAsync(all.data(), d, all.size(), cudaMemcpyDeviceToHost, ctx.stream));
  sync_stream(ctx, ctx.stream);
  for (int q = 0; q < P.g; ++q) {
    if (q == P.me) {
      P.rbase[q] = P.base;
      continue;
    }
    cudaIpcMemHandle_t hq;
    std::memcpy(&hq, all.data() + 64 * q, 64);
    void* p = nullptr;
    GGB_CUDA(cudaIpcOpenMemHandle(&p, hq, cudaIpcMemLazyEnablePeerAccess));
    P.rbase[q] = static_cast<char*>(p);
  }
}

}  // namespace

PeerAxis::~PeerAxis() {
  close_mappings(*this);
  if (err) cudaFreeHost(err);
}

namespace {
// The collective probe of one group (every member calls it, in the same order).
void probe(Ctx& ctx, int axis) {
  Comm& c = *ctx.comm;
  {
    // one probe per axis, agreed by every member: IPC-mappable peers on this node
    auto* nc = static_cast<ncclComm_t>(group_comm(c, axis));
    const int g = group_size(ctx, axis);
    int dev = ctx.device;
    // {host hash, device, process id} of every member: IPC needs peers on
    // this host, peer-accessible, and in other processes (a process cannot
    // open its own IPC handles; one-process grids, e.g. the CLI's thread per
    // rank, keep NCCL)
    int* d = c.gather.reserve_n<int>(3 * g);
    char host[256] = {};
    gethostname(host, sizeof(host) - 1);
    int hh = 5381;
    for (const char* p = host; *p; ++p) hh = hh * 33 + *p;
    const int pid = static_cast<int>(getpid());
    int mine[3] = {hh, dev, pid};
    int* dm = c.wire.reserve_n<int>(3);
    GGB_CUDA(cudaMemcpyAsync(dm, mine, sizeof(mine), cudaMemcpyHostToDevice, ctx.stream));
    GGB_NCCL_P(ncclAllGather(dm, d, 3, ncclInt32, nc, ctx.stream));
    std::vector<int> all(3 * g);
    GGB_CUDA(cudaMemcpyAsync(all.data(), d, sizeof(int) * 3 * g, cudaMemcpyDeviceToHost, ctx.stream));
    sync_stream(ctx, ctx.stream);
    bool ok = true;
    for (int q = 0; q < g; ++q) {
      if (all[3 * q] != hh) ok = false;
      if (q == group_pos(ctx, axis)) continue;
      if (all[3 * q + 2] == pid) ok = false;
      int can = 0;
      if (ok && (cudaDeviceCanAccessPeer(&can, dev, all[3 * q + 1]) != cudaSuccess || !can)) ok = false;
    }
    // agreement: the minimum over the group
    float* f = c.gather.reserve_n<float>(1);
    const float v = ok ? 1.f : 0.f;
    GGB_CUDA(cudaMemcpyAsync(f, &v, 4, cudaMemcpyHostToDevice, ctx.stream));
    GGB_NCCL_P(ncclAllReduce(f, f, 1, ncclFloat32, ncclMin, nc, ctx.stream));
    float agreed = 0.f;
    GGB_CUDA(cudaMemcpyAsync(&agreed, f, 4, cudaMemcpyDeviceToHost, ctx.stream));
    sync_stream(ctx, ctx.stream);
    c.peer_state[axis] = agreed > 0.5f ? 1 : -1;
    if (c.peer_state[axis] == 1) {
      auto P = std::make_unique<PeerAxis>();
      P->g = g;
      P->me = group_pos(ctx, axis);
      GGB_CUDA(cudaHostAlloc(&P->err, sizeof(int), cudaHostAllocMapped));
      *P->err = 0;
      GGB_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&P->err_dev), P->err, 0));
      c.peer[axis] = std::move(P);
    }
  }
}

bool eligible(const Ctx& ctx, int axis) {
  // the contraction axes X, Y, Z and the DP group's PMM grid; the D axis
  // (dp_sync's gradient sum, 1 MB a step) stays on NCCL
  if (!peer_env_on() || !ctx.comm || axis == kD) return false;
  if (axis == kPeerPmm ? pmm_size(ctx) == 1 : trivial(ctx, axis)) return false;
  return group_size(ctx, axis) <= kMaxPeers && group_comm(*ctx.comm, axis) != nullptr;
}
}  // namespace

void peer_setup(Ctx& ctx) {
  if (!ctx.comm) return;
  for (int axis : {1, 2, 3, kPeerPmm})
    if (eligible(ctx, axis)) probe(ctx, axis);
}

bool peer_ok(Ctx& ctx, int axis, int wire) {
  if (!ctx.comm || ctx.comm->aborted || wire == GGB_BF16_SUM || !eligible(ctx, axis)) return false;
  return ctx.comm->peer_state[axis] == 1;  // decided at context creation (peer_setup)
}

void* peer_slot(Ctx& ctx, int axis, size_t bytes) {
  PeerAxis& P = *ctx.comm->peer[axis];
  P.pushed = false;
  if (bytes > P.cap) grow(ctx, axis, P, bytes);
  P.parity = static_cast<int>(++P.calls & 1);
  return area(P, P.me, P.me);
}

PeerSlot peer_slot_push(Ctx& ctx, int axis, size_t bytes, bool bf16_part) {
  PeerSlot r;
  r.local = peer_slot(ctx, axis, bytes);
  PeerAxis& P = *ctx.comm->peer[axis];
  const int mode = peer_push_mode();
  if (P.g == 2 && (mode == 1 || (mode == 2 && bf16_part))) {
    r.mirror = area(P, 1 - P.me, P.me);
    P.pushed = true;
  } else {
    P.pushed = false;
  }
  return r;
}

namespace {
// arrival barrier of collective e on the group (one CTA, ctx.stream)
void launch_wait(Ctx& ctx, PeerAxis& P, uint64_t e) {
  WaitArgs w{};
  for (int q = 0; q < P.g; ++q) w.arrive[q] = reinterpret_cast<unsigned long long*>(P.rbase[q]) + P.me;
  w.mine = reinterpret_cast<const unsigned long long*>(P.base);
  w.g = P.g;
  w.me = P.me;
  w.epoch = e;
  w.timeout_ns = static_cast<unsigned long long>(ctx.comm->timeout_ms) * 1000000ull;
  w.err = P.err_dev;
  k_peer_wait<<<1, 32, 0, ctx.stream>>>(w);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}
}  // namespace

void peer_all_reduce(Ctx& ctx, int axis, int64_t rows, int64_t cols, int64_t ld, bool src_bf16, int wire, float* out,
                     int64_t ldo, bf16* outb, bf16* outlo, int64_t ldb, const float* add, int64_t ldadd,
                     int64_t row0) {
  Comm& c = *ctx.comm;
  PeerAxis& P = *c.peer[axis];
  require(ld % (src_bf16 ? 8 : 4) == 0 && (!out || ldo % 4 == 0) && (!outb || ldb % 4 == 0) &&
              (!add || ldadd % 4 == 0),
          "peer_all_reduce: row strides must be whole 16-byte vectors");
  const size_t esz = src_bf16 ? 2 : 4;
  require(static_cast<size_t>((row0 + rows) * ld) * esz <= P.cap, "peer_all_reduce: slot not reserved");
  require(rows * ld < (int64_t(1) << 32), "peer_all_reduce: block too large for 32-bit unit indices");
  const uint64_t e = ++P.epoch;
  ReduceArgs a{};
  // member q's partial: in q's own buffer (pull), or mirrored into ours by its producer (push)
  for (int q = 0; q < P.g; ++q) a.src[q] = area(P, P.pushed ? P.me : q, q) + static_cast<size_t>(row0 * ld) * esz;
  a.g = P.g;
  a.wire = wire == GGB_BF16_WIRE ? 1 : 0;
  a.rows = rows;
  a.cols = cols;
  a.ld = ld;
  a.out = out;
  a.ldo = ldo;
  a.outb = outb;
  a.outlo = outlo;
  a.ldb = ldb;
  a.add = add;
  a.ldadd = ldadd;
  // bytes this member pulls over NVLink
  const double pulled = static_cast<double>(rows) * cols * (src_bf16 ? 2 : 4) * (P.g - 1);
  ProfScope ps(ctx, kProfComm, pulled, 0);
  launch_wait(ctx, P, e);
  static const int bps = [] {  // GGB_PEER_BPS: reduction blocks per SM
    const char* e = std::getenv("GGB_PEER_BPS");
    const int v = e ? std::atoi(e) : 3;
    return v >= 1 && v <= 8 ? v : 3;
  }();
  const int blocks = ctx.num_sms * bps;
  if (src_bf16) {
    if (P.g == 2)
      k_peer_reduce<bf16, 2><<<blocks, 256, 0, ctx.stream>>>(a);
    else if (P.g == 4)
      k_peer_reduce<bf16, 4><<<blocks, 256, 0, ctx.stream>>>(a);
    else
      k_peer_reduce<bf16, 0><<<blocks, 256, 0, ctx.stream>>>(a);
  } else {
    if (P.g == 2)
      k_peer_reduce<float, 2><<<blocks, 256, 0, ctx.stream>>>(a);
    else if (P.g == 4)
      k_peer_reduce<float, 4><<<blocks, 256, 0, ctx.stream>>>(a);
    else
      k_peer_reduce<float, 0><<<blocks, 256, 0, ctx.stream>>>(a);
  }
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

namespace {

// One piece of a block permutation: rows x cols floats from a member's
// packed source block (mapped) into this rank's destination block.
struct PullPiece {
  const float* src;
  float* dst;
  int64_t lds, ldd, rows, cols;
  uint32_t unit0;  // first unit (4 floats, or 1 when unaligned) of this piece in the launch
  int vec;         // 1: float4 units
};
constexpr int kMaxPieces = 16;
struct PullArgs {
  PullPiece pc[kMaxPieces];
  int npieces;
  uint32_t total;
};

// Grid-stride over the pieces' units; every thread issues U units' loads
// (NVLink reads for remote pieces) before storing any.
__global__ void __launch_bounds__(256) k_peer_pull(PullArgs a) {
  constexpr int U = 4;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < a.total; base += U * stride) {
    float4 v[U];
    float* dst[U];
    int vec[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t t = base + u * stride;
      dst[u] = nullptr;
      vec[u] = 0;
      if (t >= a.total) continue;
      int k = 0;
      while (k + 1 < a.npieces && a.pc[k + 1].unit0 <= t) ++k;
      const PullPiece& p = a.pc[k];
      const uint32_t i = t - p.unit0;
      vec[u] = p.vec;
      if (p.vec) {
        const uint32_t cv = static_cast<uint32_t>(p.cols / 4);
        const uint32_t r = i / cv, c = (i - r * cv) * 4;
        v[u] = *reinterpret_cast<const float4*>(p.src + r * p.lds + c);
        dst[u] = p.dst + r * p.ldd + c;
      } else {
        const uint32_t cc = static_cast<uint32_t>(p.cols);
        const uint32_t r = i / cc, c = i - r * cc;
        v[u].x = p.src[r * p.lds + c];
        dst[u] = p.dst + r * p.ldd + c;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!dst[u]) continue;
      if (vec[u])
        *reinterpret_cast<float4*>(dst[u]) = v[u];
      else
        *dst[u] = v[u].x;
    }
  }
}

}  // namespace

float* peer_stage(Ctx& ctx, const float* src, int64_t lds, int64_t rows, int64_t cols, int64_t ld_stage,
                  size_t reserve_bytes) {
  require(static_cast<size_t>(rows * ld_stage) * 4 <= reserve_bytes, "peer_stage: block exceeds the group's reserve");
  float* slot = static_cast<float*>(peer_slot(ctx, kPeerPmm, reserve_bytes));
  if (rows > 0 && cols > 0)
    GGB_CUDA(cudaMemcpy2DAsync(slot, ld_stage * 4, src, lds * 4, cols * 4, rows, cudaMemcpyDeviceToDevice,
                               ctx.stream));
  return slot;
}

void peer_pull(Ctx& ctx, const std::vector<PeerPiece>& pieces) {
  Comm& c = *ctx.comm;
  PeerAxis& P = *c.peer[kPeerPmm];
  const uint64_t e = ++P.epoch;
  PullArgs a{};
  double bytes = 0;
  uint64_t units = 0;
  int np = 0;
  for (const PeerPiece& x : pieces) {
    if (x.rows <= 0 || x.cols <= 0) continue;
    require(np < kMaxPieces, "peer_pull: too many pieces");
    require(x.member >= 0 && x.member < P.g, "peer_pull: member outside the group");
    const float* base = reinterpret_cast<const float*>(area(P, x.member, x.member));
    PullPiece& p = a.pc[np++];
    p.src = base + x.src_off;
    p.dst = x.dst;
    p.lds = x.lds;
    p.ldd = x.ldd;
    p.rows = x.rows;
    p.cols = x.cols;
    p.vec = (x.cols % 4 == 0 && x.lds % 4 == 0 && x.ldd % 4 == 0 && x.src_off % 4 == 0 &&
             (reinterpret_cast<uintptr_t>(x.dst) & 15) == 0)
                ? 1
                : 0;
    p.unit0 = static_cast<uint32_t>(units);
    units += static_cast<uint64_t>(x.rows) * (p.vec ? x.cols / 4 : x.cols);
    if (x.member != P.me) bytes += 4.0 * x.rows * x.cols;
  }
  require(units < (uint64_t(1) << 32), "peer_pull: too many units");
  a.npieces = np;
  a.total = static_cast<uint32_t>(units);
  ProfScope ps(ctx, kProfComm, bytes, 0);
  launch_wait(ctx, P, e);  // every member arrives, even with nothing to pull
  if (units == 0) return;
  const unsigned blocks = static_cast<unsigned>(
      std::min<int64_t>(ctx.num_sms * 4, ceil_div(static_cast<int64_t>(units), 256 * 4)));
  k_peer_pull<<<blocks, 256, 0, ctx.stream>>>(a);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

namespace {
int peer_chunks() {
  static const int v = [] {
    const char* e = std::getenv("GGB_PEER_CHUNKS");
    const int c = e ? std::atoi(e) : 1;
    return c >= 1 && c <= 16 ? c : 1;
  }();
  return v;
}
int peer_reserve() {
  static const int v = [] {
    const char* e = std::getenv("GGB_PEER_RESERVE");
    const int c = e ? std::atoi(e) : 16;
    return c >= 0 && c <= 64 ? c : 16;
  }();
  return v;
}
}  // namespace

void peer_pipelined(Ctx& ctx, int64_t rows, int64_t quantum, const std::function<void(int64_t, int64_t)>& produce,
                    const std::function<void(int64_t, int64_t)>& reduce) {
  const int K = peer_chunks();
  if (K <= 1 || rows < 2 * quantum) {
    produce(0, rows);
    reduce(0, rows);
    return;
  }
  Comm& c = *ctx.comm;
  if (!c.pstream) {
    int lo = 0, hi = 0;
    GGB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GGB_CUDA(cudaStreamCreateWithPriority(&c.pstream, cudaStreamNonBlocking, hi));
  }
  while (static_cast<int>(c.pev.size()) < K + 1) {
    cudaEvent_t e;
    GGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c.pev.push_back(e);
  }
  const int64_t per = round_up(ceil_div(rows, K), quantum);
  const int saved_reserve = ctx.sm_reserve;
  int k = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += per, ++k) {
    const int64_t r1 = std::min(rows, r0 + per);
    // the producer leaves SMs to the reductions of the chunks before it
    ctx.sm_reserve = k > 0 ? std::max(saved_reserve, peer_reserve()) : saved_reserve;
    produce(r0, r1);
    GGB_CUDA(cudaEventRecord(c.pev[k], ctx.stream));
    GGB_CUDA(cudaStreamWaitEvent(c.pstream, c.pev[k], 0));
    cudaStream_t saved = ctx.stream;
    ctx.stream = c.pstream;
    try {
      reduce(r0, r1);
    } catch (...) {
      ctx.stream = saved;
      ctx.sm_reserve = saved_reserve;
      throw;
    }
    ctx.stream = saved;
  }
  ctx.sm_reserve = saved_reserve;
  GGB_CUDA(cudaEventRecord(c.pev[K], c.pstream));
  GGB_CUDA(cudaStreamWaitEvent(ctx.stream, c.pev[K], 0));
}

namespace {

// In-place flat reduction of the members' copies of one buffer: out[i] =
// 0 + p_0[i] + ... (axis order; each bf16-rounded under the bf16 wire) or the
// max; float4 body, scalar tail.
struct FlatArgs {
  const float* src[kMaxPeers];
  int g, op, wire;  // op 0 sum, 1 max
  int64_t n;
  float* out;
};
__device__ __forceinline__ float flat_combine(const FlatArgs& a, float acc, float v, bool first) {
  if (a.op == 1) return first ? v : fmaxf(acc, v);
  return acc + (a.wire ? bf16_round_ref(v) : v);
}
__global__ void __launch_bounds__(256) k_peer_flat(FlatArgs a) {
  const int64_t n4 = a.n / 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 v[kMaxPeers];
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
      if (q < a.g) v[q] = reinterpret_cast<const float4*>(a.src[q])[i];
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q) {
      if (q >= a.g) break;
      r.x = flat_combine(a, r.x, v[q].x, q == 0);
      r.y = flat_combine(a, r.y, v[q].y, q == 0);
      r.z = flat_combine(a, r.z, v[q].z, q == 0);
      r.w = flat_combine(a, r.w, v[q].w, q == 0);
    }
    reinterpret_cast<float4*>(a.out)[i] = r;
  }
  for (int64_t i = 4 * n4 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    float r = 0.f;
    for (int q = 0; q < a.g; ++q) r = flat_combine(a, r, a.src[q][i], q == 0);
    a.out[i] = r;
  }
}

}  // namespace

bool peer_inplace_ok(Ctx& ctx, int axis, int wire, const float* buf) {
  if (!ctx.comm || wire == GGB_BF16_SUM || (reinterpret_cast<uintptr_t>(buf) & 15) != 0) return false;
  const Comm& c = *ctx.comm;
  // one stream per group carries the peer protocol: the compute stream
  if (ctx.stream == c.gstream || ctx.stream == c.cstream || ctx.stream == c.pstream || ctx.stream == c.rstream)
    return false;
  return peer_ok(ctx, axis, wire);
}

void peer_all_reduce_inplace(Ctx& ctx, int axis, float* buf, int64_t count, int wire, bool max) {
  if (count <= 0) return;
  Comm& c = *ctx.comm;
  float* slot = static_cast<float*>(peer_slot(ctx, axis, static_cast<size_t>(round_up(count, 4)) * 4));
  PeerAxis& P = *c.peer[axis];
  GGB_CUDA(cudaMemcpyAsync(slot, buf, static_cast<size_t>(count) * 4, cudaMemcpyDeviceToDevice, ctx.stream));
  const uint64_t e = ++P.epoch;
  FlatArgs a{};
  for (int q = 0; q < P.g; ++q) a.src[q] = reinterpret_cast<const float*>(area(P, q, q));
  a.g = P.g;
  a.op = max ? 1 : 0;
  a.wire = (!max && wire == GGB_BF16_WIRE) ? 1 : 0;
  a.n = count;
  a.out = buf;
  ProfScope ps(ctx, kProfComm, 4.0 * count * (P.g - 1), 0);
  launch_wait(ctx, P, e);
  const unsigned blocks =
      static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ctx.num_sms * 4, ceil_div(count, 4 * 256))));
  k_peer_flat<<<blocks, 256, 0, ctx.stream>>>(a);
  GGB_LAUNCH_CHECK();
  ctx.launches += 1;
}

bool peer_timed_out(const Comm& c) {
  for (const auto& p : c.peer)
    if (p && p->err && *reinterpret_cast<volatile int*>(p->err)) return true;
  return false;
}

}  // namespace ggb
