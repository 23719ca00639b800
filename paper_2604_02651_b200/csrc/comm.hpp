// Grid collectives (RankComm, comm.hpp:254-408) over NCCL: one world
// communicator plus one split per grid axis (colour = group id on the axis,
// key = coordinate on it, mirroring Communicator's per-axis Channels,
// comm.hpp:209-214). Singleton groups are free and need no communicator.
#pragma once

#include <functional>

#include "runtime.hpp"

namespace ggb {

// One axis group's peer-memory state (peer.cu): this member's IPC-exported
// [flag words | slot 0 | slot 1] buffer and every member's mapping of it.
struct PeerAxis {
  int g = 0, me = 0;
  size_t cap = 0;                // bytes per slot
  char* base = nullptr;          // this member's buffer
  char* rbase[8] = {};           // member q's buffer as mapped here (rbase[me] = base)
  uint64_t epoch = 0;            // arrival barriers issued on this group
  uint64_t calls = 0;            // slots handed out (their parity picks the slot)
  int parity = 0;                // slot of the current call
  bool pushed = false;           // the current call's producers mirror their partials (push mode)
  int* err = nullptr;            // mapped host word: a peer never arrived
  int* err_dev = nullptr;
  DevBuf stage;                  // handle exchange / barrier staging (grow)
  ~PeerAxis();
};

struct Comm {
  void* world = nullptr;     // ncclComm_t
  void* axis[4] = {};        // ncclComm_t per axis (null for singleton groups)
  void* pmm = nullptr;       // ncclComm_t of this rank's DP group (X*Y*Z ranks; null when 1)
  int size[4] = {1, 1, 1, 1};
  int pos[4] = {0, 0, 0, 0};  // coordinate on the axis
  DevBuf gather;             // all-gather staging
  DevBuf wire;               // bf16 wire staging
  // pipelined collectives: their own stream, staging and events
  cudaStream_t cstream = nullptr;
  DevBuf gather2, wire2;
  std::vector<cudaEvent_t> ev;
  // CommConfig::timeout (comm.hpp:195-198; default 60 s, GGB_COMM_TIMEOUT_MS
  // or ggb_ctx_set_comm_timeout): how long a host wait on a stream holding
  // collectives may last before the communicators are aborted
  int64_t timeout_ms = 60000;
  bool aborted = false;
  // gradient all-reduces issued beside the backward (all_reduce_sum_async)
  cudaStream_t gstream = nullptr;
  cudaEvent_t gfork = nullptr, gjoin = nullptr;
  DevBuf gwire, ggather;
  bool gpending = false;
  // peer-memory reductions per axis: 0 not probed, 1 on, -1 unavailable
  // peer-memory reshards on their own stream beside the compute (reshard_join)
  cudaStream_t rstream = nullptr;
  cudaEvent_t rfork = nullptr, rjoin = nullptr;
  bool rpending = false;
  // chunked peer reductions (peer_pipelined): their stream and events
  cudaStream_t pstream = nullptr;
  std::vector<cudaEvent_t> pev;
  // (index 4: the DP group's PMM grid, for the reshard's block permutation)
  int peer_state[5] = {0, 0, 0, 0, 0};
  std::unique_ptr<PeerAxis> peer[5];
  ~Comm();
};

/// Host wait for stream s with the collective watchdog: polls the stream,
/// the communicators' asynchronous errors (a failed / aborted peer) and the
/// deadline. On an NCCL error or the deadline, aborts every communicator of
/// the context (their in-flight kernels return) and fails with GGB_ENCCL /
/// GGB_ETIMEOUT (CommTimeout: "collective timed out: not all group members
/// arrived", comm.hpp:157-158). Without communicators: cudaStreamSynchronize.
void sync_stream(Ctx& ctx, cudaStream_t s);

int comm_get_unique_id(uint8_t out[128]);
std::unique_ptr<Comm> comm_create(const Grid& grid, int rank, const uint8_t* uid);

// In-place sum over the rank's group along `axis`. wire (ggb_precision):
// 0 fp32; 1 each member's contribution rounded to bf16 (RNE) and the fp32 sum
// taken in ascending axis order — the reference's Precision::kBf16Roundtrip
// (comm.hpp:271-303) reproduced exactly by an all-gather of bf16
// contributions; 2 bf16 payloads summed by one NCCL all-reduce.
void all_reduce_sum(Ctx& ctx, int axis, float* buf, int64_t count, int wire);
// all_reduce_sum on the gradient stream: the compute stream goes on (the
// backward's dX products need no dW), join_async makes it wait for every
// such reduction issued since the last join. Same sums as all_reduce_sum.
// GGB_ASYNC_GRAD=0 runs them inline.
void all_reduce_sum_async(Ctx& ctx, int axis, float* buf, int64_t count, int wire);
void join_async(Ctx& ctx);
void all_reduce_max(Ctx& ctx, int axis, float* buf, int64_t count);
// Row-chunked overlap of a producer and its all-reduce: chunk k
// of `rows` rows (row stride ld floats of buf) is produced on the compute
// stream by produce(r0, r1), then all-reduced along `axis` on the
// communication stream — and post-processed there by after(r0, r1) — while
// chunk k+1 is produced. Chunk bounds are multiples of `quantum` rows. The
// persistent kernels leave SMs free for the collective meanwhile. The compute
// stream waits for the last chunk before returning. Same result as producing
// everything, then one all-reduce (per-element sums are unchanged).
// GGB_COMM_CHUNKS (default 1: produce everything, then one all-reduce) sets
// the chunk count; measured on 4 B200 at C3 the chunked form is slower
// (DESIGN.md), so it is off by default.
void pipelined_all_reduce(Ctx& ctx, int axis, int64_t rows, int64_t quantum, float* buf, int64_t ld, int wire,
                          const std::function<void(int64_t, int64_t)>& produce,
                          const std::function<void(int64_t, int64_t)>& after = {});
void all_reduce_u64(Ctx& ctx, int axis, uint64_t* buf, int64_t count);  // exact integer sum
// Gathers `count` floats from every member of the axis group into out
// ([size][count], axis order).
void all_gather(Ctx& ctx, int axis, const float* in, int64_t count, float* out);
// Point-to-point block exchange on the world communicator (one NCCL group):
// every send is a (rows x cols) fp32 sub-block at ptr with leading dimension
// ld, packed, sent to world rank `peer`; every recv unpacks into its block.
struct BlockXfer {
  int peer;
  float* ptr;
  int64_t ld, rows, cols;
};
void exchange_blocks(Ctx& ctx, const std::vector<BlockXfer>& sends, const std::vector<BlockXfer>& recvs);
void barrier(Ctx& ctx);

// ---- peer-memory all-reduce over NVLink (peer.cu) ----------------------------
// peer_ok: the axis group can sum through mapped peer memory (every member
// on this node, IPC-mappable, in another process; GGB_PEER=0 disables; not
// for the NCCL-bf16 wire, not the D axis).
bool peer_ok(Ctx& ctx, int axis, int wire);
// Collective, at context creation: probes every eligible group (X, Y, Z axes,
// the DP group's PMM grid) so no later call blocks on a probe.
void peer_setup(Ctx& ctx);
// The slot the producer of the next peer_all_reduce on `axis` writes its
// partial block into (collective when it has to grow).
void* peer_slot(Ctx& ctx, int axis, size_t bytes);
// Push mode (2-member groups; bf16 partials by default, GGB_PEER_PUSH=0/1
// never / always): the producer also
// stores its partial into the peer's copy of the slot (`mirror`, NVLink
// stores overlapped with the producer's own HBM-bound work), so the
// reduction reads only local HBM. mirror is null when the group pulls.
struct PeerSlot {
  void* local = nullptr;
  void* mirror = nullptr;
};
PeerSlot peer_slot_push(Ctx& ctx, int axis, size_t bytes, bool bf16_part);
// The ordered sum 0 + p_0 + ... + p_{g-1} (axis order) of the members' slot
// blocks (rows x cols, stride ld elements), written as fp32 (out, optionally
// + add) and/or bf16 hi (+ lo = x - hi) operand copies. Partials are fp32, or
// bf16 already rounded by their producer (src_bf16: the bf16 wire's
// contributions, half the NVLink bytes); fp32 partials are rounded here under
// GGB_BF16_WIRE — either way exactly kBf16Roundtrip (comm.hpp:271-303).
// row0: first row of the slot block this call sums (a chunk of the block;
// out / outb / add point at that chunk's first row).
void peer_all_reduce(Ctx& ctx, int axis, int64_t rows, int64_t cols, int64_t ld, bool src_bf16, int wire, float* out,
                     int64_t ldo, bf16* outb, bf16* outlo, int64_t ldb, const float* add = nullptr,
                     int64_t ldadd = 0, int64_t row0 = 0);
// Producer / peer reduction overlap: rows in GGB_PEER_CHUNKS chunks (multiples
// of quantum); chunk k is produced on the compute stream (leaving
// GGB_PEER_RESERVE SMs free once a reduction may run) and reduced on the peer
// stream while chunk k+1 is produced; the compute stream waits for the last
// reduction. One chunk (default): produce, then reduce, inline.
void peer_pipelined(Ctx& ctx, int64_t rows, int64_t quantum, const std::function<void(int64_t, int64_t)>& produce,
                    const std::function<void(int64_t, int64_t)>& reduce);
bool peer_timed_out(const Comm& c);
// In-place all-reduce of a device buffer through peer memory (the buffer is
// copied into the group's slot, then summed / maxed in axis order back into
// it): the row statistics, cross-entropy terms, logits and dp_sync sums on
// the compute stream. peer_inplace_ok: the group is peer-capable and the
// call is on the compute stream (16-byte aligned buffer).
bool peer_inplace_ok(Ctx& ctx, int axis, int wire, const float* buf);
void peer_all_reduce_inplace(Ctx& ctx, int axis, float* buf, int64_t count, int wire, bool max);
// The reshard's block permutation through peer memory (group kPeerPmm, the
// ranks of this DP group): every rank stages its source block (rows x cols,
// packed with ld_stage) in its group slot, then pulls the pieces of its
// destination block from the members' slots (one kernel, after every member
// arrived). Pure copies, so bit-exact like exchange_blocks. reserve_bytes:
// the largest staged block of the group (equal on every member).
constexpr int kPeerPmm = 4;
float* peer_stage(Ctx& ctx, const float* src, int64_t lds, int64_t rows, int64_t cols, int64_t ld_stage,
                  size_t reserve_bytes);
struct PeerPiece {
  int member;       // position in the DP group (world rank mod X*Y*Z) of the provider
  int64_t src_off;  // element offset of the piece in that member's staged block
  int64_t lds;      // that block's ld_stage
  float* dst;
  int64_t ldd, rows, cols;
};
void peer_pull(Ctx& ctx, const std::vector<PeerPiece>& pieces);
// Runs f (peer_stage + peer_pull) on the reshard stream once the compute
// stream's work so far is done; the compute stream goes on until
// reshard_join. GGB_ASYNC_RESHARD=0 runs it inline.
void reshard_async(Ctx& ctx, const std::function<void()>& f);
void reshard_join(Ctx& ctx);
inline bool trivial(const Ctx& ctx, int axis) { return ctx.grid.dims[axis] == 1; }
/// A contraction's all-reduce changes values here: a multi-member group, or a
/// bf16 wire (which rounds even a single member's contribution, comm.hpp:135-145).
inline bool reduces(const Ctx& ctx, int axis, int wire) { return !trivial(ctx, axis) || wire != GGB_FP32; }

}  // namespace ggb
