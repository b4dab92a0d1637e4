// Per-rank execution plan ("stage table") for the multi-ring allreduce.
//
// The reference materialises a composite schedule of ring phases
// (pkg/src/ringbox/multiring.py:170-211) and each worker walks it with blocking
// socket transfers (pkg/src/ringbox/runtime.py:199-267).  On B200 the same
// reduction is re-expressed per rank as a short list of STEPS executed by one
// persistent kernel:
//
//   step   = { waits on peers' flags }  { segments of work }  { signals to peers }
//   segment= fold `nsrc` source buffers element-wise, in exactly the reference's
//            reduction order, over [off, off+len) and store the result into
//            `ndst` destination buffers (local or NVLink-mapped peer memory).
//
// A reduce-scatter ring phase (`view += payload`, runtime.py:248-249) becomes a
// pulled fold over the ring members (ring.py:73-103 fold order: start at the
// chunk's index, owner last), an allgather phase (`view[:] = payload`,
// runtime.py:250-251) becomes a pushed copy.  Flags are epoch-tagged, so no
// reset is ever needed and the plan can be replayed inside a CUDA graph.
//
// This header is shared by host (plan builder, CPU-testable) and device code.
#pragma once
#include <stdint.h>

#define RBX_MAX_RANKS 16
#define RBX_MAX_LEVELS 4       // non-singleton grid dims (N <= 16 -> at most 4)
#define RBX_MAX_STEPS 12
#define RBX_MAX_SEGS 384       // keeps a staged plan under the 48 KB default shared-memory window
#define RBX_MAX_WAITS 256
#define RBX_MAX_SIGS 256
#define RBX_MAX_BLOCKS 1024    // blocks per rank (flag array width)
#define RBX_NSLOTS (RBX_MAX_STEPS + 1)  // slot 0 = ENTRY, step s signals slot s+1

namespace rbx {

enum Op : int32_t { OP_ALLREDUCE = 0, OP_REDUCE_SCATTER = 1, OP_ALLGATHER = 2, OP_BARRIER = 3 };
enum Mode : int32_t {
  MODE_AUTO = 0,
  MODE_RING_DIMS = 1,
  MODE_FUSED = 2,
  MODE_FUSED_PULL = 3,
  MODE_LOCAL = 4,
  MODE_PUSH = 5  // two-shot, writes only: inputs pushed to the owners' inboxes, results pushed back
};

// Pointer-table layout per buffer in MODE_PUSH (entries relative to Seg.tbl):
//   [0, R)    every rank's buffer
//   [R, 2R)   this rank's inbox slot p (contribution of rank p to this rank's region)
//   [2R, 3R)  rank q's inbox, this rank's slot (where this rank pushes q's region)
// Other modes use only [0, R).
inline int table_entries(int mode, int nranks) { return mode == MODE_PUSH ? 3 * nranks : nranks; }

struct Seg {
  int64_t off, len;        // element range [off, off+len)
  int64_t vec_begin;       // prefix sum of body vectors within the step
  int64_t body_off;        // first element of the 16-byte aligned body
  int64_t nvec;            // body vectors
  int32_t head, tail;      // scalar elements before / after the body
  int32_t tbl;             // base index of this segment's buffer in the pointer table
  uint8_t nsrc, ndst, nlev;
  uint8_t acc;             // bit0: sources are fp32 partials, bit1: destinations are (bf16/f16 ring_dims)
  uint8_t src[RBX_MAX_RANKS];   // ranks, in fold order
  uint8_t dst[RBX_MAX_RANKS];   // ranks to store the result into
  uint8_t ctrl[RBX_MAX_RANKS];  // nested-fold control: bits0-3 "level L starts", bits4-5 levels passing up
};

struct Wait {
  uint8_t slot, peer, all, pad;  // all=1: every block of `peer` must have signalled; 0: matching block only
};

struct Step {
  int32_t seg0, nseg;
  int32_t wait0, nwait;
  int32_t sig0, nsig;      // signals go to slot (step index + 1) of each listed peer
  int32_t tile, pad_;      // work tile of this step in vectors (0: the plan's tile)
  int64_t total_vec;
};

// Device-resident plan of ONE rank.  Pointers are filled in by the runtime.
struct alignas(16) Plan {  // 16-byte multiple: plans[v] is staged with int4 loads
  int32_t me, nranks, nsteps, nentry;
  int32_t nosync, vec;     // vec = elements per 16-byte vector for this dtype
  int32_t nblocks, tile;   // tile: vectors per round-robin work tile (0 = one contiguous range per CTA)
  int32_t dyn;             // after its first tile a CTA claims the next tile from a per-step counter
  int32_t tail_split;      // dyn: the last nb tiles' worth of a step is cut into tiles this many times smaller
  int32_t fence_every, pad2_;  // dyn: fence.sys after every this many tiles (bounds writes in flight; 0 = never)
  uint8_t entry_peers[RBX_MAX_RANKS];
  uint32_t* sig[RBX_MAX_RANKS];   // signal area of every rank (mapped)
  uint32_t* my_sig;               // == sig[me]
  void* const* ptrs;              // pointer table (device array)
  Step steps[RBX_MAX_STEPS];
  Wait waits[RBX_MAX_WAITS];
  uint8_t sigs[RBX_MAX_SIGS];
  Seg segs[RBX_MAX_SEGS];
};

static_assert(sizeof(Plan) % 16 == 0, "plans are staged into shared memory with 16-byte loads");

// Signal-area layout (uint32 words) of one rank.
struct SigLayout {
  static constexpr int64_t flags_words = (int64_t)RBX_NSLOTS * RBX_MAX_RANKS * RBX_MAX_BLOCKS;
  static constexpr int64_t epoch_off = flags_words;            // epoch[RBX_MAX_BLOCKS]: [0] epoch, [1] exit count
  static constexpr int64_t tiles_off = epoch_off + 16;         // per-step tile counters (dynamic work tiles)
  static constexpr int64_t abort_off = epoch_off + RBX_MAX_BLOCKS;
  static constexpr int64_t words = abort_off + 32;
  static constexpr int64_t bytes = words * 4;
};

#ifdef __CUDACC__
__host__ __device__
#endif
inline int64_t flag_index(int slot, int from_rank, int block) {
  return ((int64_t)slot * RBX_MAX_RANKS + from_rank) * RBX_MAX_BLOCKS + block;
}

}  // namespace rbx

#ifndef __CUDACC_RTC__
#include <string>
#include <vector>

namespace rbx {

struct Geometry {
  std::vector<int> dims;  // as given (may contain 1s)
  int nranks = 1;
  bool init(const int* d, int nd, std::string* err);
  void coords(int rank, int* c) const;
  int rank_of(const int* c) const;
  std::vector<int> ring(int rank, int dim) const;  // ordered by coord[dim]
  std::vector<int> active_dims() const;            // indices with d > 1
};

void chunk_bounds(int64_t count, int64_t n, int64_t i, int64_t* off, int64_t* len);
// region owned by `rank` after reduce-scatter over dims [0, upto) (runtime.py:187-196)
void region_after(const Geometry& g, int rank, int64_t count, int upto_active, int64_t* off, int64_t* len);
// ranks in the order the reference's schedule folds them for `rank`'s owned region
std::vector<int> fold_order(const Geometry& g, int rank);
std::vector<uint8_t> fold_ctrl(const Geometry& g);  // per position in fold_order

struct PlanSpec {
  Op op = OP_ALLREDUCE;
  Mode mode = MODE_FUSED;
  int vec = 4;             // elements per 16B vector of the dtype
  bool partials_fp32 = false;  // RING_DIMS with bf16/f16: inter-stage partials in fp32 workspaces
                               // (table entries [R, 2R) = every rank's workspace)
  int mis = 0;             // (base address % 16) / itemsize, same on every rank; -1: never vectorise
  int64_t lo = 0, hi = -1; // element window [lo, hi) (hi < 0: whole buffer)
  int nblocks = 148;
};

// Append the plan of `rank` for one buffer (pointer-table base `tbl`) to `p`.
// Multiple buffers (bucket lists) are merged step-by-step: call once per
// buffer with the same spec; the step structure must match.
bool build_plan(const Geometry& g, int rank, int64_t count, const PlanSpec& spec, int tbl, Plan* p,
                bool first, std::string* err);
// Local (single-GPU, no synchronisation) plan over all virtual ranks' buffers.
bool build_local_plan(const Geometry& g, int64_t count, int vec, int mis, int nblocks, Plan* p, std::string* err,
                      int64_t lo = 0, int64_t hi = -1);
// Flatten a plan into int64s for host-side inspection (tests).
int64_t describe_plan(const Plan& p, int64_t* out, int64_t cap);

// MODE_PUSH inbox geometry of one buffer: every owner keeps one slot per rank,
// each large enough for the largest owned region plus a 16-byte phase pad.
int64_t inbox_slot_bytes(const Geometry& g, int64_t count, int itemsize);
inline int64_t inbox_buffer_bytes(const Geometry& g, int64_t count, int itemsize) {
  return (int64_t)g.nranks * inbox_slot_bytes(g, count, itemsize);
}

}  // namespace rbx
#endif
