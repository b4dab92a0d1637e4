// Specialised RING_DIMS kernel: the paper's multi-ring algorithm, one stage
// per grid dimension, on a per-rank communicator (grids (2,2), (2,4), (4,2),
// (2,2,2) of the B200 box).
//
// Reference: multiring_schedule (pkg/src/ringbox/multiring.py:170-211) runs a
// reduce-scatter over dimension 0, then over dimension 1 on the shrunken
// region, ... (182-197), then the all-gathers in reverse (199-209); each ring
// pass is ring_pass_transfers (ring.py:73-103) executed by _run_phases
// (runtime.py:199-267).  Here every stage is one pass over the stage's region:
//
//   RS stage s (s < m-1)  fold the d_s ring members' partials of my region
//                         after dims 0..s (pulled over NVLink, rotated order:
//                         start at my chunk index, my own value last) into my
//                         buffer -- exactly the ring's `view += payload`
//                         sequence for every element;
//   RS stage m-1          the same fold, the result pushed into every member
//                         of the last ring (its first all-gather step fused in);
//   AG stage i (m-2..0)   push my region after dims 0..i+1 (now final) into the
//                         other members of ring i (`view[:] = payload`).
//
// Synchronisation without grid-wide barriers: every stage's region is cut on
// ONE absolute tile grid of the buffer (tile k = elements [k*TE, (k+1)*TE)),
// and tile k is always processed by CTA k mod nb, on every rank and in every
// stage.  Every element a CTA touches in stage s was therefore produced, on
// every peer, by the CTA with the same index -- so each dependency is a
// MATCHED wait on one flag per (peer, CTA) instead of an ALL-CTA barrier
// (the generic step interpreter's RING_DIMS pays one ALL barrier per stage).
//
// The same engine runs MODE_PUSH (two-shot, NVLink writes only): one stage per
// peer scatters this rank's input of that peer's owned region into the peer's
// inbox, then one stage folds the owned region from the own buffer and the
// inbox slots in the nested reference order and pushes the result into every
// buffer.  Posted writes need no round trip, so with few SMs (a collective
// overlapping compute) pushes move 1.5-2x the bytes per SM that pulls do
// (profiles/r02_nvlink_few_ctas_2gpu.jsonl).
#pragma once
#include "rbx_fused.cuh"

namespace rbx {

#define RBX_RINGS_MAX_STAGES 9  // RING_DIMS: 2m-1 <= 7; PUSH: N-1 scatter stages + 1 fold (N <= 8)

struct RingStage {
  int64_t off, len;                 // element region of the stage
  const char* src[RBX_MAX_RANKS];   // RS: ring members' buffers in fold order; AG: {my buffer}
  char* dst[RBX_MAX_RANKS];         // RS: {my buffer}, last RS: ring members (rotated); AG: other ring members
  uint8_t nsrc, ndst, nwait, nsig;
  uint8_t local_only;               // every destination is this rank's own buffer (see the release below)
  uint8_t nlev;                     // nesting depth of the fold (1: one ring; PUSH folds all dims at once)
  uint8_t wait_slot, sig_slot;      // flag slots of the stage's waits and signals
  uint8_t wait_peer[RBX_MAX_RANKS]; // matched waits before the stage
  uint8_t sig_peer[RBX_MAX_RANKS];  // matched release signals after it
  uint8_t ctrl[RBX_MAX_RANKS];      // nested-fold control per operand (rbx::fold_ctrl)
};

struct RingsArgs {
  int me, nstages, nentry, nexit;
  int exit_slot;
  int group_first, group_count;     // stages [first, first+count) may run in any order (PUSH scatter)
  uint32_t* my_sig;
  uint32_t* sig[RBX_MAX_RANKS];     // every rank's signal area (mapped)
  uint8_t entry_peer[RBX_MAX_RANKS];
  uint8_t exit_peer[RBX_MAX_RANKS]; // matched exit waits (slot nstages)
  uint64_t timeout_ns;
  ErrRecord* err;
  unsigned long long* trace;
  int fault_milli;
  RingStage st[RBX_RINGS_MAX_STAGES];
};

// Tile = 128 16-byte vectors (one warp, 4 vectors per lane).  Tile k is owned by
// CTA k mod nb (the unit of the matched flags) and, inside it, by warp
// (k / nb) mod W: the ownership of every element is the same in every stage
// and on every rank, and a CTA's share of any region differs from another's
// by at most one tile.
constexpr int kRingTileVec = 128;

// One warp folds NSRC operands (single ring level) over vectors [v0, v1) (at most
// one tile), 8 loads in flight per lane; NSRC == 1 is the all-gather copy.
template <typename T, int NSRC, int NLEV>
__device__ __forceinline__ void ring_tile(const RingStage& S, int64_t v0, int64_t v1, int lane) {
  constexpr int VEC = Traits<T>::VEC;
  constexpr int U = NSRC >= 8 ? 1 : (8 / NSRC > 4 ? 4 : 8 / NSRC);
  for (int64_t p = v0 + lane; p < v1; p += (int64_t)U * 32) {
    int4 raw[U][NSRC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = p + (int64_t)u * 32;
#pragma unroll
      for (int j = 0; j < NSRC; ++j) raw[u][j] = v < v1 ? ld_stream(S.src[j] + v * 16) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = p + (int64_t)u * 32;
      int4 out;
      if (NSRC == 1) {
        out = raw[u][0];
      } else {
        FoldState<T, VEC, NLEV> f;
#pragma unroll
        for (int j = 0; j < NSRC; ++j) {
          typename Traits<T>::Acc x[VEC];
#pragma unroll
          for (int l = 0; l < VEC; ++l) x[l] = Traits<T>::lane(raw[u][j], l);
          f.feed(S.ctrl[j], x);
        }
        out = pack_result(f);
      }
      if (v < v1)
        for (int d = 0; d < S.ndst; ++d) __stcg(reinterpret_cast<int4*>(S.dst[d] + v * 16), out);
    }
  }
}

template <typename T, int NSRC, int NLEV>
__device__ __forceinline__ void ring_scalar(const RingStage& S, int64_t e) {
  using Tr = Traits<T>;
  using Bt = typename Tr::Bits;
  const int64_t byte = e * (int64_t)sizeof(T);
  Bt out;
  if (NSRC == 1) {
    out = __ldcg(reinterpret_cast<const Bt*>(S.src[0] + byte));
  } else {
    FoldState<T, 1, NLEV> f;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      typename Tr::Acc x[1] = {Tr::from_bits(__ldcg(reinterpret_cast<const Bt*>(S.src[j] + byte)))};
      f.feed(S.ctrl[j], x);
    }
    out = Tr::to_bits(f.result(0));
  }
  for (int d = 0; d < S.ndst; ++d) __stcg(reinterpret_cast<Bt*>(S.dst[d] + byte), out);
}

// CTA b's share of one stage: its warps walk the tiles they own inside the region.
// tlimit >= 0 (fault injection): at most that many tiles per warp.
template <typename T, int NSRC, int NLEV>
__device__ void ring_stage(const RingStage& S, int b, int nb, int64_t tlimit) {
  constexpr int VEC = Traits<T>::VEC;
  constexpr int64_t TE = (int64_t)kRingTileVec * VEC;  // elements per tile
  if (S.len <= 0) return;
  const int W = blockDim.x / 32, w = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t e0 = S.off, e1 = S.off + S.len;
  const int64_t k0 = e0 / TE, k1 = (e1 + TE - 1) / TE;
  // first k >= k0 with k = b (mod nb) and ((k - b) / nb) = w (mod W)
  int64_t k = k0 + (((int64_t)b - k0) % nb + nb) % nb;
  const int64_t j = (k - b) / nb;
  k += (int64_t)nb * ((((int64_t)w - j) % W + W) % W);
  int64_t done = 0;
  for (; k < k1; k += (int64_t)nb * W) {
    if (tlimit >= 0 && done++ >= tlimit) break;
    const int64_t a0 = k * TE > e0 ? k * TE : e0, a1 = (k + 1) * TE < e1 ? (k + 1) * TE : e1;
    const int64_t v0 = (a0 + VEC - 1) / VEC, v1 = a1 / VEC;  // whole vectors inside [a0, a1)
    if (v0 < v1) {
      ring_tile<T, NSRC, NLEV>(S, v0, v1, lane);
      for (int64_t e = a0 + lane; e < v0 * VEC; e += 32) ring_scalar<T, NSRC, NLEV>(S, e);
      for (int64_t e = v1 * VEC + lane; e < a1; e += 32) ring_scalar<T, NSRC, NLEV>(S, e);
    } else {
      for (int64_t e = a0 + lane; e < a1; e += 32) ring_scalar<T, NSRC, NLEV>(S, e);
    }
  }
}

template <typename T>
__device__ __forceinline__ void ring_stage_dispatch(const RingsArgs& a, const RingStage& S, int b, int nb,
                                                    int64_t tlimit) {
  switch (S.nsrc * 8 + S.nlev) {
    case 1 * 8 + 1: ring_stage<T, 1, 1>(S, b, nb, tlimit); break;
    case 2 * 8 + 1: ring_stage<T, 2, 1>(S, b, nb, tlimit); break;
    case 4 * 8 + 1: ring_stage<T, 4, 1>(S, b, nb, tlimit); break;
    case 8 * 8 + 1: ring_stage<T, 8, 1>(S, b, nb, tlimit); break;
    case 4 * 8 + 2: ring_stage<T, 4, 2>(S, b, nb, tlimit); break;  // PUSH over (2,2)
    case 8 * 8 + 2: ring_stage<T, 8, 2>(S, b, nb, tlimit); break;  // PUSH over (2,4) / (4,2)
    case 8 * 8 + 3: ring_stage<T, 8, 3>(S, b, nb, tlimit); break;  // PUSH over (2,2,2)
    default: break;
  }
}

// matched wait: thread q < n polls flags[slot][peer q][b]; false on timeout/abort (recorded)
__device__ __forceinline__ bool rings_wait(const RingsArgs& a, int n, const uint8_t* peers, int slot, int b,
                                           uint32_t e, uint64_t t0, volatile uint32_t* abort_word, int* s_fail) {
  if ((int)threadIdx.x < n) {
    const int q = peers[threadIdx.x];
    if (!fused_spin(a.my_sig + flag_index(slot, q, b), e, abort_word, t0, a.timeout_ns)) {
      *s_fail = 1;
      if (atomicCAS(&a.err->code, 0, 3) == 0) {
        a.err->rank = a.me;
        a.err->step = slot;
        a.err->peer = q;
      }
      *abort_word = 1u;
    }
  }
  __syncthreads();
  return !*s_fail;
}

template <typename T>
__global__ void __launch_bounds__(512, 1) rbx_rings_kernel(const __grid_constant__ RingsArgs a) {
  const int b = blockIdx.x, nb = gridDim.x;
  __shared__ uint32_t s_epoch;
  __shared__ int s_fail;
  pdl_wait();
  uint32_t* my_sig = a.my_sig;
  volatile uint32_t* abort_word = (volatile uint32_t*)(my_sig + SigLayout::abort_off);
  unsigned long long* tr = nullptr;
  if (a.trace && threadIdx.x == 0 && (b == 0 || b == nb - 1)) tr = a.trace + (b == 0 ? 0 : 32);
  if (tr) {
    tr[29] = tr[31];
    tr[0] = global_ns();
  }
  if (threadIdx.x == 0) {
    s_fail = 0;
    s_epoch = *(volatile uint32_t*)(my_sig + SigLayout::epoch_off) + 1u;
  }
  __syncthreads();
  const uint32_t e = s_epoch;
  const uint64_t t0 = global_ns();
  // ENTRY (slot 0): every ring partner's inputs are ready (relaxed: nothing written yet).
  // PUSH has none: no peer ever reads this rank's buffer (see rbx_plan.cpp MODE_PUSH)
  if ((int)threadIdx.x < a.nentry) st_relaxed_sys(a.sig[a.entry_peer[threadIdx.x]] + flag_index(0, a.me, b), e);
  if (a.nentry && !rings_wait(a, a.nentry, a.entry_peer, 0, b, e, t0, abort_word, &s_fail)) return;
  if (tr) tr[2] = global_ns();
  pdl_launch_dependents();
  for (int s = 0; s < a.nstages; ++s) {
    const RingStage& S = a.st[s];
    if (S.nwait && !rings_wait(a, S.nwait, S.wait_peer, S.wait_slot, b, e, t0, abort_word, &s_fail)) return;
    if (tr && s < 9) tr[3 + 3 * s] = global_ns();
    if (s == 0 && a.fault_milli >= 0) {  // injected crash: part of stage 0, then die without signalling
      const int64_t per_warp = S.len / ((int64_t)kRingTileVec * Traits<T>::VEC) / ((int64_t)nb * (blockDim.x / 32)) + 1;
      ring_stage_dispatch<T>(a, S, b, nb, per_warp * a.fault_milli / 1000);
      return;
    }
    int last = s;
    if (s == a.group_first && a.group_count > 1) {
      // a group of independent stages (PUSH: the scatter into every peer's inbox): no
      // waits between them and only the last one signals, so each CTA runs them in its
      // own rotation and at any moment the GPU's pushes go to every peer, not to one
      last = s + a.group_count - 1;
      for (int i = 0; i < a.group_count; ++i) ring_stage_dispatch<T>(a, a.st[s + (i + b) % a.group_count], b, nb, -1);
      s = last;
    } else {
      ring_stage_dispatch<T>(a, S, b, nb, -1);
    }
    const RingStage& L = a.st[last];
    if (tr && s < 9) tr[4 + 3 * s] = global_ns();
    __syncthreads();  // the release is cumulative over the CTA's writes ordered by bar.sync
    if ((int)threadIdx.x < L.nsig) {
      uint32_t* f = a.sig[L.sig_peer[threadIdx.x]] + flag_index(L.sig_slot, a.me, b);
      if (L.local_only) {
        // the stage wrote only this GPU's memory, which peers read through this GPU's L2:
        // a GPU-scope fence puts the writes there before the flag leaves (0.45 us instead
        // of the 3.7 us system-scope release that has to drain NVLink pushes)
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        st_relaxed_sys(f, e);
      } else {
        st_release_sys(f, e);
      }
    }
    if (tr && s < 9) tr[5 + 3 * s] = global_ns();
  }
  // EXIT: the last all-gather pushes into me have landed (earlier levels were waited on by
  // the stage that forwarded them), and transitively every partner is done reading me
  if (!rings_wait(a, a.nexit, a.exit_peer, a.exit_slot, b, e, t0, abort_word, &s_fail)) return;
  if (tr) tr[30] = global_ns();
  if (threadIdx.x == 0) {
    unsigned int* done = reinterpret_cast<unsigned int*>(my_sig + SigLayout::epoch_off + 1);
    if (atomicAdd(done, 1u) == (unsigned)nb - 1u) {
      *done = 0u;
      *(volatile uint32_t*)(my_sig + SigLayout::epoch_off) = e;
    }
  }
  if (tr) tr[31] = global_ns();
}

}  // namespace rbx
