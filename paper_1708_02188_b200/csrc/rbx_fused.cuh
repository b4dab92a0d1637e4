// Specialised FUSED allreduce kernel: the hot path of a per-rank communicator
// (configs 1-3 of BASELINE.json, the bench, DDP buckets).
//
// Reference: one allreduce walks the composite multi-ring schedule
// (pkg/src/ringbox/multiring.py:170-211) through _run_phases
// (pkg/src/ringbox/runtime.py:199-267): reduce-scatter phases `view += payload`
// (248-249) then all-gather phases `view[:] = payload` (250-251).  Here one
// launch does all of it for the rank's owned region (runtime.py:187-196):
//
//   ENTRY   every CTA tells its matched CTA on every peer "my inputs are
//           ready" (relaxed sys store) and waits for the same from them;
//   FOLD    16-byte loads of the region from all N buffers (own HBM + N-1
//           NVLink-mapped peers), folded in registers in the reference's
//           nested order (FoldState, rbx_kernel.cuh), the result stored with
//           16-byte stores into all N buffers -- reduce-scatter and all-gather
//           in one pass, bit-identical to replay().  The same loop with one
//           destination (my buffer) is reduce_scatter alone (runtime.py:
//           278-284); with one source (my region) and the N-1 peers as
//           destinations it is allgather alone (runtime.py:287-292);
//   EXIT    st.release.sys "my pushes landed / I am done reading you" to the
//           matched CTA of every peer, then wait for theirs.
//
// Compared with the generic step interpreter (rbx_step_kernel) this kernel
// is a straight loop with the fold width and nesting depth as template
// parameters: no plan in shared memory, no call boundary, no spills (the
// interpreter's __noinline__ fold bodies spilled their operand arrays), all
// loads of a pass issued before any arithmetic, and work tiles claimed
// dynamically so CTAs that get more NVLink bandwidth take more tiles.
// Programmatic dependent launch lets the CTAs become resident while the
// previous kernel on the stream drains; griddepcontrol.wait precedes every
// read of memory another kernel wrote.
#pragma once
#include "rbx_kernel.cuh"

namespace rbx {

#ifndef RBX_FUSED_LD
#define RBX_FUSED_LD 8  // 16-byte loads in flight per thread per pass
#endif

struct FusedSeg {
  int64_t vec_begin, nvec, body_off;  // body vectors of the region (step vector space) and first body element
  int64_t off;                        // first element of the region (scalar head starts here)
  int32_t head, tail;                 // scalar elements before / after the body
  const char* src[RBX_MAX_RANKS];     // every rank's buffer, in fold order
  char* dst[RBX_MAX_RANKS];           // every rank's buffer, rotated after me
};

template <int MAXSEG>
struct FusedArgsT {
  int nseg, me, npeers;
  int64_t total_vec;
  uint32_t* my_sig;
  uint32_t* peer_sig[RBX_MAX_RANKS];  // signal areas of the peers (mapped), in peer_rank order
  uint8_t peer_rank[RBX_MAX_RANKS];
  uint8_t ctrl[RBX_MAX_RANKS];        // nested-fold control per fold position (rank independent)
  uint64_t timeout_ns;
  ErrRecord* err;
  unsigned long long* trace;
  int fault_milli;                    // rbx_comm_inject_fault: -1 off
  int dbg;                            // experiment knobs (env RBX_FUSED_DBG; 0 in production): bit0 relaxed
                                      // exit signal, bit1 no exit wait, bit2 fence.sys before exit, bit3 no entry,
                                      // bit4 static round-robin tiles instead of dynamic claiming (safe)
  FusedSeg seg[MAXSEG];
};


// One pass of U vectors per thread starting at step vector `lo`: all NSRC x U
// loads first, then the folds, then NDST x U stores.  FULL: every vector is in
// range and in segment `s0` (no predicates, no segment search).  NSRC == 1 is a
// copy (the all-gather half): the loaded bits are stored as they are.
template <typename T, int NSRC, int NLEV, int NDST, int U, bool FULL, int MAXSEG>
__device__ __forceinline__ void fused_pass(const FusedArgsT<MAXSEG>& a, int s0, int64_t lo) {
  constexpr int VEC = Traits<T>::VEC;
  int4 raw[U][NSRC];
  int seg[U];
  int64_t byte[U];
  bool ok[U];
  int s = s0;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t v = lo + (int64_t)u * blockDim.x + threadIdx.x;
    if (FULL) {
      ok[u] = true;
      seg[u] = s0;
    } else {
      ok[u] = v < a.total_vec;
      if (MAXSEG > 1)
        while (s + 1 < a.nseg && v >= a.seg[s].vec_begin + a.seg[s].nvec) ++s;
      seg[u] = s;
    }
    const FusedSeg& sg = a.seg[seg[u]];
    byte[u] = (sg.body_off + (v - sg.vec_begin) * VEC) * (int64_t)sizeof(T);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const FusedSeg& sg = a.seg[seg[u]];
#pragma unroll
    for (int j = 0; j < NSRC; ++j) raw[u][j] = ok[u] ? ld_stream(sg.src[j] + byte[u]) : make_int4(0, 0, 0, 0);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    int4 packed;
    if constexpr (NSRC == 1) {
      packed = raw[u][0];
    } else {
      FoldState<T, VEC, NLEV> st;
#pragma unroll
      for (int j = 0; j < NSRC; ++j) {
        typename Traits<T>::Acc x[VEC];
#pragma unroll
        for (int l = 0; l < VEC; ++l) x[l] = Traits<T>::lane(raw[u][j], l);
        st.feed(a.ctrl[j], x);
      }
      packed = pack_result(st);
    }
    if (ok[u]) {
      const FusedSeg& sg = a.seg[seg[u]];
#pragma unroll
      for (int d = 0; d < NDST; ++d) __stcg(reinterpret_cast<int4*>(sg.dst[d] + byte[u]), packed);
    }
  }
}

// spin until *f >= e (epoch-tagged); false on timeout / abort
__device__ __forceinline__ bool fused_spin(const uint32_t* f, uint32_t e, volatile uint32_t* abort_word, uint64_t t0,
                                           uint64_t timeout_ns) {
  uint32_t it = 0;
  while (!flag_reached(ld_relaxed_sys(f), e)) {
    if ((++it & 255u) == 0) {
      if (*abort_word) return false;
      if (global_ns() - t0 > timeout_ns) return false;
      __nanosleep(32);
    }
  }
  (void)ld_acquire_sys(f);
  return true;
}

// one element of a misaligned region edge, same fold (a copy when NSRC == 1)
template <typename T, int NSRC, int NLEV, int NDST, int MAXSEG>
__device__ __forceinline__ void fused_scalar(const FusedArgsT<MAXSEG>& a, const FusedSeg& sg, int64_t elem) {
  using Tr = Traits<T>;
  using Bt = typename Tr::Bits;
  const int64_t byte = elem * (int64_t)sizeof(T);
  Bt out;
  if constexpr (NSRC == 1) {
    out = __ldcg(reinterpret_cast<const Bt*>(sg.src[0] + byte));
  } else {
    FoldState<T, 1, NLEV> st;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      typename Tr::Acc x[1] = {Tr::from_bits(__ldcg(reinterpret_cast<const Bt*>(sg.src[j] + byte)))};
      st.feed(a.ctrl[j], x);
    }
    out = Tr::to_bits(st.result(0));
  }
#pragma unroll
  for (int d = 0; d < NDST; ++d) __stcg(reinterpret_cast<Bt*>(sg.dst[d] + byte), out);
}

#ifndef RBX_FUSED_RS_LD
#define RBX_FUSED_RS_LD 16  // the same for reduce-scatter alone (loads only, one local store)
#endif

// vectors per thread per pass for a fold of nsrc operands into ndst buffers (the
// deeper reduce-scatter pass spills the 64-bit accumulators of 8-byte types; the
// 7-destination copy of a bucket list spills its segment bookkeeping at 8)
template <typename T>
__host__ __device__ constexpr int fused_unroll(int nsrc, int ndst, int maxseg) {
  const int ld = (ndst == 1 && nsrc > 1 && sizeof(T) < 8) ? RBX_FUSED_RS_LD
                 : (nsrc == 1 && ndst >= 7 && maxseg > 1) ? RBX_FUSED_LD / 2
                                                          : RBX_FUSED_LD;
  return ld / nsrc > 0 ? ld / nsrc : 1;
}

template <typename T, int NSRC, int NLEV, int NDST, int MAXSEG>
__global__ void __launch_bounds__(512, 1) rbx_fused_kernel(const __grid_constant__ FusedArgsT<MAXSEG> a) {
  constexpr int U = fused_unroll<T>(NSRC, NDST, MAXSEG);
  const int b = blockIdx.x, nb = gridDim.x;
  __shared__ uint32_t s_epoch;
  __shared__ int s_fail, s_next;
  const uint64_t t_start = global_ns();
  // nothing above touched memory: from here on we read memory the previous kernel
  // on the stream may have written (programmatic dependent launch)
  pdl_wait();
  unsigned long long* tr = nullptr;
  if (a.trace && threadIdx.x == 0 && (b == 0 || b == nb - 1)) tr = a.trace + (b == 0 ? 0 : 32);
  if (tr) {  // timeline: [0] start [3] dependency resolved [1] epoch read [2] entry done [4] folded
             // [5] released [30] exit flags seen [31] exit; [29] previous launch's exit
    tr[29] = tr[31];
    tr[0] = t_start;
    tr[3] = global_ns();
  }
  uint32_t* my_sig = a.my_sig;
  volatile uint32_t* abort_word = (volatile uint32_t*)(my_sig + SigLayout::abort_off);
  if (threadIdx.x == 0) {
    s_fail = 0;
    s_epoch = *(volatile uint32_t*)(my_sig + SigLayout::epoch_off) + 1u;
  }
  __syncthreads();
  const uint32_t e = s_epoch;
  const uint64_t t0 = global_ns();
  if (tr) tr[1] = t0;
  // ENTRY (slot 0): relaxed -- nothing of this launch has been written yet
  if ((int)threadIdx.x < a.npeers && !(a.dbg & 8)) st_relaxed_sys(a.peer_sig[threadIdx.x] + flag_index(0, a.me, b), e);
  if ((int)threadIdx.x < a.npeers && !(a.dbg & 8)) {
    const int q = a.peer_rank[threadIdx.x];
    if (!fused_spin(my_sig + flag_index(0, q, b), e, abort_word, t0, a.timeout_ns)) {
      s_fail = 1;
      if (atomicCAS(&a.err->code, 0, 3) == 0) {
        a.err->rank = a.me;
        a.err->step = 0;
        a.err->peer = q;
      }
      *abort_word = 1u;
    }
  }
  __syncthreads();
  if (s_fail) return;
  if (tr) tr[2] = global_ns();
  // every CTA of this grid is resident: a dependent kernel may start its prologue
  pdl_launch_dependents();

  // FOLD: tile t = vectors [t*tile, (t+1)*tile); CTA b starts with tile b, then claims
  // nb, nb+1, ... from the per-launch counter (claim issued before the tile's loads)
  const int64_t tile = (int64_t)U * blockDim.x;  // one pass of the block
  const int64_t ntiles = (a.total_vec + tile - 1) / tile;
  const int64_t tlimit = a.fault_milli < 0 ? ntiles : ntiles * a.fault_milli / 1000;
  unsigned int* ctr = reinterpret_cast<unsigned int*>(my_sig + SigLayout::tiles_off);
  for (int64_t t = b; t < tlimit;) {
    unsigned int nxt = 0;
    if (threadIdx.x == 0 && ntiles > nb && !(a.dbg & 16)) nxt = (unsigned)nb + atomicAdd(ctr, 1u);
    const int64_t lo = t * tile;
    int s_cur = 0;  // segment of the tile's first vector
    if (MAXSEG > 1)
      while (s_cur + 1 < a.nseg && lo >= a.seg[s_cur].vec_begin + a.seg[s_cur].nvec) ++s_cur;
    const FusedSeg& sg = a.seg[s_cur];
    const bool full_tile = lo + tile <= a.total_vec && (MAXSEG == 1 || lo + tile <= sg.vec_begin + sg.nvec);
    for (int64_t p = lo; p < lo + tile; p += (int64_t)U * blockDim.x) {
      if (full_tile)
        fused_pass<T, NSRC, NLEV, NDST, U, true, MAXSEG>(a, s_cur, p);
      else
        fused_pass<T, NSRC, NLEV, NDST, U, false, MAXSEG>(a, s_cur, p);
    }
    if (ntiles <= nb) break;  // one tile per CTA, no counter
    if (a.dbg & 16) {         // A/B: static round-robin ownership (CTA b: tiles b, b+nb, ...)
      t += nb;
      continue;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_next = (int)nxt;
    __syncthreads();
    t = s_next;
  }
  if (a.fault_milli >= 0) return;  // injected crash: no signals, the epoch is not advanced
  // scalar head/tail of segment k (misaligned region edges): CTA k mod nb
  for (int k = b % nb; k < a.nseg; k += nb) {
    const FusedSeg& sg = a.seg[k];
    for (int i = threadIdx.x; i < sg.head + sg.tail; i += blockDim.x)
      fused_scalar<T, NSRC, NLEV, NDST, MAXSEG>(
          a, sg, i < sg.head ? sg.off + i : sg.body_off + sg.nvec * Traits<T>::VEC + (i - sg.head));
  }
  if (tr) tr[4] = global_ns();
  // EXIT (slot 1): release my pushes to every peer's matched CTA, then wait for theirs.
  // st.release.sys is cumulative over the CTA's writes ordered before it by bar.sync.
  __syncthreads();
  if ((int)threadIdx.x < a.npeers) {
    if (a.dbg & 1)
      st_relaxed_sys(a.peer_sig[threadIdx.x] + flag_index(1, a.me, b), e);
    else
      st_release_sys(a.peer_sig[threadIdx.x] + flag_index(1, a.me, b), e);
  }
  if (tr) tr[5] = global_ns();
  if ((int)threadIdx.x < a.npeers && !(a.dbg & 2)) {
    const int q = a.peer_rank[threadIdx.x];
    if (!fused_spin(my_sig + flag_index(1, q, b), e, abort_word, t0, a.timeout_ns)) {
      s_fail = 1;
      if (atomicCAS(&a.err->code, 0, 3) == 0) {
        a.err->rank = a.me;
        a.err->step = 1;
        a.err->peer = q;
      }
      *abort_word = 1u;
    }
  }
  __syncthreads();
  if (s_fail) return;
  if (tr) tr[30] = global_ns();
  // the last CTA to finish rewinds the tile counter and publishes the epoch (the next
  // launch on the stream starts after this one completes, so no fence is needed)
  if (threadIdx.x == 0) {
    unsigned int* done = reinterpret_cast<unsigned int*>(my_sig + SigLayout::epoch_off + 1);
    if (atomicAdd(done, 1u) == (unsigned)nb - 1u) {
      *done = 0u;
      *ctr = 0u;
      *(volatile uint32_t*)(my_sig + SigLayout::epoch_off) = e;
    }
  }
  if (a.dbg & 4) __threadfence_system();
  if (tr) tr[31] = global_ns();
}

// (operand count, nesting depth, destinations) with a specialised kernel, for
// every factorization of the B200 box's 2, 4 and 8 GPUs: allreduce (fold N,
// store N), reduce-scatter (fold N, store 1), all-gather (copy 1, store N-1).
#define RBX_FUSED_SHAPES(X)                                                                    \
  X(2, 1, 2) X(4, 1, 4) X(4, 2, 4) X(8, 1, 8) X(8, 2, 8) X(8, 3, 8)                            \
  X(2, 1, 1) X(4, 1, 1) X(4, 2, 1) X(8, 1, 1) X(8, 2, 1) X(8, 3, 1)                            \
  X(1, 1, 1) X(1, 1, 3) X(1, 1, 7)
#define RBX_FUSED_MAXSEG 16

}  // namespace rbx

