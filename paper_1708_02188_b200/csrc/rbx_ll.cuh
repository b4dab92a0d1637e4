// Low-latency (LL) allreduce for small messages: one launch, no flags, no
// fences, no entry barrier.
//
// Every datum travels as one 8-byte word {payload u32, epoch u32} stored with a
// single 64-bit relaxed.sys store, which is single-copy atomic, so a receiver
// that sees the current epoch in the upper half also sees the payload: the
// data carries its own ready flag.  That removes the st.release.sys /
// ld.acquire.sys pair (~4 us of fence per step on B200, tools/entry_probe.cu)
// and the ENTRY handshake: no peer ever touches this rank's buffer.
//
//   1. scatter: every element of peer q's owned region goes into q's LL area,
//      slot [me] (one word per 2/4-byte element, two per 8-byte element);
//   2. fold: for my owned region, fold my buffer and the N-1 slots in the
//      reference order (FUSED's nested rotated fold, rbx_plan.cpp fold_order /
//      fold_ctrl) -- bit-identical to every other mode; store the result into
//      my buffer and push it as LL words into every peer's gather slot [me];
//   3. gather: copy every peer's owned result from my gather slots.
//
// ONE-SHOT variant (tiny buffers, and N = 2 where it moves the same bytes):
// every rank pushes its whole buffer to every peer and then folds EVERY
// element itself, each owned region in its owner's reference order, so all
// ranks compute the same bits with one NVLink hop instead of two.  Its slots
// are double-buffered by epoch parity: rank r can only be one launch ahead of
// a peer that has not finished reading (r's launch e+1 needs that peer's
// words of launch e+1, sent after the peer's launch e completed).
//
// Slot reuse needs no credits: rank r's next launch starts only after this one
// saw every owner's result for every element, and an owner produces element
// i's result only after reading r's word i.  Allreduce only (reduce-scatter
// alone would break that argument).
//
// Reference mapping: one LL launch = the whole phase loop of _run_phases
// (pkg/src/ringbox/runtime.py:199-267) for a small buffer; the epoch in every
// word plays the role of the frame header check (runtime.py:229-245).
#pragma once
#include "rbx_kernel.cuh"

namespace rbx {

#define RBX_LL_MAX_BYTES (1 << 20)       // per-rank payload cap of two-shot LL (bytes of the user buffer)
#define RBX_LL_ONESHOT_MAX_BYTES (1 << 16)  // per-rank payload cap of one-shot LL

// LL area of one rank (u64 words): two-shot scatter[R][cap] and gather[R][cap],
// then one-shot slots[2 parities][R][cap1].
__host__ __device__ inline int64_t ll_cap_words(int nranks) {
  return (RBX_LL_MAX_BYTES / 2 + nranks - 1) / nranks + 16;
}
__host__ __device__ inline int64_t ll_cap1_words() { return RBX_LL_ONESHOT_MAX_BYTES / 2; }
__host__ __device__ inline int64_t ll_oneshot_off(int nranks) { return 2 * (int64_t)nranks * ll_cap_words(nranks); }
__host__ __device__ inline int64_t ll_area_bytes(int nranks) {
  return (ll_oneshot_off(nranks) + 2 * (int64_t)nranks * ll_cap1_words()) * 8;
}

struct LLRank {
  char* buf;                            // this rank's buffer (only this rank touches it)
  unsigned long long* area[RBX_MAX_RANKS];  // every rank's LL area, mapped ([me] = own)
  uint32_t* my_sig;                     // epoch word, done counter, abort word
  int64_t off[RBX_MAX_RANKS], len[RBX_MAX_RANKS];  // owned regions (elements)
  uint8_t order[RBX_MAX_RANKS], ctrl[RBX_MAX_RANKS];  // fold order of my region
  int me;
};

struct LLOrders {  // one-shot: the fold order of every owner's region
  uint8_t of[RBX_MAX_RANKS][RBX_MAX_RANKS];
};

// MAXV: ranks hosted by one launch (1 for a per-rank communicator, up to 16 for
// a virtual one).  The per-rank form keeps the kernel parameters under 1 KB;
// the 16-rank form is ~7.5 KB, which measurably slows the host-side launch.
template <int MAXV>
struct LLArgsT {
  int nranks, nlev, nb;  // nb CTAs per rank
  int nhosted;           // ranks hosted by this launch
  int oneshot;           // 1: one-shot variant
  int fault;             // fault injection (runtime.py:429-432): -1 off, 0 die at entry, 1 die after the scatter
  int64_t cap;           // words per slot
  uint64_t timeout_ns;
  ErrRecord* err;
  unsigned long long* trace;  // optional timeline (RBX_TRACE), same slots as rbx_step_kernel
  LLOrders orders;
  LLRank rank[MAXV];
};
using LLArgs = LLArgsT<RBX_MAX_RANKS>;

__device__ __forceinline__ void st_ll(unsigned long long* p, uint32_t data, uint32_t e) {
  const unsigned long long v = ((unsigned long long)e << 32) | data;
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_ll(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// LL word format of a dtype.  A fold UNIT is what one thread folds at once:
// 2-byte types pack two elements per 32-bit payload (unit = 1 word, 2 lanes),
// 4-byte types one element per word, 8-byte types one element in two words.
// Words of a region are numbered from the region's first element; a region of
// `len` elements has nunits(len) * WPU words, never more than len * WPU, so
// element-offset based slot addressing (one-shot) cannot overlap.
template <typename T>
struct LLFmt {
  static constexpr int ES = sizeof(T);
  static constexpr int WPU = ES == 8 ? 2 : 1;  // words per unit
  static constexpr int LPU = ES == 2 ? 2 : 1;  // lanes (elements) per unit
  using Acc = typename Traits<T>::Acc;
  __device__ static int64_t nunits(int64_t len) { return ES == 2 ? (len + 1) / 2 : len; }
  __device__ static int64_t nwords(int64_t len) { return nunits(len) * WPU; }
  // payload of word w of the region [o, o+len) of buf
  __device__ static uint32_t load(const char* buf, int64_t o, int64_t len, int64_t w) {
    if (ES == 2) {
      const unsigned short* p = reinterpret_cast<const unsigned short*>(buf) + o + 2 * w;
      const uint32_t lo = __ldcg(p);
      const uint32_t hi = 2 * w + 1 < len ? (uint32_t)__ldcg(p + 1) : 0u;
      return lo | (hi << 16);
    }
    return __ldcg(reinterpret_cast<const unsigned int*>(buf + o * (int64_t)ES) + w);
  }
  __device__ static void store(char* buf, int64_t o, int64_t len, int64_t w, uint32_t v) {
    if (ES == 2) {
      unsigned short* p = reinterpret_cast<unsigned short*>(buf) + o + 2 * w;
      p[0] = (unsigned short)v;
      if (2 * w + 1 < len) p[1] = (unsigned short)(v >> 16);
      return;
    }
    reinterpret_cast<unsigned int*>(buf + o * (int64_t)ES)[w] = v;
  }
  __device__ static void lanes(const uint32_t (&w)[WPU], Acc (&x)[LPU]) {
    using B = typename Traits<T>::Bits;
    if (ES == 2) {
      x[0] = Traits<T>::from_bits((B)(w[0] & 0xffffu));
      x[LPU - 1] = Traits<T>::from_bits((B)(w[0] >> 16));
    } else if (ES == 8) {
      x[0] = Traits<T>::from_bits((B)(((unsigned long long)w[WPU - 1] << 32) | w[0]));
    } else {
      x[0] = Traits<T>::from_bits((B)w[0]);
    }
  }
  __device__ static void pack(const Acc (&x)[LPU], uint32_t (&w)[WPU]) {
    if (ES == 2) {
      w[0] = (uint32_t)Traits<T>::to_bits(x[0]) | ((uint32_t)Traits<T>::to_bits(x[LPU - 1]) << 16);
    } else if (ES == 8) {
      const unsigned long long b = (unsigned long long)Traits<T>::to_bits(x[0]);
      w[0] = (uint32_t)b;
      w[WPU - 1] = (uint32_t)(b >> 32);
    } else {
      w[0] = (uint32_t)Traits<T>::to_bits(x[0]);
    }
  }
};

struct LLWait {
  uint32_t e;
  uint64_t t0, timeout_ns;
  volatile uint32_t* abort_word;
  bool failed;
  int peer;  // rank whose word timed out first (-1: the abort word was raised elsewhere)
  // payload of the word at p (written by rank `from`) once its epoch is current
  // (0 on timeout/abort, failed set)
  __device__ __forceinline__ uint32_t get(const unsigned long long* p, int from) {
    uint32_t it = 0;
    while (true) {
      const unsigned long long v = ld_ll(p);
      if ((uint32_t)(v >> 32) == e) return (uint32_t)v;
      if (failed) return 0;
      if ((++it & 1023u) == 0) {
        if (*abort_word || global_ns() - t0 > timeout_ns) {
          failed = true;
          if (!*abort_word) peer = from;
          return 0;
        }
      }
    }
  }
};

// Fold unit u of the region [o, o+len) from N sources in `order` (my own words
// straight from buf, the others from LL slots: slot(p) + word index), then
// return the packed result words.
template <typename T, typename SlotFn>
__device__ __forceinline__ void ll_fold_unit(const LLRank& R, const uint8_t* order, int N, int nlev, int64_t o,
                                             int64_t len, int64_t u, SlotFn slot, LLWait& wt,
                                             uint32_t (&res)[LLFmt<T>::WPU]) {
  using F = LLFmt<T>;
  using Acc = typename Traits<T>::Acc;
  constexpr int WPU = F::WPU, LPU = F::LPU;
  const uint32_t e = wt.e;
  // issue every source's word(s) at once, then re-poll the ones not yet current
  unsigned long long raw[RBX_MAX_RANKS][WPU];
#pragma unroll
  for (int k = 0; k < RBX_MAX_RANKS; ++k) {
    if (k < N) {
      const int p = order[k];
#pragma unroll
      for (int j = 0; j < WPU; ++j)
        raw[k][j] = p == R.me ? (((unsigned long long)e << 32) | F::load(R.buf, o, len, u * WPU + j))
                              : ld_ll(slot(p) + u * WPU + j);
    }
  }
  FoldState<T, LPU, RBX_MAX_LEVELS> f;
#pragma unroll
  for (int k = 0; k < RBX_MAX_RANKS; ++k) {
    if (k < N) {
      const int p = order[k];
      uint32_t w[WPU];
#pragma unroll
      for (int j = 0; j < WPU; ++j)
        w[j] = (uint32_t)(raw[k][j] >> 32) == e ? (uint32_t)raw[k][j] : wt.get(slot(p) + u * WPU + j, p);
      Acc x[LPU];
      F::lanes(w, x);
      f.feed(R.ctrl[k], x);
    }
  }
  // the result sits at level nlev-1; carry it up to the top level with selects on
  // static indices (picking f.a[nlev-1] directly made ptxas index a local-memory
  // copy of the accumulators for 2-lane units)
#pragma unroll
  for (int L = 1; L < RBX_MAX_LEVELS; ++L) {
    const bool above = L >= nlev;
#pragma unroll
    for (int l = 0; l < LPU; ++l) f.a[L][l] = above ? f.a[L - 1][l] : f.a[L][l];
  }
  Acc r[LPU];
#pragma unroll
  for (int l = 0; l < LPU; ++l) r[l] = f.a[RBX_MAX_LEVELS - 1][l];
  F::pack(r, res);
}

template <typename T, int MAXV>
__global__ void __launch_bounds__(512, 1) rbx_ll_kernel(const __grid_constant__ LLArgsT<MAXV> a) {
  using F = LLFmt<T>;
  constexpr int WPU = F::WPU;
  constexpr int U = 4;  // words per thread in flight (scatter / gather)
  const int v = blockIdx.x / a.nb, b = blockIdx.x % a.nb;
  const LLRank& R = a.rank[v];
  const int N = a.nranks, me = R.me;
  const int64_t cap = a.cap;
  __shared__ int s_fail, s_peer;
  pdl_wait();  // before any memory access (programmatic dependent launch)
  // timeline of thread 0 of the first and last CTA of the first hosted rank:
  // [0] start [1] epoch read [3] pushed [4] folded [5] gathered [30] done [31] exit
  unsigned long long* tr = nullptr;
  if (a.trace && threadIdx.x == 0 && v == 0 && (b == 0 || b == a.nb - 1)) tr = a.trace + (b == 0 ? 0 : 32);
  if (tr) {
    tr[29] = tr[31];
    tr[0] = global_ns();
  }
  if (threadIdx.x == 0) {
    s_fail = 0;
    s_peer = -1;
  }
  __syncthreads();
  pdl_launch_dependents();
  if (a.fault == 0) return;  // injected crash before any data moved
  // every thread reads the epoch itself (one broadcast load, no barrier behind it), so
  // its latency overlaps the first data loads instead of preceding them.  It cannot
  // change during this launch: the last CTA to finish publishes the next one.
  const uint32_t e0 = *(volatile uint32_t*)(R.my_sig + SigLayout::epoch_off) + 1u;
  LLWait wt{e0, global_ns(), a.timeout_ns, (volatile uint32_t*)(R.my_sig + SigLayout::abort_off), false, -1};
  if (tr) tr[1] = global_ns();
  const uint32_t e = wt.e;
  const int64_t tid = (int64_t)b * blockDim.x + threadIdx.x, nthr = (int64_t)a.nb * blockDim.x;
  unsigned long long* own = R.area[me];

  if (a.oneshot) {
    // my whole buffer -> every peer's slot [parity][me]; then fold every unit.
    // The same thread pushes and folds unit u of region q (it overwrites it last).
    const int64_t par = (int64_t)(e & 1u) * N * ll_cap1_words();
    for (int q = 0; q < N; ++q) {
      const int64_t o = R.off[q], len = R.len[q], nu = F::nunits(len);
      for (int64_t u = tid; u < nu; u += nthr) {
#pragma unroll
        for (int j = 0; j < WPU; ++j) {
          const uint32_t d = F::load(R.buf, o, len, u * WPU + j);
          for (int k = 1; k < N; ++k)
            st_ll(R.area[(me + k) % N] + ll_oneshot_off(N) + par + (int64_t)me * ll_cap1_words() + o * WPU + u * WPU + j,
                  d, e);
        }
      }
    }
    if (tr) tr[3] = global_ns();
    if (a.fault > 0) return;  // injected crash after the push
    const unsigned long long* slots = own + ll_oneshot_off(N) + par;
    for (int q = 0; q < N; ++q) {
      const int64_t o = R.off[q], len = R.len[q], nu = F::nunits(len);
      auto slot = [&](int p) { return slots + (int64_t)p * ll_cap1_words() + o * WPU; };
      for (int64_t u = tid; u < nu; u += nthr) {
        uint32_t res[WPU];
        ll_fold_unit<T>(R, a.orders.of[q], N, a.nlev, o, len, u, slot, wt, res);
        if (!wt.failed) {
#pragma unroll
          for (int j = 0; j < WPU; ++j) F::store(R.buf, o, len, u * WPU + j, res[j]);
        }
      }
    }
    if (tr) tr[4] = tr[5] = global_ns();
  } else {
    // 1. scatter my input of every peer's region into that peer's slot [me]
    for (int k = 1; k < N; ++k) {
      const int q = (me + k) % N;
      const int64_t o = R.off[q], len = R.len[q], nw = F::nwords(len);
      unsigned long long* dst = R.area[q] + (int64_t)me * cap;
      for (int64_t w0 = tid; w0 < nw; w0 += nthr * U) {
        uint32_t d[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t w = w0 + u * nthr;
          d[u] = w < nw ? F::load(R.buf, o, len, w) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t w = w0 + u * nthr;
          if (w < nw) st_ll(dst + w, d[u], e);
        }
      }
    }
    if (tr) tr[3] = global_ns();
    if (a.fault > 0) return;  // injected crash: my inputs are in the owners' slots, nothing else happens
    // 2. fold my region in the reference order; result -> my buffer + every peer's gather slot [me]
    {
      const int64_t o = R.off[me], len = R.len[me], nu = F::nunits(len);
      auto slot = [&](int p) { return (const unsigned long long*)(own + (int64_t)p * cap); };
      for (int64_t u = tid; u < nu; u += nthr) {
        uint32_t res[WPU];
        ll_fold_unit<T>(R, R.order, N, a.nlev, o, len, u, slot, wt, res);
#pragma unroll
        for (int j = 0; j < WPU; ++j) F::store(R.buf, o, len, u * WPU + j, res[j]);
        for (int k = 1; k < N; ++k) {
          unsigned long long* dst = R.area[(me + k) % N] + (int64_t)(N + me) * cap + u * WPU;
#pragma unroll
          for (int j = 0; j < WPU; ++j) st_ll(dst + j, res[j], e);
        }
      }
    }
    if (tr) tr[4] = global_ns();
    // 3. gather every peer's result from my gather slots
    for (int k = 1; k < N; ++k) {
      const int q = (me + k) % N;
      const int64_t o = R.off[q], len = R.len[q], nw = F::nwords(len);
      const unsigned long long* src = own + (int64_t)(N + q) * cap;
      for (int64_t w0 = tid; w0 < nw; w0 += nthr * U) {
        unsigned long long raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t w = w0 + u * nthr;
          raw[u] = w < nw ? ld_ll(src + w) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t w = w0 + u * nthr;
          if (w < nw) {
            const uint32_t d = (uint32_t)(raw[u] >> 32) == e ? (uint32_t)raw[u] : wt.get(src + w, q);
            if (!wt.failed) F::store(R.buf, o, len, w, d);
          }
        }
      }
    }
    if (tr) tr[5] = global_ns();
  }

  if (tr) tr[30] = global_ns();
  if (wt.failed) {
    s_fail = 1;
    if (wt.peer >= 0) s_peer = wt.peer;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (s_fail) {
    if (atomicCAS(&a.err->code, 0, 3) == 0) {
      a.err->rank = me;
      a.err->step = 0;
      a.err->peer = s_peer;
    }
    *wt.abort_word = 1u;
    return;  // the epoch is not advanced: the communicator is in an error state
  }
  // the last CTA of this rank publishes the epoch (same protocol as rbx_step_kernel)
  unsigned int* done = reinterpret_cast<unsigned int*>(R.my_sig + SigLayout::epoch_off + 1);
  if (atomicAdd(done, 1u) == (unsigned)a.nb - 1u) {
    *done = 0u;
    *(volatile uint32_t*)(R.my_sig + SigLayout::epoch_off) = e;
  }
  if (tr) tr[31] = global_ns();
}

}  // namespace rbx
