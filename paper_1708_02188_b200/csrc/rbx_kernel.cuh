// sm_100a persistent step-interpreter kernel for the multi-ring allreduce.
//
// One CTA-group of `nblocks` CTAs per rank executes the rank's Plan
// (rbx_plan.h).  Every step: (1) wait for the peers' epoch-tagged flags
// (ld.acquire.sys on the rank's own signal area, written remotely over
// NVLink), (2) fold the step's segments: 16-byte coalesced loads from the
// local buffer and from NVLink-mapped peer buffers, reduced in registers in
// exactly the reference's order, then 16-byte stores into the local buffer
// and/or straight into peer buffers (push), (3) publish completion with a
// st.release.sys into each consumer's signal area.
//
// Reference mapping: a ring phase ADD (`view += payload`,
// pkg/src/ringbox/runtime.py:248-249) is one position of the fold; REPLACE
// (`view[:] = payload`, runtime.py:250-251) is a push/pull copy.  The frame
// header checks (runtime.py:229-245) become epoch-tagged flags and a
// watchdog that reports the peer and step on timeout (CollectiveError).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <type_traits>

#include "rbx_plan.h"

namespace rbx {

// ------------------------------------------------------------------ dtypes --
// Each dtype defines how a 16-byte vector (int4) splits into VEC lanes, how a
// lane widens to the accumulator type and how the result narrows back.  All
// conversions are bit manipulations on registers (no address-taken arrays).
__device__ __forceinline__ uint32_t word(const int4& r, int i) {
  return (uint32_t)(i == 0 ? r.x : i == 1 ? r.y : i == 2 ? r.z : r.w);
}
__device__ __forceinline__ void set_word(int4& r, int i, uint32_t v) {
  if (i == 0)
    r.x = (int)v;
  else if (i == 1)
    r.y = (int)v;
  else if (i == 2)
    r.z = (int)v;
  else
    r.w = (int)v;
}

template <typename T>
struct Traits;
template <>
struct Traits<float> {
  using Acc = float;
  using Bits = uint32_t;
  static constexpr int VEC = 4;
  __device__ static Acc lane(const int4& r, int l) { return __uint_as_float(word(r, l)); }
  __device__ static void put(int4& r, int l, Acc x) { set_word(r, l, __float_as_uint(x)); }
  __device__ static Acc from_bits(Bits b) { return __uint_as_float(b); }
  __device__ static Bits to_bits(Acc x) { return __float_as_uint(x); }
  __device__ static Acc add(Acc a, Acc b) { return __fadd_rn(a, b); }
};
template <>
struct Traits<double> {
  using Acc = double;
  using Bits = unsigned long long;
  static constexpr int VEC = 2;
  __device__ static Acc lane(const int4& r, int l) {
    return __hiloint2double((int)word(r, 2 * l + 1), (int)word(r, 2 * l));
  }
  __device__ static void put(int4& r, int l, Acc x) {
    set_word(r, 2 * l, (uint32_t)__double2loint(x));
    set_word(r, 2 * l + 1, (uint32_t)__double2hiint(x));
  }
  __device__ static Acc from_bits(Bits b) { return __longlong_as_double((long long)b); }
  __device__ static Bits to_bits(Acc x) { return (Bits)__double_as_longlong(x); }
  __device__ static Acc add(Acc a, Acc b) { return __dadd_rn(a, b); }
};
template <>
struct Traits<unsigned long long> {  // int64: wrapping add (numpy semantics)
  using Acc = unsigned long long;
  using Bits = unsigned long long;
  static constexpr int VEC = 2;
  __device__ static Acc lane(const int4& r, int l) { return ((Acc)word(r, 2 * l + 1) << 32) | (Acc)word(r, 2 * l); }
  __device__ static void put(int4& r, int l, Acc x) {
    set_word(r, 2 * l, (uint32_t)x);
    set_word(r, 2 * l + 1, (uint32_t)(x >> 32));
  }
  __device__ static Acc from_bits(Bits b) { return b; }
  __device__ static Bits to_bits(Acc x) { return x; }
  __device__ static Acc add(Acc a, Acc b) { return a + b; }
};
template <>
struct Traits<unsigned int> {  // int32: wrapping add
  using Acc = unsigned int;
  using Bits = uint32_t;
  static constexpr int VEC = 4;
  __device__ static Acc lane(const int4& r, int l) { return word(r, l); }
  __device__ static void put(int4& r, int l, Acc x) { set_word(r, l, x); }
  __device__ static Acc from_bits(Bits b) { return b; }
  __device__ static Bits to_bits(Acc x) { return x; }
  __device__ static Acc add(Acc a, Acc b) { return a + b; }
};
template <>
struct Traits<__nv_bfloat16> {  // bf16 storage, fp32 accumulation, one RNE at the end
  using Acc = float;
  using Bits = unsigned short;
  static constexpr int VEC = 8;
  __device__ static Acc lane(const int4& r, int l) {
    const uint32_t w = word(r, l >> 1);
    return __uint_as_float((l & 1) ? (w & 0xffff0000u) : (w << 16));
  }
  __device__ static uint32_t narrow(Acc x) { return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(x)); }
  __device__ static void put(int4& r, int l, Acc x) {
    const uint32_t h = narrow(x);
    const uint32_t w = word(r, l >> 1);
    set_word(r, l >> 1, (l & 1) ? ((w & 0xffffu) | (h << 16)) : ((w & 0xffff0000u) | h));
  }
  __device__ static Acc from_bits(Bits b) { return __uint_as_float((uint32_t)b << 16); }
  __device__ static Bits to_bits(Acc x) { return (Bits)narrow(x); }
  __device__ static Acc add(Acc a, Acc b) { return __fadd_rn(a, b); }
};
template <>
struct Traits<__half> {  // f16 storage, fp32 accumulation
  using Acc = float;
  using Bits = unsigned short;
  static constexpr int VEC = 8;
  __device__ static Acc lane(const int4& r, int l) {
    const uint32_t w = word(r, l >> 1);
    return __half2float(__ushort_as_half((unsigned short)((l & 1) ? (w >> 16) : (w & 0xffffu))));
  }
  __device__ static uint32_t narrow(Acc x) { return (uint32_t)__half_as_ushort(__float2half_rn(x)); }
  __device__ static void put(int4& r, int l, Acc x) {
    const uint32_t h = narrow(x);
    const uint32_t w = word(r, l >> 1);
    set_word(r, l >> 1, (l & 1) ? ((w & 0xffffu) | (h << 16)) : ((w & 0xffff0000u) | h));
  }
  __device__ static Acc from_bits(Bits b) { return __half2float(__ushort_as_half(b)); }
  __device__ static Bits to_bits(Acc x) { return (Bits)narrow(x); }
  __device__ static Acc add(Acc a, Acc b) { return __fadd_rn(a, b); }
};

// ------------------------------------------------------------ primitives --
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// 16-byte streaming load that bypasses L1 (peer data may change between
// steps).  `volatile` keeps every load of a batch ahead of the arithmetic that
// consumes it: ptxas otherwise interleaves them in pairs to save registers,
// halving the bytes in flight (Little's law on HBM/NVLink latency).
__device__ __forceinline__ int4 ld_stream(const char* p) {
  int4 v;
  asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while the previous
// kernel on the stream drains; griddepcontrol.wait blocks until that kernel has
// completed and its memory is visible (a no-op for a normally launched kernel).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Nested left fold (dim 0 innermost), fed one operand at a time.  ctrl[j]:
// bit L set -> level L starts a new group at position j; bits 4-5 = number of
// levels whose group closes at j (capped at nlev-1), so the closed value is
// handed one level up.  Level nlev-1 holds the result after the last operand.
template <typename T, int LANES, int NLEV>
struct FoldState {
  using Acc = typename Traits<T>::Acc;
  Acc a[NLEV][LANES];
  __device__ __forceinline__ FoldState() {
#pragma unroll
    for (int L = 0; L < NLEV; ++L)
#pragma unroll
      for (int l = 0; l < LANES; ++l) a[L][l] = Acc(0);
  }
  __device__ __forceinline__ void feed(uint32_t c, const Acc (&x)[LANES]) {
    const uint32_t up = c >> 4;
#pragma unroll
    for (int l = 0; l < LANES; ++l) a[0][l] = (c & 1u) ? x[l] : Traits<T>::add(a[0][l], x[l]);
#pragma unroll
    for (int L = 1; L < NLEV; ++L) {
      if (up >= (uint32_t)L) {
#pragma unroll
        for (int l = 0; l < LANES; ++l) a[L][l] = (c & (1u << L)) ? a[L - 1][l] : Traits<T>::add(a[L][l], a[L - 1][l]);
      }
    }
  }
  __device__ __forceinline__ Acc result(int l) const { return a[NLEV - 1][l]; }
};

// 16 bytes of results from the accumulators of one vector.  16-bit types
// narrow lane pairs with one cvt.rn.{bf16x2,f16x2}.f32 each: the same RNE as
// the per-lane narrow, with half the conversions and no bit inserts.
template <typename T, int LANES, int NLEV>
__device__ __forceinline__ int4 pack_result(const FoldState<T, LANES, NLEV>& st) {
  int4 packed = make_int4(0, 0, 0, 0);
  if constexpr (sizeof(T) == 2 && LANES % 2 == 0) {
#pragma unroll
    for (int i = 0; i < LANES / 2; ++i) {
      uint32_t w;
      if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(st.result(2 * i), st.result(2 * i + 1));
        w = *reinterpret_cast<const uint32_t*>(&h);
      } else {
        const __half2 h = __floats2half2_rn(st.result(2 * i), st.result(2 * i + 1));
        w = *reinterpret_cast<const uint32_t*>(&h);
      }
      set_word(packed, i, w);
    }
  } else {
#pragma unroll
    for (int l = 0; l < LANES; ++l) Traits<T>::put(packed, l, st.result(l));
  }
  return packed;
}

struct SegCtx {
  const char* src[RBX_MAX_RANKS];
  char* dst[RBX_MAX_RANKS];
  uint8_t ctrl[RBX_MAX_RANKS];
  int ndst, nlev;
};

// Body of one segment, vectors [v0, v1) (relative to seg.body_off).  The
// 16-byte loads of a batch of up to 8 operands (x U independent vectors) are
// all issued before any arithmetic, so every thread keeps ~8 NVLink/HBM
// requests in flight; operands stay raw (int4) until folded.
template <typename T, int NSRC, int NLEV>
__device__ __noinline__ void fold_body(const SegCtx& sc, int64_t body_off, int64_t v0, int64_t v1) {
  constexpr int VEC = Traits<T>::VEC;
  constexpr int B = NSRC < 8 ? NSRC : 8;  // operands per load batch
#ifndef RBX_LD_DEPTH
#define RBX_LD_DEPTH 8  // 16-byte loads in flight per thread per batch (16: callee-saved spills, -30%)
#endif
  constexpr int U_LD = RBX_LD_DEPTH / B > 0 ? RBX_LD_DEPTH / B : 1;
  constexpr int U_ACC = 32 / (NLEV * VEC) > 0 ? 32 / (NLEV * VEC) : 1;
  constexpr int U = NSRC == 1 ? 8 : (U_LD < U_ACC ? U_LD : U_ACC);
  const int64_t base = body_off * (int64_t)sizeof(T);
  const int64_t stride = (int64_t)blockDim.x * U;
  if (NSRC == 1) {  // REPLACE: bitwise copy (runtime.py:250-251)
    const char* p = sc.src[0] + base;
    for (int64_t v = v0 + threadIdx.x; v < v1; v += stride) {
      int4 raw[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t idx = v + (int64_t)u * blockDim.x;
        if (idx < v1) raw[u] = ld_stream(p + idx * 16);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t idx = v + (int64_t)u * blockDim.x;
        if (idx < v1)
          for (int d = 0; d < sc.ndst; ++d) __stcg(reinterpret_cast<int4*>(sc.dst[d] + base + idx * 16), raw[u]);
      }
    }
    return;
  }
  for (int64_t v = v0 + threadIdx.x; v < v1; v += stride) {
    FoldState<T, VEC, NLEV> st[U];
    // every operand is defined on every path (zero for vectors past the end): an
    // operand array that is only conditionally written is what made ptxas spill it
    const bool full = v + (int64_t)(U - 1) * blockDim.x < v1;
#pragma unroll
    for (int j0 = 0; j0 < NSRC; j0 += B) {
      int4 raw[U][B];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t idx = v + (int64_t)u * blockDim.x;
#pragma unroll
        for (int k = 0; k < B; ++k)
          if (j0 + k < NSRC) {
            const char* p = NSRC > 8 ? ((const char* volatile*)sc.src)[j0 + k] : sc.src[j0 + k];
            raw[u][k] = (full || idx < v1) ? ld_stream(p + base + idx * 16) : make_int4(0, 0, 0, 0);
          } else {
            raw[u][k] = make_int4(0, 0, 0, 0);
          }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int k = 0; k < B; ++k)
          if (j0 + k < NSRC) {
            typename Traits<T>::Acc x[VEC];
#pragma unroll
            for (int l = 0; l < VEC; ++l) x[l] = Traits<T>::lane(raw[u][k], l);
            st[u].feed(sc.ctrl[j0 + k], x);
          }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t idx = v + (int64_t)u * blockDim.x;
      if (idx < v1) {
        const int4 packed = pack_result(st[u]);
        for (int d = 0; d < sc.ndst; ++d) __stcg(reinterpret_cast<int4*>(sc.dst[d] + base + idx * 16), packed);
      }
    }
  }
}

template <typename T, int NSRC, int NLEV>
__device__ __forceinline__ void fold_scalar(const SegCtx& sc, int64_t elem) {
  using Tr = Traits<T>;
  using B = typename Tr::Bits;
  const int64_t byte = elem * (int64_t)sizeof(T);
  if (NSRC == 1) {  // REPLACE: bitwise copy
    const B v = __ldcg(reinterpret_cast<const B*>(sc.src[0] + byte));
    for (int d = 0; d < sc.ndst; ++d) __stcg(reinterpret_cast<B*>(sc.dst[d] + byte), v);
    return;
  }
  FoldState<T, 1, NLEV> st;
#pragma unroll
  for (int j = 0; j < NSRC; ++j) {
    typename Tr::Acc x[1] = {Tr::from_bits(__ldcg(reinterpret_cast<const B*>(sc.src[j] + byte)))};
    st.feed(sc.ctrl[j], x);
  }
  const B out = Tr::to_bits(st.result(0));
  for (int d = 0; d < sc.ndst; ++d) __stcg(reinterpret_cast<B*>(sc.dst[d] + byte), out);
}

// ---- RING_DIMS with bf16/f16: stage partials kept in fp32 workspaces --------
// One ring fold (single level) where the sources (ACC bit0) and/or the
// destinations (ACC bit1) are fp32 partial arrays instead of T buffers: a
// vector unit is VEC elements (16 bytes of T, 32 bytes of fp32).  Rounding to
// T happens once, in the last dimension's fold (parity policy: fold the
// fp32-upcast inputs in the reference order, one RNE at the end).
template <typename T, int NSRC, int ACC>
__device__ __noinline__ void fold_body_acc(const SegCtx& sc, int64_t body_off, int64_t v0, int64_t v1) {
  using Acc = typename Traits<T>::Acc;
  constexpr int VEC = Traits<T>::VEC;
  if constexpr (sizeof(Acc) == 4 && VEC == 8) {
    for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
      const int64_t e = body_off + v * VEC;  // first element of this vector
      constexpr int B = NSRC < 4 ? NSRC : 4;  // operands per load batch (8 x 16-byte loads in flight)
      FoldState<T, VEC, 1> st;
#pragma unroll
      for (int j0 = 0; j0 < NSRC; j0 += B) {
        int4 raw[B][2];
#pragma unroll
        for (int k = 0; k < B; ++k) {
          if (j0 + k < NSRC) {
            if (ACC & 1) {
              raw[k][0] = ld_stream(sc.src[j0 + k] + e * 4);
              raw[k][1] = ld_stream(sc.src[j0 + k] + e * 4 + 16);
            } else {
              raw[k][0] = ld_stream(sc.src[j0 + k] + e * (int64_t)sizeof(T));
            }
          }
        }
#pragma unroll
        for (int k = 0; k < B; ++k) {
          if (j0 + k < NSRC) {
            Acc x[VEC];
#pragma unroll
            for (int l = 0; l < VEC; ++l)
              x[l] = (ACC & 1) ? __uint_as_float(word(raw[k][l >> 2], l & 3)) : Traits<T>::lane(raw[k][0], l);
            st.feed(sc.ctrl[j0 + k], x);
          }
        }
      }
      if (ACC & 2) {
        int4 lo, hi;
        lo = make_int4(__float_as_int(st.result(0)), __float_as_int(st.result(1)), __float_as_int(st.result(2)),
                       __float_as_int(st.result(3)));
        hi = make_int4(__float_as_int(st.result(4)), __float_as_int(st.result(5)), __float_as_int(st.result(6)),
                       __float_as_int(st.result(7)));
        for (int d = 0; d < sc.ndst; ++d) {
          __stcg(reinterpret_cast<int4*>(sc.dst[d] + e * 4), lo);
          __stcg(reinterpret_cast<int4*>(sc.dst[d] + e * 4 + 16), hi);
        }
      } else {
        const int4 packed = pack_result(st);
        for (int d = 0; d < sc.ndst; ++d)
          __stcg(reinterpret_cast<int4*>(sc.dst[d] + e * (int64_t)sizeof(T)), packed);
      }
    }
  }
}

template <typename T, int NSRC, int ACC>
__device__ __forceinline__ void fold_scalar_acc(const SegCtx& sc, int64_t elem) {
  using Tr = Traits<T>;
  using Acc = typename Tr::Acc;
  if constexpr (sizeof(Acc) == 4 && Tr::VEC == 8) {
    FoldState<T, 1, 1> st;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      Acc x[1];
      if (ACC & 1)
        x[0] = __ldcg(reinterpret_cast<const float*>(sc.src[j] + elem * 4));
      else
        x[0] = Tr::from_bits(__ldcg(reinterpret_cast<const typename Tr::Bits*>(sc.src[j] + elem * (int64_t)sizeof(T))));
      st.feed(sc.ctrl[j], x);
    }
    for (int d = 0; d < sc.ndst; ++d) {
      if (ACC & 2)
        __stcg(reinterpret_cast<float*>(sc.dst[d] + elem * 4), st.result(0));
      else
        __stcg(reinterpret_cast<typename Tr::Bits*>(sc.dst[d] + elem * (int64_t)sizeof(T)), Tr::to_bits(st.result(0)));
    }
  }
}

#define RBX_ACC_SHAPES(X)                                                                                  \
  X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

template <typename T>
__device__ __forceinline__ void dispatch_body_acc(int nsrc, int acc, const SegCtx& sc, int64_t body_off, int64_t v0,
                                                  int64_t v1) {
  if constexpr (sizeof(typename Traits<T>::Acc) == 4 && Traits<T>::VEC == 8) {
    switch (nsrc * 4 + acc) {
#define RBX_ACC_CASE(N)                                            \
  case N * 4 + 1: fold_body_acc<T, N, 1>(sc, body_off, v0, v1); break; \
  case N * 4 + 2: fold_body_acc<T, N, 2>(sc, body_off, v0, v1); break; \
  case N * 4 + 3: fold_body_acc<T, N, 3>(sc, body_off, v0, v1); break;
      RBX_ACC_SHAPES(RBX_ACC_CASE)
#undef RBX_ACC_CASE
      default: break;
    }
  }
}

template <typename T>
__device__ __forceinline__ void dispatch_scalar_acc(int nsrc, int acc, const SegCtx& sc, int64_t elem) {
  if constexpr (sizeof(typename Traits<T>::Acc) == 4 && Traits<T>::VEC == 8) {
    switch (nsrc * 4 + acc) {
#define RBX_ACC_CASE(N)                                 \
  case N * 4 + 1: fold_scalar_acc<T, N, 1>(sc, elem); break; \
  case N * 4 + 2: fold_scalar_acc<T, N, 2>(sc, elem); break; \
  case N * 4 + 3: fold_scalar_acc<T, N, 3>(sc, elem); break;
      RBX_ACC_SHAPES(RBX_ACC_CASE)
#undef RBX_ACC_CASE
      default: break;
    }
  }
}

// (operand count, nesting depth) pairs that grid factorizations of <= 16 ranks produce.
#ifndef RBX_FOLD_SHAPES
#define RBX_FOLD_SHAPES(X)                                                                              \
  X(1, 1) X(2, 1) X(3, 1) X(4, 1) X(5, 1) X(6, 1) X(7, 1) X(8, 1) X(9, 1) X(10, 1) X(11, 1) X(12, 1)     \
  X(13, 1) X(14, 1) X(15, 1) X(16, 1) X(4, 2) X(6, 2) X(8, 2) X(9, 2) X(10, 2) X(12, 2) X(14, 2)         \
  X(15, 2) X(16, 2) X(8, 3) X(12, 3) X(16, 3) X(16, 4)
#endif

template <typename T>
__device__ __forceinline__ void dispatch_body(int nsrc, int nlev, const SegCtx& sc, int64_t body_off, int64_t v0,
                                              int64_t v1) {
  switch (nsrc * 8 + nlev) {
#define RBX_CASE(N, L) \
  case N * 8 + L:      \
    fold_body<T, N, L>(sc, body_off, v0, v1); break;
    RBX_FOLD_SHAPES(RBX_CASE)
#undef RBX_CASE
    default: break;
  }
}

template <typename T>
__device__ __forceinline__ void dispatch_scalar(int nsrc, int nlev, const SegCtx& sc, int64_t elem) {
  switch (nsrc * 8 + nlev) {
#define RBX_CASE(N, L) \
  case N * 8 + L:      \
    fold_scalar<T, N, L>(sc, elem); break;
    RBX_FOLD_SHAPES(RBX_CASE)
#undef RBX_CASE
    default: break;
  }
}

struct ErrRecord {  // host-mapped; first failure wins
  int code, rank, step, peer;
};

struct KernelArgs {
  const Plan* plans;     // one per rank hosted by this launch
  int nblocks;           // CTAs per rank
  int plan_bytes;        // bytes of each Plan staged in shared memory
  uint64_t timeout_ns;
  ErrRecord* err;
  unsigned long long* trace;  // optional 64-word timeline (first/last CTA), or null
  // fault injection (Workload.crash_phase, runtime.py:393-394, 429-432): -1 off; else the rank
  // processes only the first fault_milli/1000 of its first data step's work tiles and its CTAs
  // return without signalling -- a rank that dies with part of its data pushed
  int fault_milli;
};

__device__ __forceinline__ bool flag_reached(uint32_t v, uint32_t e) { return (int32_t)(v - e) >= 0; }

// Spin until flags[slot][peer][blk] >= e.  Returns false on timeout/abort.
__device__ __forceinline__ bool spin_flag(const uint32_t* f, uint32_t e, volatile uint32_t* abort_word,
                                          uint64_t t0, uint64_t timeout_ns) {
  // poll with relaxed loads (cheap), then one acquire to order the data reads
  uint32_t it = 0;
  while (!flag_reached(ld_relaxed_sys(f), e)) {
    if ((++it & 255u) == 0) {
      if (*abort_word) return false;
      if (global_ns() - t0 > timeout_ns) return false;
      __nanosleep(64);
    }
  }
  (void)ld_acquire_sys(f);
  return true;
}

// Bytes of a Plan that a launch needs in shared memory: everything up to the
// segment array plus the segments actually used.
__host__ __device__ constexpr size_t plan_smem_bytes(int nsegs) {
  return offsetof(Plan, segs) + (size_t)nsegs * sizeof(Seg);
}

// Work of one step for CTA b: the step's body vectors (all segments
// concatenated) are cut into tiles of `tile` vectors dealt round-robin to the
// CTAs (tile == 0: one contiguous range per CTA).
template <typename T>
__device__ __forceinline__ void run_step_work(const Plan& P, const Step& st, int b, int nb, SegCtx& s_seg,
                                              int& s_cur /* thread-local: same value in every thread */,
                                              unsigned int* tile_ctr, int* s_next, int fault_milli = -1) {
  const int64_t T_vec = st.total_vec;
  auto setup = [&](int k) {
    const Seg& sg = P.segs[st.seg0 + k];
    __syncthreads();  // s_seg reuse
    if (threadIdx.x < sg.nsrc) {
      s_seg.src[threadIdx.x] = (const char*)P.ptrs[sg.tbl + sg.src[threadIdx.x]];
      s_seg.ctrl[threadIdx.x] = sg.ctrl[threadIdx.x];
    }
    if (threadIdx.x < sg.ndst) s_seg.dst[threadIdx.x] = (char*)P.ptrs[sg.tbl + sg.dst[threadIdx.x]];
    if (threadIdx.x == 0) {
      s_seg.ndst = sg.ndst;
      s_seg.nlev = sg.nlev;
    }
    __syncthreads();
  };
  auto body = [&](int64_t lo, int64_t hi) {  // [lo, hi) in step vector space
    int k = 0;
    while (k < st.nseg) {
      const Seg& sg = P.segs[st.seg0 + k];
      const int64_t a = lo > sg.vec_begin ? lo : sg.vec_begin;
      const int64_t z = hi < sg.vec_begin + sg.nvec ? hi : sg.vec_begin + sg.nvec;
      if (sg.vec_begin >= hi) break;
      if (a < z) {
        if (s_cur != k) {
          setup(k);
          s_cur = k;
        }
        if (sg.acc)
          dispatch_body_acc<T>(sg.nsrc, sg.acc, s_seg, sg.body_off, a - sg.vec_begin, z - sg.vec_begin);
        else
          dispatch_body<T>(sg.nsrc, sg.nlev, s_seg, sg.body_off, a - sg.vec_begin, z - sg.vec_begin);
      }
      ++k;
    }
  };
  const int64_t step_tile = st.tile > 0 ? st.tile : P.tile;
  // injected fault: only the first fault_milli/1000 of the step's work units are processed
  auto cut = [&](int64_t units) -> int64_t { return fault_milli < 0 ? units : units * fault_milli / 1000; };
  if (step_tile <= 0) {
    const int64_t my0 = T_vec * b / nb, my1 = T_vec * (b + 1) / nb;
    if (my0 < my1 && b < cut(nb)) body(my0, my1);
  } else if (tile_ctr && (T_vec + step_tile - 1) / step_tile > nb) {
    // Dynamic tiles: CTA b starts with tile b, then claims tiles nb, nb+1, ...
    // from this step's counter.  The claim for the next tile is issued before
    // the current tile's loads, so its latency hides under them; CTAs that
    // get more NVLink bandwidth simply take more tiles (no fixed tail).
    // With tail_split > 1 the last nb tiles' worth of vectors is cut into smaller
    // tiles, so the CTAs finish the step within a small tile of each other.
    const int64_t tile = step_tile;
    const int64_t split = P.tail_split > 1 ? P.tail_split : 1;
    const int64_t small = tile / split > 0 ? tile / split : 1;
    const int64_t nbig = split > 1 ? (T_vec > (int64_t)nb * tile ? (T_vec - (int64_t)nb * tile) / tile : 0)
                                   : (T_vec + tile - 1) / tile;
    const int64_t big_end = nbig * tile;
    const int64_t ntiles = nbig + (split > 1 ? (T_vec - big_end + small - 1) / small : 0);
    const int64_t tlimit = cut(ntiles);
    int64_t t = b;
    int done_tiles = 0;
    while (t < tlimit) {
      unsigned int nxt = 0;
      if (threadIdx.x == 0) nxt = (unsigned)nb + atomicAdd(tile_ctr, 1u);
      const int64_t lo = t < nbig ? t * tile : big_end + (t - nbig) * small;
      const int64_t len = t < nbig ? tile : small;
      body(lo, lo + len < T_vec ? lo + len : T_vec);
      if (P.fence_every > 0 && ++done_tiles % P.fence_every == 0) __threadfence_system();
      __syncthreads();  // every thread has read *s_next for this tile
      if (threadIdx.x == 0) *s_next = (int)nxt;
      __syncthreads();
      t = *s_next;
    }
  } else {
    const int64_t tile = step_tile;
    const int64_t tlimit = cut((T_vec + tile - 1) / tile);
    for (int64_t t = b; t * tile < T_vec && t < tlimit; t += nb) {
      const int64_t lo = t * tile;
      body(lo, lo + tile < T_vec ? lo + tile : T_vec);
    }
  }
  if (fault_milli >= 0) return;  // a dying rank leaves its scalar edges undone
  for (int k = b % nb; k < st.nseg; k += nb) {  // scalar head/tail of segment k: CTA k mod nb
    const Seg& sg = P.segs[st.seg0 + k];
    if (sg.head + sg.tail == 0) continue;
    if (s_cur != k) {
      setup(k);
      s_cur = k;
    }
    for (int i = threadIdx.x; i < sg.head + sg.tail; i += blockDim.x) {
      const int64_t elem = i < sg.head ? sg.off + i : sg.body_off + sg.nvec * P.vec + (i - sg.head);
      if (sg.acc)
        dispatch_scalar_acc<T>(sg.nsrc, sg.acc, s_seg, elem);
      else
        dispatch_scalar<T>(sg.nsrc, sg.nlev, s_seg, elem);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(512, 1) rbx_step_kernel(KernelArgs args) {
  extern __shared__ __align__(16) unsigned char s_plan_raw[];
  const int vrank = blockIdx.x / args.nblocks;
  const int b = blockIdx.x % args.nblocks;
  const int nb = args.nblocks;
  __shared__ uint32_t s_epoch;
  __shared__ int s_fail;
  __shared__ SegCtx s_seg;
  __shared__ int s_next;
  // optional timeline (RBX_TRACE): first and last CTA of the first rank
  unsigned long long* tr = nullptr;
  if (args.trace && threadIdx.x == 0 && vrank == 0 && (b == 0 || b == nb - 1)) tr = args.trace + (b == 0 ? 0 : 32);
  if (tr) {
    tr[29] = tr[31];  // previous launch's exit on this comm: start - prev exit = launch gap
    tr[0] = global_ns();
  }
  {  // stage this rank's plan in shared memory (one coalesced copy instead of
     // chains of dependent global loads on the critical path of every step)
    const int4* src = reinterpret_cast<const int4*>(args.plans + vrank);
    int4* dst = reinterpret_cast<int4*>(s_plan_raw);
    const int words = (int)((args.plan_bytes + 15) / 16);
    for (int i = threadIdx.x; i < words; i += blockDim.x) dst[i] = __ldg(src + i);
    if (tr) tr[20] = global_ns();  // slots 20-24: prologue detail (plans of <= 5 steps)
  }
  const Plan& P = *reinterpret_cast<const Plan*>(s_plan_raw);
  __syncthreads();
  if (tr) tr[21] = global_ns();
  uint32_t* my_sig = P.my_sig;
  volatile uint32_t* abort_word = my_sig ? (volatile uint32_t*)(my_sig + SigLayout::abort_off) : nullptr;
  const uint64_t t0 = P.nosync ? 0 : global_ns();

  if (threadIdx.x == 0) {
    s_fail = 0;
    // one epoch per rank (all CTAs of a launch agree; launches on a stream are
    // ordered, so the previous launch's final increment is visible here)
    s_epoch = P.nosync ? 0u : *(volatile uint32_t*)(my_sig + SigLayout::epoch_off) + 1u;
    if (tr) tr[22] = global_ns();
  }
  __syncthreads();
  const uint32_t e = s_epoch;
  if (tr) tr[1] = global_ns();

  if (!P.nosync && threadIdx.x < P.nentry) {  // ENTRY: "my stream reached the collective"
    // No release needed: this launch has written nothing yet, and everything
    // earlier on the stream (the caller's inputs) is complete in L2, which is
    // where peer reads are served.  A relaxed store saves ~2 us per launch.
    const int q = P.entry_peers[threadIdx.x];
    st_relaxed_sys(P.sig[q] + flag_index(0, P.me, b), e);
  }
  if (tr) tr[2] = global_ns();
  if (tr) tr[23] = global_ns();

  for (int s = 0; s < P.nsteps; ++s) {
    const Step& st = P.steps[s];
    // ---- wait ----
    if (!P.nosync && st.nwait) {
      bool ok = true;
      for (int w = 0; w < st.nwait && ok; ++w) {
        const Wait wt = P.waits[st.wait0 + w];
        const uint32_t* base = my_sig + flag_index(wt.slot, wt.peer, 0);
        if (wt.all) {
          for (int k = threadIdx.x; k < nb && ok; k += blockDim.x) ok = spin_flag(base + k, e, abort_word, t0, args.timeout_ns);
        } else if ((int)threadIdx.x == (w % blockDim.x)) {
          ok = spin_flag(base + b, e, abort_word, t0, args.timeout_ns);
        }
        if (!ok) {
          s_fail = 1;
          if (atomicCAS(&args.err->code, 0, 3) == 0) {
            args.err->rank = P.me;
            args.err->step = s;
            args.err->peer = wt.peer;
          }
          *abort_word = 1u;
        }
      }
      __syncthreads();
      if (s_fail) return;
    }
    if (tr && s < 9) tr[3 + 3 * s] = global_ns();
    // ---- work ----
    if (st.nseg) {
      int cur = -1;  // segment whose pointers are in s_seg (thread-local, uniform)
      unsigned int* ctr = (P.dyn && !P.nosync && P.tile > 0)
                              ? reinterpret_cast<unsigned int*>(my_sig + SigLayout::tiles_off + s) : nullptr;
      run_step_work<T>(P, st, b, nb, s_seg, cur, ctr, &s_next, args.fault_milli);
      if (args.fault_milli >= 0) return;  // injected crash: no signals, the epoch is not advanced
    }
    if (tr && s < 9) tr[4 + 3 * s] = global_ns();
    // ---- signal ----
    if (!P.nosync && st.nsig) {
      __syncthreads();
      if ((int)threadIdx.x < st.nsig) {
        // st.release.sys is cumulative over the CTA's writes ordered before it by
        // bar.sync, so peers that acquire the flag see our pushed data.
        const int q = P.sigs[st.sig0 + threadIdx.x];
        st_release_sys(P.sig[q] + flag_index(s + 1, P.me, b), e);
      }
    }
    if (tr && s < 9) tr[5 + 3 * s] = global_ns();
  }
  if (tr) tr[30] = global_ns();
  if (!P.nosync) {  // the last CTA of this rank to finish publishes the new epoch
    __syncthreads();
    if (threadIdx.x == 0) {
      // every CTA has read the epoch before it arrives here; the next launch on
      // the stream starts after this one completes, so no fence is needed
      unsigned int* done = reinterpret_cast<unsigned int*>(my_sig + SigLayout::epoch_off + 1);
      if (atomicAdd(done, 1u) == (unsigned)nb - 1u) {
        *done = 0u;
        if (P.dyn)  // every CTA has made its last claim: rewind the tile counters
          for (int s = 0; s < P.nsteps; ++s) my_sig[SigLayout::tiles_off + s] = 0u;
        *(volatile uint32_t*)(my_sig + SigLayout::epoch_off) = e;
      }
    }
  }
  if (tr) tr[31] = global_ns();
}

}  // namespace rbx
