// Specialised 1-GPU local-reduce kernel (MODE_LOCAL): every rank of a grid is
// a buffer in this GPU's HBM; each owned region is folded from all V buffers
// in the reference order (same FoldState as the step kernel) and written to all
// V buffers.  No flags, no step interpreter, no call boundary: one grid-stride
// loop over the concatenated body vectors of the V regions, so a warp streams
// 8 x 16-byte loads and 8 x 16-byte stores per vector with nothing else in the
// way.  HBM-bound: 2 x V x S bytes per launch.  Used for the shapes below; the
// generic step kernel serves every other (V, depth).
#pragma once
#include "rbx_kernel.cuh"

namespace rbx {

#define RBX_LOCAL_MAX_SEGS 16

struct LocalSeg {
  int64_t vec_begin, nvec, body_off;  // body vectors of the region, global vector space
  const char* src[RBX_MAX_RANKS];     // V buffers in fold order
  uint8_t ctrl[RBX_MAX_RANKS];
};

struct LocalArgs {
  int nseg;
  int hint;  // cache policy of the streaming loads/stores (env RBX_LOCAL_HINT): 0 .cg/.cg, 1 .cs/.cs,
             // 2 L2::evict_first policy on both, 3 .nc L1::no_allocate loads + .cs stores,
             // 4 as 3 with an L2 256-byte prefetch hint on the loads
  int64_t total_vec;
  char* dst[RBX_MAX_RANKS];  // every rank's buffer
  LocalSeg seg[RBX_LOCAL_MAX_SEGS];
  // scalar head/tail elements (misaligned region edges), done by CTA 0
  int nscalar;
  int64_t scalar_elem[2 * RBX_LOCAL_MAX_SEGS * 8];
  uint8_t scalar_seg[2 * RBX_LOCAL_MAX_SEGS * 8];
};

__device__ __forceinline__ int4 ld_hint(const char* p, int hint, uint64_t pol) {
  int4 v;
  if (hint == 1)
    asm volatile("ld.global.cs.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else if (hint == 2)
    asm volatile("ld.global.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
  else if (hint == 4)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
  return v;
}
__device__ __forceinline__ void st_hint(char* p, int4 v, int hint, uint64_t pol) {
  if (hint == 2)
    asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(pol)
                 : "memory");
  else
    asm volatile("st.global.cs.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <typename T, int V, int NLEV>
__global__ void __launch_bounds__(512) rbx_local_kernel(const __grid_constant__ LocalArgs a) {
  constexpr int VEC = Traits<T>::VEC;
  uint64_t pol = 0;
  if (a.hint == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int s = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.total_vec; v += stride) {
    while (v >= a.seg[s].vec_begin + a.seg[s].nvec) ++s;  // v only grows
    const LocalSeg& sg = a.seg[s];
    const int64_t byte = (sg.body_off + (v - sg.vec_begin) * VEC) * (int64_t)sizeof(T);
    int4 raw[V];
    if (a.hint == 0) {
#pragma unroll
      for (int j = 0; j < V; ++j) raw[j] = ld_stream(sg.src[j] + byte);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) raw[j] = ld_hint(sg.src[j] + byte, a.hint, pol);
    }
    FoldState<T, VEC, NLEV> st;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      typename Traits<T>::Acc x[VEC];
#pragma unroll
      for (int l = 0; l < VEC; ++l) x[l] = Traits<T>::lane(raw[j], l);
      st.feed(sg.ctrl[j], x);
    }
    const int4 packed = pack_result(st);
    if (a.hint == 0) {
#pragma unroll
      for (int d = 0; d < V; ++d) __stcg(reinterpret_cast<int4*>(a.dst[d] + byte), packed);
    } else {
#pragma unroll
      for (int d = 0; d < V; ++d) st_hint(a.dst[d] + byte, packed, a.hint, pol);
    }
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < a.nscalar; i += blockDim.x) {
      const LocalSeg& sg = a.seg[a.scalar_seg[i]];
      SegCtx sc;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        sc.src[j] = sg.src[j];
        sc.ctrl[j] = sg.ctrl[j];
      }
#pragma unroll
      for (int d = 0; d < V; ++d) sc.dst[d] = a.dst[d];
      sc.ndst = V;
      sc.nlev = NLEV;
      fold_scalar<T, V, NLEV>(sc, a.scalar_elem[i]);
    }
  }
}

// (V, depth) shapes with a specialised kernel: the B200 box's 8-GPU grids
// (2x2x2, 2x4 / 4x2, 8) and the 2/4-GPU ones.
#define RBX_LOCAL_SHAPES(X) X(8, 3) X(8, 2) X(8, 1) X(4, 2) X(4, 1) X(2, 1)

}  // namespace rbx
