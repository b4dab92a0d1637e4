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
  int64_t total_vec;
  char* dst[RBX_MAX_RANKS];  // every rank's buffer
  LocalSeg seg[RBX_LOCAL_MAX_SEGS];
  // scalar head/tail elements (misaligned region edges), done by CTA 0
  int nscalar;
  int64_t scalar_elem[2 * RBX_LOCAL_MAX_SEGS * 8];
  uint8_t scalar_seg[2 * RBX_LOCAL_MAX_SEGS * 8];
};

template <typename T, int V, int NLEV>
__global__ void __launch_bounds__(512) rbx_local_kernel(const __grid_constant__ LocalArgs a) {
  constexpr int VEC = Traits<T>::VEC;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int s = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < a.total_vec; v += stride) {
    while (v >= a.seg[s].vec_begin + a.seg[s].nvec) ++s;  // v only grows
    const LocalSeg& sg = a.seg[s];
    const int64_t byte = (sg.body_off + (v - sg.vec_begin) * VEC) * (int64_t)sizeof(T);
    int4 raw[V];
#pragma unroll
    for (int j = 0; j < V; ++j) raw[j] = ld_stream(sg.src[j] + byte);
    FoldState<T, VEC, NLEV> st;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      typename Traits<T>::Acc x[VEC];
#pragma unroll
      for (int l = 0; l < VEC; ++l) x[l] = Traits<T>::lane(raw[j], l);
      st.feed(sg.ctrl[j], x);
    }
    const int4 packed = pack_result(st);
#pragma unroll
    for (int d = 0; d < V; ++d) __stcg(reinterpret_cast<int4*>(a.dst[d] + byte), packed);
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
