// Instantiations of the specialised FUSED kernel (rbx_fused.cuh) for dtype i64:
// one TU per dtype so the builds run in parallel.  Also the RING_DIMS kernel (rbx_rings.cuh).
#include "rbx_fused.cuh"
#include "rbx_rings.cuh"

namespace rbx {
const void* fused_kernel_i64(int nsrc, int nlev, int ndst, int maxseg) {
#define RBX_FUSED_CASE(N, L, D)                                                                                        \
  if (nsrc == N && nlev == L && ndst == D)                                                                             \
    return maxseg == 1 ? reinterpret_cast<const void*>(&rbx_fused_kernel<unsigned long long, N, L, D, 1>)              \
                       : reinterpret_cast<const void*>(&rbx_fused_kernel<unsigned long long, N, L, D, RBX_FUSED_MAXSEG>);
  RBX_FUSED_SHAPES(RBX_FUSED_CASE)
#undef RBX_FUSED_CASE
  return nullptr;
}
const void* rings_kernel_i64() { return reinterpret_cast<const void*>(&rbx_rings_kernel<unsigned long long>); }
}  // namespace rbx
