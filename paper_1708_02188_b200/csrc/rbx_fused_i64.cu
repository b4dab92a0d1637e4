// Instantiations of the specialised FUSED kernel (rbx_fused.cuh) for dtype i64:
// one TU per dtype so the builds run in parallel.
#include "rbx_fused.cuh"

namespace rbx {
const void* fused_kernel_i64(int nsrc, int nlev, int maxseg) {
#define RBX_FUSED_CASE(N, L)                                                                          \
  if (nsrc == N && nlev == L)                                                                         \
    return maxseg == 1 ? reinterpret_cast<const void*>(&rbx_fused_kernel<unsigned long long, N, L, 1>)                \
                       : reinterpret_cast<const void*>(&rbx_fused_kernel<unsigned long long, N, L, RBX_FUSED_MAXSEG>);
  RBX_FUSED_SHAPES(RBX_FUSED_CASE)
#undef RBX_FUSED_CASE
  return nullptr;
}
}  // namespace rbx
