// Instantiations for dtype i64 (one TU per dtype: parallel builds): the step
// kernel and the specialised local-reduce kernels.
#include "rbx_kernel.cuh"
#include "rbx_local.cuh"
#include "rbx_ll.cuh"

namespace rbx {
const void* step_kernel_i64() { return reinterpret_cast<const void*>(&rbx_step_kernel<unsigned long long>); }
const void* ll_kernel_i64(int maxv) {
  return maxv == 1 ? reinterpret_cast<const void*>(&rbx_ll_kernel<unsigned long long, 1>)
                   : reinterpret_cast<const void*>(&rbx_ll_kernel<unsigned long long, RBX_MAX_RANKS>);
}

const void* local_kernel_i64(int v, int nlev) {
#define RBX_LOCAL_CASE(V, L) \
  if (v == V && nlev == L) return reinterpret_cast<const void*>(&rbx_local_kernel<unsigned long long, V, L>);
  RBX_LOCAL_SHAPES(RBX_LOCAL_CASE)
#undef RBX_LOCAL_CASE
  return nullptr;
}
}  // namespace rbx
