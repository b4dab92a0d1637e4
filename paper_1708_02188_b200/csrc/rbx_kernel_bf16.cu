// Instantiations for dtype bf16 (one TU per dtype: parallel builds): the step
// kernel and the specialised local-reduce kernels.
#include "rbx_kernel.cuh"
#include "rbx_local.cuh"
#include "rbx_ll.cuh"

namespace rbx {
const void* step_kernel_bf16() { return reinterpret_cast<const void*>(&rbx_step_kernel<__nv_bfloat16>); }
const void* ll_kernel_bf16(int maxv) {
  return maxv == 1 ? reinterpret_cast<const void*>(&rbx_ll_kernel<__nv_bfloat16, 1>)
                   : reinterpret_cast<const void*>(&rbx_ll_kernel<__nv_bfloat16, RBX_MAX_RANKS>);
}

const void* local_kernel_bf16(int v, int nlev) {
#define RBX_LOCAL_CASE(V, L) \
  if (v == V && nlev == L) return reinterpret_cast<const void*>(&rbx_local_kernel<__nv_bfloat16, V, L>);
  RBX_LOCAL_SHAPES(RBX_LOCAL_CASE)
#undef RBX_LOCAL_CASE
  return nullptr;
}
}  // namespace rbx
