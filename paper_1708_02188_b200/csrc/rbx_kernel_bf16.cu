// Instantiation of the step kernel for dtype bf16 (one TU per dtype: parallel builds).
#include "rbx_kernel.cuh"

namespace rbx {
const void* step_kernel_bf16() { return reinterpret_cast<const void*>(&rbx_step_kernel<__nv_bfloat16>); }
}  // namespace rbx
