// Instantiation of the step kernel for dtype f16 (one TU per dtype: parallel builds).
#include "rbx_kernel.cuh"

namespace rbx {
const void* step_kernel_f16() { return reinterpret_cast<const void*>(&rbx_step_kernel<__half>); }
}  // namespace rbx
