// Instantiation of the step kernel for dtype f32 (one TU per dtype: parallel builds).
#include "rbx_kernel.cuh"

namespace rbx {
const void* step_kernel_f32() { return reinterpret_cast<const void*>(&rbx_step_kernel<float>); }
}  // namespace rbx
