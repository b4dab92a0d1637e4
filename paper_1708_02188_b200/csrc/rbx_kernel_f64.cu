// Instantiation of the step kernel for dtype f64 (one TU per dtype: parallel builds).
#include "rbx_kernel.cuh"

namespace rbx {
const void* step_kernel_f64() { return reinterpret_cast<const void*>(&rbx_step_kernel<double>); }
}  // namespace rbx
