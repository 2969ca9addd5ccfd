// k_fused_multi_f32.cu -- translation unit of the multi-chain fused sweep kernel, float (fused.cuh)
#include "fused.cuh"
#include "kptr.h"

namespace cps {
const void* fused_multi_ptr_f32(int rows) {
  return rows == 2 ? (const void*)k_sweep_fused_multi<float, 2> : (const void*)k_sweep_fused_multi<float, 1>;
}
}  // namespace cps
