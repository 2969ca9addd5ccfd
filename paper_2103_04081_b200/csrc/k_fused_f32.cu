// k_fused_f32.cu -- translation unit of the fused single-cluster sweep kernel, float (fused.cuh)
#include "fused.cuh"
#include "kptr.h"

namespace cps {
const void* fused_ptr_f32(int rows) {
  return rows == 2 ? (const void*)k_sweep_fused<float, 2> : (const void*)k_sweep_fused<float, 1>;
}
}  // namespace cps
