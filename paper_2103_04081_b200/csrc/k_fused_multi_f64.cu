// k_fused_multi_f64.cu -- translation unit of the multi-chain fused sweep kernel, double (fused.cuh)
#include "fused.cuh"
#include "kptr.h"

namespace cps {
const void* fused_multi_ptr_f64(int rows) {
  return rows == 2 ? (const void*)k_sweep_fused_multi<double, 2> : (const void*)k_sweep_fused_multi<double, 1>;
}
}  // namespace cps
