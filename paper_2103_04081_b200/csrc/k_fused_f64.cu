// k_fused_f64.cu -- translation unit of the fused single-cluster sweep kernel, double (fused.cuh)
#include "fused.cuh"
#include "kptr.h"

namespace cps {
const void* fused_ptr_f64(int rows) {
  return rows == 2 ? (const void*)k_sweep_fused<double, 2> : (const void*)k_sweep_fused<double, 1>;
}
}  // namespace cps
