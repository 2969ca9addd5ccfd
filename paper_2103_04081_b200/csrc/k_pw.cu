// k_pw.cu -- translation unit of the persistent cooperative sweep kernel (sweep_wide.cuh)
#include "sweep_wide.cuh"
#include "kptr.h"

namespace cps {
PWKernel pw_kernel(int R) {
  return R <= 16 ? k_sweep_wide<16> : R <= 32 ? k_sweep_wide<32> : R <= 56 ? k_sweep_wide<56> : k_sweep_wide<64>;
}
}  // namespace cps
