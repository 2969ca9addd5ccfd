// kptr.h -- kernel entry points compiled in their own translation units (k_*.cu) so that the build
// compiles them in parallel and a change to one kernel family recompiles only its unit.  Each getter
// returns the __global__ function pointer the launch code in cpsgd.cu passes to cudaLaunchKernelEx.
#pragma once
#include <cstddef>

namespace cps {

struct PWParams;
template <typename T>
struct FusedParams;

using PWKernel = void (*)(PWParams);
PWKernel pw_kernel(int R);  // k_pw.cu: k_sweep_wide<RMAX>, RMAX = R rounded up to 16 (32, 56, 64)

// k_fused_{f32,f64}.cu, k_fused_multi_{f32,f64}.cu: k_sweep_fused<T, ROWS> / k_sweep_fused_multi<T, ROWS>
const void* fused_ptr_f32(int rows);
const void* fused_ptr_f64(int rows);
const void* fused_multi_ptr_f32(int rows);
const void* fused_multi_ptr_f64(int rows);

template <typename T, int ROWS>
inline void (*fused_k())(FusedParams<T>) {
  return (void (*)(FusedParams<T>))(sizeof(T) == 8 ? fused_ptr_f64(ROWS) : fused_ptr_f32(ROWS));
}
template <typename T, int ROWS>
inline void (*fused_multi_k())(const FusedParams<T>*, int) {
  return (void (*)(const FusedParams<T>*, int))(sizeof(T) == 8 ? fused_multi_ptr_f64(ROWS) : fused_multi_ptr_f32(ROWS));
}

}  // namespace cps
