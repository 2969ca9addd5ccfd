// Test-only: compares the product's device Philox (paper_2103_04081_b200/csrc/philox.cuh) with
// cuRAND's curand_Philox4x32_10 (library routine, /usr/local/cuda/include/curand_philox4x32_x.h)
// on n counters.  Built on demand by tests/test_gpu_parity.py.
#include <cstdint>
#include <curand_philox4x32_x.h>

#include "../../paper_2103_04081_b200/csrc/philox.cuh"

__global__ void k_check(const uint4* ctr, const uint2* key, uint4* ours, uint4* theirs, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  cps::U4 c{ctr[i].x, ctr[i].y, ctr[i].z, ctr[i].w};
  cps::U4 o = cps::philox10(c, key[i].x, key[i].y);
  ours[i] = make_uint4(o.x, o.y, o.z, o.w);
  theirs[i] = curand_Philox4x32_10(ctr[i], key[i]);
}

extern "C" int philox_check(const void* ctr, const void* key, void* ours, void* theirs, int n) {
  k_check<<<(n + 255) / 256, 256>>>((const uint4*)ctr, (const uint2*)key, (uint4*)ours, (uint4*)theirs, n);
  return (int)cudaDeviceSynchronize();
}
