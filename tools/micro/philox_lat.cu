// Latency of one Philox4x32-10 draw word + 64-bit scaling (the persistent kernel's per-draw chain), one warp alone
// vs. one warp of a 448-thread CTA whose other warps wait at a barrier.  nvcc ... -I../../paper_2103_04081_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "philox.cuh"
using namespace cps;
__global__ void k(uint64_t seed, uint64_t T, long long* out, uint64_t* sink) {
  uint64_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 64) {
    for (int i = 0; i < 16; ++i) {
      const uint64_t rr = scale_draw(draw_word(seed + acc, 7, threadIdx.x, 0, 1), T);
      acc += rr & 1;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / 16; sink[0] = acc; }
  __syncthreads();
}
int main() {
  long long* o; uint64_t* s; long long h;
  cudaMalloc(&o, 8); cudaMalloc(&s, 8);
  for (int nt : {32, 448}) {
    for (int r = 0; r < 3; ++r) k<<<1, nt>>>(1234, 1ull << 40, o, s);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("%d threads: %lld cycles per dependent draw\n", nt, h);
  }
  return 0;
}
