// micro-benchmark: random 512-byte row gathers from a buffer of S bytes (TLB reach test on B200)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
// each warp: nseg random segments of `seg` bytes (lanes read 16 B each, seg/512 loads per lane)
__global__ void k(const float4* __restrict__ X, uint64_t nrows, int row_vec, int seg_vec, int nseg, uint64_t seed, float* out) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int s = 0; s < nseg; s += 4) {
    float4 v[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t row = mix(seed ^ (w * 1000003ULL + s + u)) % nrows;
      const float4* p = X + row * row_vec;
#pragma unroll
      for (int t = 0; t < 2; ++t) v[u][t] = (lane + 32 * t < seg_vec) ? __ldg(p + lane + 32 * t) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int t = 0; t < 2; ++t) { acc.x += v[u][t].x; acc.y += v[u][t].y; }
  }
  if (acc.x == 12345.f) out[0] = acc.y;
}
int main() {
  size_t free_b, tot;
  cudaMemGetInfo(&free_b, &tot);
  const size_t maxS = (size_t)64 << 30;
  float4* X; float* out;
  if (cudaMalloc(&X, maxS) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(X, 0, maxS);
  cudaMalloc(&out, 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int segB : {512, 1024}) {
    for (size_t S : {(size_t)256 << 20, (size_t)1 << 30, (size_t)4 << 30, (size_t)16 << 30, (size_t)32 << 30, (size_t)64 << 30}) {
      const int row_vec = 8192 / 16;  // rows of 8 KB (like a 2000-float fiber)
      const uint64_t nrows = S / 8192;
      const int seg_vec = segB / 16;
      const int blocks = 148 * 8, threads = 256, nseg = 64;
      k<<<blocks, threads>>>(X, nrows, row_vec, seg_vec, nseg, 1, out);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(X, nrows, row_vec, seg_vec, nseg, 7 + r, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double bytes = 5.0 * blocks * (threads / 32) * nseg * segB;
      printf("seg %4d B, buffer %6.2f GB: %7.1f GB/s\n", segB, S / 1073741824.0, bytes / (ms * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
