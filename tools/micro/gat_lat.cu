// latency of one "chunk" of the fused gather: 16 CTAs x 256 threads, each warp-load 128 B of a random
// 1.6 KB fiber segment, 16 fibers x 2 rows per thread in flight; buffer size swept (TLB reach).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
__global__ void k(const float* __restrict__ X, uint64_t nfib, int rep, long long* cyc, float* out, int pf) {
  __shared__ int64_t fb[16];
  float acc = 0.f;
  long long tot = 0;
  for (int r = 0; r < rep; ++r) {
    if (threadIdx.x < 16) fb[threadIdx.x] = (int64_t)(mix(blockIdx.x * 7919ULL + r * 131ULL + threadIdx.x) % nfib) * 400;
    __syncthreads();
    if (pf) {
      for (int e = threadIdx.x; e < 16 * 14; e += 256) {
        const int lb = e / 14, l = e % 14;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(X + fb[lb] + (l * 32 < 400 ? l * 32 : 399)));
      }
      long long w = clock64();
      while (clock64() - w < 20000) {}
    }
    __syncthreads();
    long long t0 = clock64();
    float xv[16][2];
#pragma unroll
    for (int c = 0; c < 16; ++c)
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int i = threadIdx.x + 256 * u;
        xv[c][u] = i < 400 ? __ldg(X + fb[c] + i) : 0.f;
      }
#pragma unroll
    for (int c = 0; c < 16; ++c) acc += xv[c][0] + xv[c][1];
    if (acc == -1.f) out[0] = 1;
    long long t1 = clock64();
    tot += t1 - t0;
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = tot / rep;
  out[blockIdx.x * 256 + threadIdx.x] = acc;
}
int main() {
  float* X; long long* c; float* o; long long h[16];
  const size_t maxb = 8ull << 30;
  cudaMalloc(&X, maxb); cudaMemset(X, 0, maxb); cudaMalloc(&c, 16 * 8); cudaMalloc(&o, 1 << 20);
  for (int pf : {0, 1})
    for (size_t mb : {32, 128, 256, 1024, 4096, 8192}) {
      const uint64_t nfib = (mb << 20) / 1600;
      k<<<16, 256>>>(X, nfib, 20, c, o, pf);
      cudaDeviceSynchronize();
      cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
      long long s = 0; for (int i = 0; i < 16; ++i) s += h[i];
      printf("prefetch=%d buffer %5zu MB: chunk latency %lld cycles\n", pf, mb, s / 16);
    }
  return 0;
}
