#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void nb(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__global__ void k1(long long* cyc, int mode) {
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int i = 0; i < 100; ++i) nb(1, 32);
  }
  long long t1 = clock64();
  if (mode) __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
__global__ void k2(long long* cyc, double x) {
  __shared__ double s[64];
  long long t0 = clock64();
  double d = x;
  for (int i = 0; i < 100; ++i) d = __drcp_rn(d + 1.0);
  long long t1 = clock64();
  s[threadIdx.x % 64] = d;
  __syncthreads();
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = (long long)s[5]; }
}
int main() {
  long long* c; long long h[3]; cudaMalloc(&c, 64);
  for (int m = 0; m < 2; ++m) { k1<<<1, 256>>>(c, m); k1<<<1, 256>>>(c, m); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("mode %d: 100 x bar.sync(1,32) = %lld cyc, then syncthreads %lld\n", m, h[0], h[1]); }
  k2<<<1, 256>>>(c, 1.0); k2<<<1, 256>>>(c, 1.0); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("100 drcp 256 thr: %lld cyc; sync %lld\n", h[0], h[1]);
  k2<<<1, 32>>>(c, 1.0); k2<<<1, 32>>>(c, 1.0); cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost); printf("100 drcp 32 thr: %lld cyc\n", h[0]);
  return 0;
}
