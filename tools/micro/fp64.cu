// micro-benchmark: fp64 / fp32 FMA latency and throughput, smem latency, __syncthreads cost on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat64(double* out, double a, double b, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat32(float* out, float a, float b, int n, long long* cyc) {
  float x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fmaf(x, b, a);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void thr64(double* out, double a, double b, int n, long long* cyc) {
  double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, b, a); x1 = fma(x1, b, a); x2 = fma(x2, b, a); x3 = fma(x3, b, a);
    x4 = fma(x4, b, a); x5 = fma(x5, b, a); x6 = fma(x6, b, a); x7 = fma(x7, b, a);
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void syncs(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void divs(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void rcps(double* out, double a, int n, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __drcp_rn(x + 1.0);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void barw(int n, long long* cyc) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("bar.sync 1, 32;");
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* d; float* f; long long* c; long long h;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&f, 1 << 20); cudaMalloc(&c, 64);
  int n = 10000;
  lat64<<<1, 32>>>(d, 1.0, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cyc\n", (double)h / n);
  lat32<<<1, 32>>>(f, 1.f, 0.999f, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cyc\n", (double)h / n);
  for (int w : {1, 4, 8, 16, 32}) {
    thr64<<<1, 32 * w>>>(d, 1.0, 0.999, n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput %2d warps/SM: %.2f DFMA/cyc/SM\n", w, 8.0 * n * 32 * w / h);
  }
  syncs<<<1, 256>>>(n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads 256 thr: %.2f cyc\n", (double)h / n);
  divs<<<1, 32>>>(d, 1.0, 1000, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp64 1/x dependent: %.2f cyc\n", (double)h / 1000);
  rcps<<<1, 32>>>(d, 1.0, 1000, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("__drcp_rn dependent: %.2f cyc\n", (double)h / 1000);
  barw<<<1, 32>>>(n, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("bar.sync 1,32 (1 warp): %.2f cyc\n", (double)h / n);
  cudaDeviceSynchronize();
  return 0;
}
