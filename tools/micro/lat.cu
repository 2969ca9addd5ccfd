// latency microbenchmark: dependent chains of one warp (and bar.sync with 448 threads) on this part
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* outd, float* outf, long long* t, int n) {
  __shared__ double sd[64];
  __shared__ float sf[64];
  __shared__ int si[64];
  const int tid = threadIdx.x;
  if (tid < 64) { sd[tid] = 1.0 + tid * 1e-9; sf[tid] = 1.f; si[tid] = (tid + 1) & 63; }
  __syncthreads();
  double x = outd[tid], y = 1.0000001;
  float xf = outf[tid], yf = 1.0001f;
  long long t0, t1;
  if (tid < 32) {
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
    t1 = clock64();
    if (tid == 0) t[0] = t1 - t0;
    // FFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) xf = fmaf(xf, yf, 1e-9f);
    t1 = clock64();
    if (tid == 0) t[1] = t1 - t0;
    // LDS pointer chase
    int j = tid & 63;
    t0 = clock64();
    for (int i = 0; i < n; ++i) j = si[j];
    t1 = clock64();
    if (tid == 0) t[2] = t1 - t0;
    outd[tid] = x + j;
    // MUFU rcp64h + 2 Newton (rcp_nr form)
    double z = x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(z));
      double e = fma(-z, r, 1.0);
      r = fma(r, e, r);
      z = r + 1.0;
    }
    t1 = clock64();
    if (tid == 0) t[3] = t1 - t0;
    outd[tid] += z;
    // SHFL chain
    int v = tid;
    t0 = clock64();
    for (int i = 0; i < n; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
    t1 = clock64();
    if (tid == 0) t[4] = t1 - t0;
    outd[tid] += v;
    // fp64 division (__ddiv_rn)
    z = x;
    t0 = clock64();
    for (int i = 0; i < n; ++i) z = __ddiv_rn(1.0, z + 1.0);
    t1 = clock64();
    if (tid == 0) t[5] = t1 - t0;
    outd[tid] += z;
    // LDS.64 double chase (value-dependent address)
    double w = sd[tid & 63];
    t0 = clock64();
    for (int i = 0; i < n; ++i) w = sd[((int)(w * 0.0)) + (i & 63)] + w * 0.0;
    t1 = clock64();
    if (tid == 0) t[6] = t1 - t0;
    outd[tid] += w;
  }
  __syncthreads();
  // bar.sync round trip with the whole block
  t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) t[7] = t1 - t0;
  // global load chain (L2-resident): pointer chase
  if (tid == 0) {
    const int* g = reinterpret_cast<const int*>(outf + 1024);
    int p = 0;
    t0 = clock64();
    for (int i = 0; i < 64; ++i) p = __ldcg(g + p);
    t1 = clock64();
    t[8] = (t1 - t0) * n / 64;
    outd[0] += p;
  }
}
int main() {
  double* d; float* f; long long* t;
  cudaMalloc(&d, 1 << 20); cudaMalloc(&f, 1 << 22); cudaMalloc(&t, 1024);
  cudaMemset(d, 0, 1 << 20); cudaMemset(f, 0, 1 << 22);
  // chase table: next index (stride 32 ints = 128 B)
  int h[1 << 16];
  for (int i = 0; i < (1 << 16); ++i) h[i] = (i + 4096 + 32) % (1 << 16);
  cudaMemcpy(((char*)f) + 4096, h, sizeof h, cudaMemcpyHostToDevice);
  const int n = 1000;
  for (int rep = 0; rep < 2; ++rep) k<<<1, 448>>>(d, f, t, n);
  cudaDeviceSynchronize();
  long long ht[16];
  cudaMemcpy(ht, t, sizeof ht, cudaMemcpyDeviceToHost);
  const char* nm[] = {"DFMA", "FFMA", "LDS.32 chase", "rcp64h+2DFMA+DADD", "SHFL+IADD", "DDIV", "LDS.64+DFMA", "bar.sync 448", "LDG.cg L2 chase"};
  for (int i = 0; i < 9; ++i) printf("%-22s %6.1f cycles/iter\n", nm[i], (double)ht[i] / n);
  return 0;
}
