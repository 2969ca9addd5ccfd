// Dependent-load latency on B200: pointer chase (ld.global.cg) over a buffer resident in L2, from CTA b of a 148-CTA
// grid (one active thread per CTA, the others idle), stride 4 KB .. 64 KB, and after the buffer was rewritten by
// other SMs (each CTA writes a slice, grid-wide barrier via a second launch).  Prints cycles per load per CTA
// (min / median / max over the CTAs): the spread shows near / far L2 (two dies).
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__global__ void chase(const uint32_t* buf, int steps, long long* out, uint32_t* sink) {
  if (threadIdx.x) return;
  uint32_t i = (blockIdx.x * 977u) % 4096u;
  for (int s = 0; s < 64; ++s) i = __ldcg(buf + i * 64);  // warm (into L2)
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) i = __ldcg(buf + i * 64);
  long long t1 = clock64();
  out[blockIdx.x] = (t1 - t0) / steps;
  sink[blockIdx.x] = i;
}
__global__ void rewrite(uint32_t* buf, int n) {  // every CTA rewrites a slice with the same permutation values
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) buf[e] = buf[e];
}
int main() {
  const int N = 4096;  // nodes, 256 B apart (64 words)
  std::vector<uint32_t> h((size_t)N * 64, 0);
  std::vector<uint32_t> perm(N);
  for (int i = 0; i < N; ++i) perm[i] = i;
  srand(3);
  for (int i = N - 1; i > 0; --i) std::swap(perm[i], perm[rand() % (i + 1)]);
  for (int i = 0; i < N; ++i) h[(size_t)perm[i] * 64] = perm[(i + 1) % N];
  uint32_t *d, *sink;
  long long* out;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&sink, 4096);
  cudaMalloc(&out, 148 * 8);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  std::vector<long long> o(148);
  for (int mode = 0; mode < 2; ++mode) {
    if (mode) rewrite<<<148, 256>>>(d, N * 64);
    chase<<<148, 32>>>(d, 2000, out, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(o.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
    std::sort(o.begin(), o.end());
    printf("%s: cycles per dependent L2 load: min %lld  median %lld  max %lld\n", mode ? "after a rewrite by other SMs" : "resident",
           o[0], o[74], o[147]);
  }
  return 0;
}
