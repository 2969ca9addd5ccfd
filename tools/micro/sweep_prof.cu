// micro-benchmark: blk_sweep_inverse standalone (cycles per pivot) on sm_100a
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;
__global__ void k(const double* G, int R, double* out, long long* cyc) {
  __shared__ double Gm[64 * 65];
  __shared__ double rowbuf[128];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G[e];
  __syncthreads();
  long long t0 = clock64();
  int rk = 0;
  for (int rep = 0; rep < 500; ++rep) {
    for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G[e];
    __syncthreads();
    rk = blk_sweep_inverse(Gm, R, 1e-12, rowbuf, swept);
  }
  long long t1 = clock64();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = Gm[(e / R) * (R + 1) + e % R];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = rk; }
}
int main() {
  for (int R : {20}) {
    std::vector<double> A(200 * R), G(R * R, 0.0);
    unsigned s = 1;
    for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) G[i * R + j] += A[r * R + i] * A[r * R + j];
    double *dG, *dO; long long* dc; long long hc[2];
    cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 16);
    cudaMemcpy(dG, G.data(), 8 * R * R, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 1; ++rep) k<<<1, 256>>>(dG, R, dO, dc);
    cudaMemcpy(hc, dc, 16, cudaMemcpyDeviceToHost);
    std::vector<double> W(R * R);
    cudaMemcpy(W.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
    double err = 0;  // ||G W - I||
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) { double t = 0; for (int c = 0; c < R; ++c) t += G[i * R + c] * W[c * R + j]; t -= (i == j); err = fmax(err, fabs(t)); }
    printf("R=%2d: %lld cyc (%.0f/pivot), rank %lld, max|GW-I| %.2e\n", R, hc[0], (double)hc[0] / R, hc[1], err);
  }
  return 0;
}
