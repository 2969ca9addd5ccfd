// micro-benchmark + check: blk4_sweep_inverse vs blk_sweep_inverse (cycles, agreement, rank rule)
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;
template <int V>
__global__ void k(const double* G, int R, double tol, double* out, long long* cyc) {
  __shared__ double Gm[64 * 65];
  __shared__ __align__(16) double buf[512];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G[e];
  __syncthreads();
  long long t0 = clock64();
  int rk = V == 4 ? grp_sweep_dispatch(Gm, R, tol, buf, swept) : cta_sweep_inverse_pivoted<16>(Gm, R, tol, buf, swept, buf + 64);
  long long t1 = clock64();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = Gm[(e / R) * (R + 1) + e % R];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = rk; }
}
int main() {
  for (int dup : {0, 1})
  for (int R : {1, 3, 5, 10, 20, 32, 50, 64}) {
    std::vector<double> A(200 * R), G(R * R, 0.0);
    unsigned s = 1 + R;
    for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
    if (dup && R > 2) for (int r = 0; r < 200; ++r) A[r * R + R / 2] = A[r * R + 1] * 2.0;  // dependent column
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) G[i * R + j] += A[r * R + i] * A[r * R + j];
    double d0 = 0; for (int i = 0; i < R; ++i) d0 = fmax(d0, G[i * R + i]);
    double tol = 200 * 2.220446049250313e-16 * d0;
    double *dG, *dO; long long* dc; long long h4[2], h1[2];
    cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 16);
    cudaMemcpy(dG, G.data(), 8 * R * R, cudaMemcpyHostToDevice);
    std::vector<double> W4(R * R), W1(R * R);
    for (int rep = 0; rep < 3; ++rep) k<4><<<1, 256>>>(dG, R, tol, dO, dc);
    cudaMemcpy(h4, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W4.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
    for (int rep = 0; rep < 3; ++rep) k<1><<<1, 256>>>(dG, R, tol, dO, dc);
    cudaMemcpy(h1, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W1.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
    double dif = 0, nrm = 0;
    for (int e = 0; e < R * R; ++e) { dif = fmax(dif, fabs(W4[e] - W1[e])); nrm = fmax(nrm, fabs(W1[e])); }
    printf("dup=%d R=%2d: lc %6lld cyc rank %lld | pivoted %6lld cyc rank %lld | max|Wlc-Wpiv|/max|W1| %.2e\n", dup, R, h4[0], h4[1], h1[0], h1[1], dif / nrm);
  }
  return 0;
}
