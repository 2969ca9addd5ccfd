// per-phase cycle accounting of the lane-per-column sweep (software-pipelined form), summed over pivots
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;
template <int RMAX>
__device__ void lc_prof(long long* ts, double* Gm, int R, double tol, double* colbuf, int* swept) {
  constexpr int NT = (RMAX + 31) / 32 * 32;
  const int tid = threadIdx.x, RS = R + 1;
  long long acc[5] = {0, 0, 0, 0, 0};
  if (tid < NT) {
    const int c = tid;
    double v[RMAX];
#pragma unroll
    for (int t = 0; t < RMAX; ++t) v[t] = (t < R && c < R) ? Gm[t * RS + c] : (t == c ? 1.0 : 0.0);
    bool pend = false, kp = false;
    double fp = 0.0;
    const double* cbp = colbuf;
    int b = 0;
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
      long long t0 = clock64();
      double* cb = colbuf + b * RMAX;
      b = (b == 2) ? 0 : b + 1;
      if (c < RMAX) cb[c >= k ? c - k : c - k + RMAX] = v[0];
      if (NT == 32) __syncwarp(); else named_bar_sync(1, NT);
      long long t1 = clock64();
      const double d = cb[0];
      if (d == -12345.0) v[0] = 0;
      long long t2 = clock64();
      if (pend) {
#pragma unroll
        for (int t = 1; t < RMAX - 1; ++t) v[t] = fma(-cbp[t + 1], fp, kp ? 0.0 : v[t]);
      }
      if (v[RMAX - 2] == -12345.0) v[0] = 1;
      long long t3 = clock64();
      if (d > tol) {
        const double dinv = __drcp_rn(d);
        const bool isk = (c == k);
        const double f = isk ? -dinv : v[0] * dinv;
        const double n0 = fma(-cb[1], f, isk ? 0.0 : v[1]);
#pragma unroll
        for (int t = 1; t < RMAX - 1; ++t) v[t] = v[t + 1];
        v[0] = n0;
        v[RMAX - 1] = f;
        pend = true; kp = isk; fp = f; cbp = cb;
      } else {
        const double v0 = v[0];
#pragma unroll
        for (int t = 1; t < RMAX; ++t) v[t - 1] = v[t];
        v[RMAX - 1] = v0;
        pend = false;
      }
      if (v[0] == -12345.0) v[1] = 0;
      long long t4 = clock64();
      acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3;
    }
    if (c < R) for (int t = 0; t < RMAX; ++t) { const int i = t - (RMAX - R); if (i >= 0) Gm[i * RS + c] = -v[t]; }
  }
  if (tid == 0) for (int i = 0; i < 4; ++i) ts[i] = acc[i];
}
template <int RMAX>
__global__ void k(const double* G, int R, double tol, double* out, long long* cyc) {
  __shared__ double Gm[64 * 65];
  __shared__ __align__(16) double buf[512];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G[e];
  __syncthreads();
  long long t0 = clock64();
  lc_prof<RMAX>(cyc + 2, Gm, R, tol, buf, swept);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
}
template <int RMAX>
void run(int R) {
  std::vector<double> A(200 * R), G(R * R, 0.0);
  unsigned s = 1 + R;
  for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
  for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) G[i * R + j] += A[r * R + i] * A[r * R + j];
  double *dG, *dO; long long* dc; long long h[8];
  cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 64);
  cudaMemcpy(dG, G.data(), 8 * R * R, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) k<RMAX><<<1, 256>>>(dG, R, 1e-12, dO, dc);
  cudaMemcpy(h, dc, 48, cudaMemcpyDeviceToHost);
  printf("R=%d RMAX=%d total %lld | per pivot: publish+sync %.0f  d %.0f  pending %.0f  pivot %.0f\n", R, RMAX, h[0],
         (double)h[2] / R, (double)h[3] / R, (double)h[4] / R, (double)h[5] / R);
}
int main() { run<24>(20); run<32>(32); run<56>(50); return 0; }
