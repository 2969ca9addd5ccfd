// micro-benchmark + check: blk4_sweep_inverse vs blk_sweep_inverse (cycles, agreement, rank rule)
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;
template <int RMAX>
__device__ int lc_dbg(long long* ts, double* Gm, int R, double tol, double* colbuf /* 2*RMAX */, int* swept /* R */) {
  constexpr int NT = (RMAX + 31) / 32 * 32;
  const int tid = threadIdx.x, RS = R + 1;
  if (tid < NT) {
    const int c = tid;
    double v[RMAX];
#pragma unroll
    for (int t = 0; t < RMAX; ++t) v[t] = (t < R && c < R) ? Gm[t * RS + c] : (t == c ? 1.0 : 0.0);
    for (int j = tid; j < R; j += NT) swept[j] = 0;
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
      if (tid == 0 && k == 3) ts[0] = clock64();
      if (tid == 0 && k == 4) ts[5] = clock64();
      double* cb = colbuf + (k & 1) * RMAX;
      if (c < RMAX) cb[c >= k ? c - k : c - k + RMAX] = v[0];
      if (NT == 32) __syncwarp();
      else named_bar_sync(1, NT);
      if (tid == 0 && k == 3) ts[1] = clock64();
      const double d = cb[0];
      if (d > tol) {  // uniform
        if (tid == 0 && k == 3) ts[2] = clock64();
        const double dinv = __drcp_rn(d);
        if (tid == 0 && k == 3) ts[3] = clock64();
        const bool isk = (c == k);
        const double f = isk ? -dinv : v[0] * dinv;
#pragma unroll
        for (int u = 0; u < RMAX; u += 2) {  // (c_u, c_{u+1}) per broadcast load
          const double2 cc = *reinterpret_cast<const double2*>(cb + u);
          if (u >= 1) v[u - 1] = fma(-cc.x, f, isk ? 0.0 : v[u]);
          v[u] = fma(-cc.y, f, isk ? 0.0 : v[u + 1]);
        }
        v[RMAX - 1] = f;
        if (tid == 0 && k == 3) ts[4] = clock64();
        if (tid == 0) swept[k] = 1;
      } else {
        const double v0 = v[0];
#pragma unroll
        for (int t = 1; t < RMAX; ++t) v[t - 1] = v[t];
        v[RMAX - 1] = v0;
      }
    }
    if (NT == 32) __syncwarp();
    else named_bar_sync(1, NT);
    if (c < R) {
#pragma unroll
      for (int t = 0; t < RMAX; ++t) {
        const int i = t - (RMAX - R);  // slot t holds row (R + t) mod RMAX
        if (i >= 0) Gm[i * RS + c] = (swept[i] && swept[c]) ? -v[t] : 0.0;
      }
    }
  }
  __syncthreads();
  int rank = 0;
  for (int j = 0; j < R; ++j) rank += swept[j];
  return rank;
}

template <int V>
__global__ void k(const double* G, int R, double tol, double* out, long long* cyc) {
  __shared__ double Gm[64 * 65];
  __shared__ double buf[512];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G[e];
  __syncthreads();
  long long t0 = clock64();
  int rk = lc_dbg<24>(cyc + 2, Gm, R, tol, buf, swept);
  long long t1 = clock64();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = Gm[(e / R) * (R + 1) + e % R];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = rk; }
}
int main() {
  for (int dup : {0})
  for (int R : {20}) {
    std::vector<double> A(200 * R), G(R * R, 0.0);
    unsigned s = 1 + R;
    for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
    if (dup && R > 2) for (int r = 0; r < 200; ++r) A[r * R + R / 2] = A[r * R + 1] * 2.0;  // dependent column
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) G[i * R + j] += A[r * R + i] * A[r * R + j];
    double d0 = 0; for (int i = 0; i < R; ++i) d0 = fmax(d0, G[i * R + i]);
    double tol = 200 * 2.220446049250313e-16 * d0;
    double *dG, *dO; long long* dc; long long h4[16], h1[16];
    cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 128);
    cudaMemcpy(dG, G.data(), 8 * R * R, cudaMemcpyHostToDevice);
    std::vector<double> W4(R * R), W1(R * R);
    for (int rep = 0; rep < 3; ++rep) k<4><<<1, 256>>>(dG, R, tol, dO, dc);
    cudaMemcpy(h4, dc, 128, cudaMemcpyDeviceToHost); cudaMemcpy(W4.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
    h1[0] = h1[1] = 0; W1 = W4;
    printf("publish+sync %lld  ld d %lld  rcp %lld  update %lld | pivot start-to-start %lld\n", h4[3]-h4[2], h4[4]-h4[3], h4[5]-h4[4], h4[6]-h4[5], h4[7]-h4[2]);
    double dif = 0, nrm = 0;
    for (int e = 0; e < R * R; ++e) { dif = fmax(dif, fabs(W4[e] - W1[e])); nrm = fmax(nrm, fabs(W1[e])); }
    printf("dup=%d R=%2d: lc %6lld cyc rank %lld | blk %6lld cyc rank %lld | max|Wlc-Wblk|/max|W1| %.2e\n", dup, R, h4[0], h4[1], h1[0], h1[1], dif / nrm);
  }
  return 0;
}
