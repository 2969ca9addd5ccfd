// micro-benchmark: blk_sweep_inverse standalone (cycles per pivot) on sm_100a
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;
__device__ int blk_sweep_dbg(long long* ts, double* Gm, int R, double tol, double* rowbuf /* 2*64 */, int* swept /* R */) {
  const int tid = threadIdx.x, RS = R + 1;
  const int nb = (R + 3) >> 2, nact = nb * nb;
  const int nthr = ((nact + 31) >> 5) << 5;
  if (tid < nthr) {
    const bool act = tid < nact;
    const int bi = act ? tid / nb : -1, bj = act ? tid % nb : -1;
    const int i0 = 4 * (act ? bi : 0), j0 = 4 * (act ? bj : 0);
    double v[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        v[a][c] = (act && i0 + a < R && j0 + c < R) ? Gm[(i0 + a) * RS + j0 + c] : 0.0;
    if (bi == 0)
#pragma unroll
      for (int c = 0; c < 4; ++c) rowbuf[j0 + c] = v[0][c];  // row 0 (zero past R)
    for (int j = tid; j < R; j += nthr) swept[j] = 0;
    named_bar_sync(1, nthr);
    for (int k = 0; k < R; ++k) {
      const double* rk = rowbuf + (k & 1) * 64;
      double* rn = rowbuf + ((k + 1) & 1) * 64;
      if (tid == 0 && k == 10) ts[0] = clock64();
      const double d = rk[k];
      if (tid == 0 && k == 10) ts[1] = clock64();
      if (d > tol) {  // uniform across the participating threads
        const double dinv = __drcp_rn(d);
        if (tid == 0 && k == 10) ts[2] = clock64();
        const double2 ri01 = *reinterpret_cast<const double2*>(rk + i0);
        const double2 ri23 = *reinterpret_cast<const double2*>(rk + i0 + 2);
        const double2 rj01 = *reinterpret_cast<const double2*>(rk + j0);
        const double2 rj23 = *reinterpret_cast<const double2*>(rk + j0 + 2);
        const double ri[4] = {ri01.x, ri01.y, ri23.x, ri23.y};
        const double f[4] = {rj01.x * dinv, rj01.y * dinv, rj23.x * dinv, rj23.y * dinv};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) v[a][c] = fma(-ri[a], f[c], v[a][c]);
        if (tid == 0 && k == 10) ts[3] = clock64();
        const int kb = k >> 2, ks = k & 3;
        if (bi == kb)  // row k: M_kj / d
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) v[a][c] = (a == ks) ? f[c] : v[a][c];
        if (bj == kb)  // column k: M_ik / d, and M_kk = -1/d
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              v[a][c] = (c == ks) ? ((bi == kb && a == ks) ? -dinv : ri[a] * dinv) : v[a][c];
        if (tid == 0) swept[k] = 1;
      }
      if (k + 1 < R && bi == ((k + 1) >> 2)) {  // publish row k+1 for the next pivot
        const int a = (k + 1) & 3;
#pragma unroll
        for (int c = 0; c < 4; ++c) rn[j0 + c] = a == 0 ? v[0][c] : a == 1 ? v[1][c] : a == 2 ? v[2][c] : v[3][c];
      }
      if (tid == 0 && k == 10) ts[4] = clock64();
      named_bar_sync(1, nthr);
      if (tid == 0 && k == 10) ts[5] = clock64();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = i0 + a, j = j0 + c;
        if (act && i < R && j < R) Gm[i * RS + j] = (swept[i] && swept[j]) ? -v[a][c] : 0.0;
      }
  }
  __syncthreads();
  int rank = 0;
  for (int j = 0; j < R; ++j) rank += swept[j];
  return rank;
}


__global__ void k(const double* G, int R, double* out, long long* cyc) {
  __shared__ double Gm[64 * 65];
  __shared__ double rowbuf[128];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G[e];
  __syncthreads();
  long long t0 = clock64();
  int rk = blk_sweep_dbg(cyc + 2, Gm, R, 1e-12, rowbuf, swept);
  long long t1 = clock64();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = Gm[(e / R) * (R + 1) + e % R];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = rk; }
}
int main() {
  for (int R : {5, 20, 32, 50, 64}) {
    std::vector<double> A(200 * R), G(R * R, 0.0);
    unsigned s = 1;
    for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) G[i * R + j] += A[r * R + i] * A[r * R + j];
    double *dG, *dO; long long* dc; long long hc[8];
    cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 64);
    cudaMemcpy(dG, G.data(), 8 * R * R, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) k<<<1, 256>>>(dG, R, dO, dc);
    cudaMemcpy(hc, dc, 64, cudaMemcpyDeviceToHost);
    std::vector<double> W(R * R);
    cudaMemcpy(W.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
    double err = 0;  // ||G W - I||
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) { double t = 0; for (int c = 0; c < R; ++c) t += G[i * R + c] * W[c * R + j]; t -= (i == j); err = fmax(err, fabs(t)); }
    printf("ts: d %lld rcp %lld upd %lld rest %lld bar %lld\n", hc[3]-hc[2], hc[4]-hc[3], hc[5]-hc[4], hc[6]-hc[5], hc[7]-hc[6]);
    printf("R=%2d: %lld cyc (%.0f/pivot), rank %lld, max|GW-I| %.2e\n", R, hc[0], (double)hc[0] / R, hc[1], err);
  }
  return 0;
}
