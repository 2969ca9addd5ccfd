// micro-benchmark + check: blk4_sweep_inverse vs blk_sweep_inverse (cycles, agreement, rank rule)
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;
__device__ int blk4_dbg(long long* ts, double* Gm, int R, double tol, double* colbuf /* 2*64*4 */, int* swept /* R */) {
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
    // column block 0: colbuf[par][row][4]
    if (bj == 0)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        double2* d = reinterpret_cast<double2*>(colbuf + (i0 + a) * 4);
        d[0] = make_double2(v[a][0], v[a][1]);
        d[1] = make_double2(v[a][2], v[a][3]);
      }
    for (int j = tid; j < R; j += nthr) swept[j] = 0;
    named_bar_sync(1, nthr);
    if (tid == 0) ts[0] = clock64();
    for (int kb = 0; kb < nb; ++kb) {
      const double* cb = colbuf + (kb & 1) * 256;
      double* cn = colbuf + ((kb + 1) & 1) * 256;
      const int k0 = 4 * kb;
      // D = M_KK, swept one pivot at a time (every thread, identical arithmetic)
      double D[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double2 x = *reinterpret_cast<const double2*>(cb + (k0 + a) * 4);
        const double2 y = *reinterpret_cast<const double2*>(cb + (k0 + a) * 4 + 2);
        D[a][0] = x.x; D[a][1] = x.y; D[a][2] = y.x; D[a][3] = y.y;
      }
      bool piv[4];
      if (tid == 0 && kb == 0) ts[1] = clock64();

#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const double d = D[s][s];
        piv[s] = (k0 + s < R) && d > tol;
        if (piv[s]) {
          const double dinv = __drcp_rn(d);
          double col[4], row[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            col[a] = D[a][s];
            row[a] = D[s][a] * dinv;
          }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double nv = fma(-col[a], row[c], D[a][c]);
              nv = (a == s) ? row[c] : nv;
              nv = (c == s) ? col[a] * dinv : nv;
              D[a][c] = (a == s && c == s) ? -dinv : nv;
            }
        }
      }
      double Q[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) Q[a][c] = piv[c] ? -D[a][c] : 0.0;
      if (tid == 0 && kb == 0) ts[2] = clock64();

      if (tid == 0)
#pragma unroll
        for (int s = 0; s < 4; ++s)
          if (k0 + s < R) swept[k0 + s] = piv[s] ? 1 : 0;
      if (act) {
        double Ci[4][4], Cj[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const double2 x = *reinterpret_cast<const double2*>(cb + (i0 + a) * 4);
          const double2 y = *reinterpret_cast<const double2*>(cb + (i0 + a) * 4 + 2);
          Ci[a][0] = x.x; Ci[a][1] = x.y; Ci[a][2] = y.x; Ci[a][3] = y.y;
          const double2 z = *reinterpret_cast<const double2*>(cb + (j0 + a) * 4);
          const double2 w = *reinterpret_cast<const double2*>(cb + (j0 + a) * 4 + 2);
          Cj[a][0] = z.x; Cj[a][1] = z.y; Cj[a][2] = w.x; Cj[a][3] = w.y;
        }
        if (bi != kb && bj != kb) {
          double X[4][4];  // X = C_i Hm
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              double t = 0.0;
#pragma unroll
              for (int u = 0; u < 4; ++u) t = fma(Ci[a][u], piv[u] ? Q[u][s] : 0.0, t);
              X[a][s] = t;
            }
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double t = v[a][c];
#pragma unroll
              for (int s = 0; s < 4; ++s) t = fma(-X[a][s], Cj[c][s], t);
              v[a][c] = t;
            }
        } else if (bi == kb && bj != kb) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double t = piv[a] ? 0.0 : v[a][c];
#pragma unroll
              for (int s = 0; s < 4; ++s) t = fma(Q[a][s], Cj[c][s], t);
              v[a][c] = t;
            }
        } else if (bj == kb && bi != kb) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              double t = piv[c] ? 0.0 : v[a][c];
#pragma unroll
              for (int s = 0; s < 4; ++s) t = fma(Ci[a][s], Q[c][s], t);
              v[a][c] = t;
            }
        } else {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) v[a][c] = D[a][c];
        }
        if (tid == 0 && kb == 0) ts[3] = clock64();
        if (bj == kb + 1)  // publish the next column block
#pragma unroll
          for (int a = 0; a < 4; ++a) {
            double2* d = reinterpret_cast<double2*>(cn + (i0 + a) * 4);
            d[0] = make_double2(v[a][0], v[a][1]);
            d[1] = make_double2(v[a][2], v[a][3]);
          }
      }
      if (tid == 0 && kb == 0) ts[4] = clock64();
      named_bar_sync(1, nthr);
      if (tid == 0 && kb == 0) ts[5] = clock64();
    }
    if (tid == 0) ts[6] = clock64();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = i0 + a, j = j0 + c;
        if (act && i < R && j < R) Gm[i * RS + j] = (swept[i] && swept[j]) ? -v[a][c] : 0.0;
      }
  }
  if (tid == 0) ts[7] = clock64();
  __syncthreads();
  if (tid == 0) ts[8] = clock64();
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
  int rk = V == 4 ? blk4_dbg(cyc + 2, Gm, R, tol, buf, swept) : blk_sweep_inverse(Gm, R, tol, buf, swept);
  long long t1 = clock64();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = Gm[(e / R) * (R + 1) + e % R];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = rk; }
}
int main() {
  for (int dup : {0})
  for (int R : {1, 3, 5, 10, 20, 32, 50, 64}) {
    std::vector<double> A(200 * R), G(R * R, 0.0);
    unsigned s = 1 + R;
    for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
    if (dup && R > 2) for (int r = 0; r < 200; ++r) A[r * R + R / 2] = A[r * R + 1] * 2.0;  // dependent column
    for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) G[i * R + j] += A[r * R + i] * A[r * R + j];
    double d0 = 0; for (int i = 0; i < R; ++i) d0 = fmax(d0, G[i * R + i]);
    double tol = 200 * 2.220446049250313e-16 * d0;
    double *dG, *dO; long long* dc; long long h4[12], h1[12];
    cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 128);
    cudaMemcpy(dG, G.data(), 8 * R * R, cudaMemcpyHostToDevice);
    std::vector<double> W4(R * R), W1(R * R);
    for (int rep = 0; rep < 3; ++rep) k<4><<<1, 256>>>(dG, R, tol, dO, dc);
    cudaMemcpy(h4, dc, 128, cudaMemcpyDeviceToHost); cudaMemcpy(W4.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
    for (int rep = 0; rep < 3; ++rep) k<1><<<1, 256>>>(dG, R, tol, dO, dc);
    cudaMemcpy(h1, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W1.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
    printf("t0=start: load+D %lld Q %lld upd %lld pub %lld bar %lld | rest %lld | write %lld sync %lld\n", h4[3]-h4[2], h4[4]-h4[3], h4[5]-h4[4], h4[6]-h4[5], h4[7]-h4[6], h4[8]-h4[7], h4[9]-h4[8], h4[10]-h4[9]);
    double dif = 0, nrm = 0;
    for (int e = 0; e < R * R; ++e) { dif = fmax(dif, fabs(W4[e] - W1[e])); nrm = fmax(nrm, fabs(W1[e])); }
    printf("dup=%d R=%2d: blk4 %6lld cyc rank %lld | blk %6lld cyc rank %lld | max|W4-W1|/max|W1| %.2e\n", dup, R, h4[0], h4[1], h1[0], h1[1], dif / nrm);
  }
  return 0;
}
