// row-group sweep: thread (g, c) holds rows [g RPG, (g+1) RPG) of column c; no rotation; pivot row
// published by its owner group through shared memory.  Compared against lc_sweep_inverse.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;
template <int RMAX, int G>
__device__ int grp_sweep(double* Gm, int R, double tol, double* rowbuf, int* swept) {
  constexpr int CW = (RMAX + 31) / 32, NT = 32 * CW * G, RPG = (RMAX + G - 1) / G, RB = RPG * G + 8;
  const int tid = threadIdx.x, RS = R + 1;
  if (tid < NT) {
    const int g = tid / (32 * CW), c = tid % (32 * CW);
    double v[RPG];
#pragma unroll
    for (int t = 0; t < RPG; ++t) {
      const int row = g * RPG + t;
      v[t] = (row < R && c < R) ? Gm[row * RS + c] : (row == c ? 1.0 : 0.0);
    }
    for (int j = tid; j < R; j += NT) swept[j] = 0;
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
      double* rb = rowbuf + (k & 1) * RB;
      const int gk = k / RPG, tk = k - gk * RPG;
      if (g == gk) {
        double pv = v[0];
#pragma unroll
        for (int t = 1; t < RPG; ++t) pv = (tk == t) ? v[t] : pv;
        rb[c] = pv;
      }
      named_bar_sync(1, NT);
      const double d = rb[k];
      if (d > tol) {
        const double dinv = __drcp_rn(d);
        const bool isk = (c == k);
        const double f = isk ? -dinv : rb[c] * dinv;
#pragma unroll
        for (int t = 0; t < RPG; ++t) {
          const int row = g * RPG + t;
          v[t] = (row == k) ? f : fma(-rb[row], f, isk ? 0.0 : v[t]);
        }
        if (tid == 0) swept[k] = 1;
      }
    }
    named_bar_sync(1, NT);
    if (c < R) {
#pragma unroll
      for (int t = 0; t < RPG; ++t) {
        const int row = g * RPG + t;
        if (row < R) Gm[row * RS + c] = (swept[row] && swept[c]) ? -v[t] : 0.0;
      }
    }
  }
  __syncthreads();
  int rank = 0;
  for (int j = 0; j < R; ++j) rank += swept[j];
  return rank;
}

// variant: the owner group of row k publishes row k AND 1/d_k (computed by lane k before the barrier)
template <int RMAX, int G>
__device__ int grp_sweep2(double* Gm, int R, double tol, double* rowbuf, int* swept) {
  constexpr int CW = (RMAX + 31) / 32, NT = 32 * CW * G, RPG = (RMAX + G - 1) / G, RB = RPG * G + 8;
  const int tid = threadIdx.x, RS = R + 1;
  if (tid < NT) {
    const int g = tid / (32 * CW), c = tid % (32 * CW);
    double v[RPG];
#pragma unroll
    for (int t = 0; t < RPG; ++t) {
      const int row = g * RPG + t;
      v[t] = (row < R && c < R) ? Gm[row * RS + c] : (row == c ? 1.0 : 0.0);
    }
    for (int j = tid; j < R; j += NT) swept[j] = 0;
#pragma unroll 1
    for (int k = 0; k < R; ++k) {
      double* rb = rowbuf + (k & 1) * RB;
      const int gk = k / RPG, tk = k - gk * RPG;
      if (g == gk) {
        double pv = v[0];
#pragma unroll
        for (int t = 1; t < RPG; ++t) pv = (tk == t) ? v[t] : pv;
        rb[c] = pv;
        if (c == k) rb[RB - 1] = pv > tol ? __drcp_rn(pv) : 0.0;
      }
      named_bar_sync(1, NT);
      const double dinv = rb[RB - 1];
      if (dinv != 0.0) {  // uniform
        const bool isk = (c == k);
        const double f = isk ? -dinv : rb[c] * dinv;
#pragma unroll
        for (int t = 0; t < RPG; ++t) {
          const int row = g * RPG + t;
          v[t] = (row == k) ? f : fma(-rb[row], f, isk ? 0.0 : v[t]);
        }
        if (tid == 0) swept[k] = 1;
      }
    }
    named_bar_sync(1, NT);
    if (c < R) {
#pragma unroll
      for (int t = 0; t < RPG; ++t) {
        const int row = g * RPG + t;
        if (row < R) Gm[row * RS + c] = (swept[row] && swept[c]) ? -v[t] : 0.0;
      }
    }
  }
  __syncthreads();
  int rank = 0;
  for (int j = 0; j < R; ++j) rank += swept[j];
  return rank;
}

// 2x2 block pivots: pivots (k, k+1) share one publish, one barrier and one reciprocal (of the 2x2
// determinant); the natural-order skip rule is kept exactly (a <= tol, or Schur d' = det / a <= tol,
// degrade the pair to single steps).
template <int RMAX, int G>
__device__ int grp_sweep22(double* Gm, int R, double tol, double* rowbuf, int* swept) {
  constexpr int CW = (RMAX + 31) / 32, NT = 32 * CW * G, RPG = (RMAX + G - 1) / G, RB = RPG * G + 8;
  const int tid = threadIdx.x, RS = R + 1;
  if (tid < NT) {
    const int g = tid / (32 * CW), c = tid % (32 * CW);
    double v[RPG];
#pragma unroll
    for (int t = 0; t < RPG; ++t) {
      const int row = g * RPG + t;
      v[t] = (row < R && c < R) ? Gm[row * RS + c] : (row == c ? 1.0 : 0.0);
    }
    for (int j = tid; j < R; j += NT) swept[j] = 0;
    int par = 0;
#pragma unroll 1
    for (int k = 0; k < R; k += 2) {
      const int l = k + 1;  // may be == R (single last pivot)
      double* rb1 = rowbuf + par * 2 * RB;
      double* rb2 = rb1 + RB;
      par ^= 1;
      {
        const int gk = k / RPG, tk = k - gk * RPG;
        if (g == gk) {
          double pv = v[0];
#pragma unroll
          for (int t = 1; t < RPG; ++t) pv = (tk == t) ? v[t] : pv;
          rb1[c] = pv;
        }
        if (l < R) {
          const int gl = l / RPG, tl = l - gl * RPG;
          if (g == gl) {
            double pv = v[0];
#pragma unroll
            for (int t = 1; t < RPG; ++t) pv = (tl == t) ? v[t] : pv;
            rb2[c] = pv;
          }
        }
      }
      named_bar_sync(1, NT);
      const double a = rb1[k];
      const double b = l < R ? rb1[l] : 0.0, cc = l < R ? rb2[l] : 0.0;
      const double det = fma(a, cc, -b * b);
      const bool pair = l < R && a > tol && det > tol * a;
      if (pair) {  // uniform
        const double dinv = __drcp_rn(det);
        double f1, f2;
        if (c == k) { f1 = -cc * dinv; f2 = b * dinv; }
        else if (c == l) { f1 = b * dinv; f2 = -a * dinv; }
        else {
          const double mk = rb1[c], ml = rb2[c];
          f1 = fma(cc, mk, -b * ml) * dinv;
          f2 = fma(a, ml, -b * mk) * dinv;
        }
        const bool isp = (c == k) || (c == l);
#pragma unroll
        for (int t = 0; t < RPG; ++t) {
          const int row = g * RPG + t;
          v[t] = (row == k) ? f1 : (row == l) ? f2 : fma(-rb1[row], f1, fma(-rb2[row], f2, isp ? 0.0 : v[t]));
        }
        if (tid == 0) { swept[k] = 1; swept[l] = 1; }
      } else {
        // single steps in natural order: pivot k (if a > tol), then l on the updated values
        const bool sk = a > tol;
        if (sk) {
          const double dinv = __drcp_rn(a);
          const bool isk = (c == k);
          const double f = isk ? -dinv : rb1[c] * dinv;
#pragma unroll
          for (int t = 0; t < RPG; ++t) {
            const int row = g * RPG + t;
            v[t] = (row == k) ? f : fma(-rb1[row], f, isk ? 0.0 : v[t]);
          }
          if (tid == 0) swept[k] = 1;
        }
        if (l < R) {
          // row / column l after step k: M_lx - M_lk f_x ; its diagonal d = cc - b^2 / a (or cc)
          named_bar_sync(1, NT);  // everyone has read rb1 / rb2 of this pair
          const int gl = l / RPG, tl = l - gl * RPG;
          if (g == gl) {
            double pv = v[0];
#pragma unroll
            for (int t = 1; t < RPG; ++t) pv = (tl == t) ? v[t] : pv;
            rb2[c] = pv;
          }
          named_bar_sync(1, NT);
          const double d = rb2[l];
          if (d > tol) {
            const double dinv = __drcp_rn(d);
            const bool isl = (c == l);
            const double f = isl ? -dinv : rb2[c] * dinv;
#pragma unroll
            for (int t = 0; t < RPG; ++t) {
              const int row = g * RPG + t;
              v[t] = (row == l) ? f : fma(-rb2[row], f, isl ? 0.0 : v[t]);
            }
            if (tid == 0) swept[l] = 1;
          }
        }
      }
    }
    named_bar_sync(1, NT);
    if (c < R) {
#pragma unroll
      for (int t = 0; t < RPG; ++t) {
        const int row = g * RPG + t;
        if (row < R) Gm[row * RS + c] = (swept[row] && swept[c]) ? -v[t] : 0.0;
      }
    }
  }
  __syncthreads();
  int rank = 0;
  for (int j = 0; j < R; ++j) rank += swept[j];
  return rank;
}
template <int RMAX, int G>
__global__ void k(const double* G_, int R, double tol, double* out, long long* cyc, int which) {
  __shared__ double Gm[64 * 65];
  __shared__ __align__(16) double buf[512];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G_[e];
  __syncthreads();
  long long t0 = clock64();
  int rk = which ? grp_sweep22<RMAX, G>(Gm, R, tol, buf, swept) : grp_sweep<RMAX, G>(Gm, R, tol, buf, swept);
  long long t1 = clock64();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = Gm[(e / R) * (R + 1) + e % R];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = rk; }
}
template <int RMAX, int G>
void run(int R, int dup) {
  std::vector<double> A(200 * R), Gh(R * R, 0.0);
  unsigned s = 1 + R;
  for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
  if (dup && R > 2) for (int r = 0; r < 200; ++r) A[r * R + R / 2] = A[r * R + 1] * 2.0;
  for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) Gh[i * R + j] += A[r * R + i] * A[r * R + j];
  double d0 = 0; for (int i = 0; i < R; ++i) d0 = fmax(d0, Gh[i * R + i]);
  double tol = 200 * 2.220446049250313e-16 * d0;
  double *dG, *dO; long long* dc; long long h0[2], h1[2];
  cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 16);
  cudaMemcpy(dG, Gh.data(), 8 * R * R, cudaMemcpyHostToDevice);
  std::vector<double> W0(R * R), W1(R * R);
  for (int rep = 0; rep < 5; ++rep) k<RMAX, G><<<1, 256>>>(dG, R, tol, dO, dc, 0);
  cudaMemcpy(h0, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W0.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
  for (int rep = 0; rep < 5; ++rep) k<RMAX, G><<<1, 256>>>(dG, R, tol, dO, dc, 1);
  cudaMemcpy(h1, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W1.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
  double dif = 0, nrm = 0;
  for (int e = 0; e < R * R; ++e) { dif = fmax(dif, fabs(W0[e] - W1[e])); nrm = fmax(nrm, fabs(W0[e])); }
  printf("dup=%d R=%2d G=%d: grp %6lld (rank %lld) | grp22 %6lld (rank %lld) | rel diff %.2e  err=%s\n", dup, R, G, h0[0], h0[1],
         h1[0], h1[1], dif / nrm, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int dup : {0, 1}) {
    run<8, 4>(5, dup); run<8, 8>(5, dup);
    run<24, 2>(20, dup); run<24, 4>(20, dup); run<24, 8>(20, dup);
    run<32, 4>(32, dup); run<32, 8>(32, dup);
    run<56, 2>(50, dup); run<56, 4>(50, dup);
    run<64, 4>(64, dup);
  }
  return 0;
}
