// 4x4 block pivots for the row-group sweep inverse: pivots k..k+3 share one publish, one barrier and
// two reciprocals (2x2 block inverse of the 4x4 pivot block through its Schur complement); the
// natural-order skip rule is kept exactly (any of the four Schur diagonals <= tol degrades the block
// to the pair form).  Compared against cps::grp_sweep_inverse (2x2 pairs).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/sweep44 tools/micro/sweep44.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;

template <int RMAX, int G>
__device__ int grp_sweep44(double* Gm, int R, double tol, double* rowbuf, int* swept) {
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
    auto publish = [&](int k, double* rb) {
      const int gk = k / RPG, tk = k - gk * RPG;
      if (g == gk && c < RMAX) {  // lanes past RMAX would write past rb (into the next buffer)
        double pv = v[0];
#pragma unroll
        for (int t = 1; t < RPG; ++t) pv = (tk == t) ? v[t] : pv;
        rb[c] = pv;
      }
    };
    auto single = [&](int k, const double* rb, double d) {
      const double dinv = __drcp_rn(d);
      const bool isk = (c == k);
      const double f = isk ? -dinv : rb[c] * dinv;
#pragma unroll
      for (int t = 0; t < RPG; ++t) {
        const int row = g * RPG + t;
        v[t] = (row == k) ? f : fma(-rb[row], f, isk ? 0.0 : v[t]);
      }
      if (tid == 0) swept[k] = 1;
    };
    // pivots k, l = k + 1 (l may be R: k alone) with rows already published to rb1, rb2 + barrier
    auto pair = [&](int k, double* rb1, double* rb2) {
      const int l = k + 1;
      const double a = rb1[k];
      const double b = l < R ? rb1[l] : 0.0, cc = l < R ? rb2[l] : 0.0;
      const double det = fma(a, cc, -b * b);
      if (l < R && a > tol && det > tol * a) {
        const double dinv = __drcp_rn(det);
        double f1, f2;
        if (c == k) {
          f1 = -cc * dinv;
          f2 = b * dinv;
        } else if (c == l) {
          f1 = b * dinv;
          f2 = -a * dinv;
        } else {
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
        if (tid == 0) {
          swept[k] = 1;
          swept[l] = 1;
        }
      } else {
        if (a > tol) single(k, rb1, a);
        if (l < R) {
          named_bar_sync(1, NT);
          publish(l, rb2);
          named_bar_sync(1, NT);
          const double d = rb2[l];
          if (d > tol) single(l, rb2, d);
        }
      }
    };
    int par = 0, k = 0;
#pragma unroll 1
    for (; k + 4 <= R; k += 4) {
      double* r0 = rowbuf + par * 4 * RB;
      double* r1 = r0 + RB;
      double* r2 = r1 + RB;
      double* r3 = r2 + RB;
      par ^= 1;
      publish(k, r0);
      publish(k + 1, r1);
      publish(k + 2, r2);
      publish(k + 3, r3);
      named_bar_sync(1, NT);
      // B = [[P, Q], [Q^T, S]], P = [[a, b], [b, cc]]
      const double a = r0[k], b = r0[k + 1], q00 = r0[k + 2], q01 = r0[k + 3];
      const double cc = r1[k + 1], q10 = r1[k + 2], q11 = r1[k + 3];
      const double s00 = r2[k + 2], s01 = r2[k + 3], s11 = r3[k + 3];
      const double detP = fma(a, cc, -b * b);
      bool ok = a > tol && detP > tol * a;
      double p00 = 0, p01 = 0, p11 = 0, y00 = 0, y01 = 0, y10 = 0, y11 = 0, t00 = 0, t01 = 0, t11 = 0, detS = 0;
      if (ok) {
        const double rP = __drcp_rn(detP);
        p00 = cc * rP;
        p01 = -b * rP;
        p11 = a * rP;
        y00 = fma(p00, q00, p01 * q10);  // Y = P^{-1} Q
        y01 = fma(p00, q01, p01 * q11);
        y10 = fma(p01, q00, p11 * q10);
        y11 = fma(p01, q01, p11 * q11);
        t00 = s00 - fma(q00, y00, q10 * y10);  // S' = S - Q^T Y (Schur complement)
        t01 = s01 - fma(q00, y01, q10 * y11);
        t11 = s11 - fma(q01, y01, q11 * y11);
        detS = fma(t00, t11, -t01 * t01);
        ok = t00 > tol && detS > tol * t00;
      }
      if (ok) {  // uniform
        const double rS = __drcp_rn(detS);
        const double w00 = t11 * rS, w01 = -t01 * rS, w11 = t00 * rS;  // S'^{-1}
        const double u00 = fma(y00, w00, y01 * w01), u01 = fma(y00, w01, y01 * w11);  // U = Y S'^{-1}
        const double u10 = fma(y10, w00, y11 * w01), u11 = fma(y10, w01, y11 * w11);
        // B^{-1} = [[P^{-1} + U Y^T, -U], [-U^T, S'^{-1}]]
        const double b00 = p00 + fma(u00, y00, u01 * y01), b01 = p01 + fma(u00, y10, u01 * y11);
        const double b11 = p11 + fma(u10, y10, u11 * y11);
        const double b02 = -u00, b03 = -u01, b12 = -u10, b13 = -u11, b22 = w00, b23 = w01, b33 = w11;
        const int jc = c - k;
        const bool isp = (unsigned)jc < 4u;
        double f0, f1, f2, f3;
        if (isp) {  // the negated column jc of B^{-1}
          f0 = -(jc == 0 ? b00 : jc == 1 ? b01 : jc == 2 ? b02 : b03);
          f1 = -(jc == 0 ? b01 : jc == 1 ? b11 : jc == 2 ? b12 : b13);
          f2 = -(jc == 0 ? b02 : jc == 1 ? b12 : jc == 2 ? b22 : b23);
          f3 = -(jc == 0 ? b03 : jc == 1 ? b13 : jc == 2 ? b23 : b33);
        } else {  // B^{-1} M_Pc
          const double m0 = r0[c], m1 = r1[c], m2 = r2[c], m3 = r3[c];
          f0 = fma(b00, m0, fma(b01, m1, fma(b02, m2, b03 * m3)));
          f1 = fma(b01, m0, fma(b11, m1, fma(b12, m2, b13 * m3)));
          f2 = fma(b02, m0, fma(b12, m1, fma(b22, m2, b23 * m3)));
          f3 = fma(b03, m0, fma(b13, m1, fma(b23, m2, b33 * m3)));
        }
#pragma unroll
        for (int t = 0; t < RPG; ++t) {
          const int row = g * RPG + t, jr = row - k;
          const double upd =
              fma(-r0[row], f0, fma(-r1[row], f1, fma(-r2[row], f2, fma(-r3[row], f3, isp ? 0.0 : v[t]))));
          v[t] = jr == 0 ? f0 : jr == 1 ? f1 : jr == 2 ? f2 : jr == 3 ? f3 : upd;
        }
        if (tid == 0) swept[k] = swept[k + 1] = swept[k + 2] = swept[k + 3] = 1;
      } else {  // the pair form for (k, k+1), then (k+2, k+3) on the updated values
        pair(k, r0, r1);
        named_bar_sync(1, NT);  // every thread done with r2, r3
        publish(k + 2, r2);
        publish(k + 3, r3);
        named_bar_sync(1, NT);
        pair(k + 2, r2, r3);
      }
    }
#pragma unroll 1
    for (; k < R; k += 2) {
      double* r0 = rowbuf + par * 4 * RB;
      double* r1 = r0 + RB;
      par ^= 1;
      publish(k, r0);
      if (k + 1 < R) publish(k + 1, r1);
      named_bar_sync(1, NT);
      pair(k, r0, r1);
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
  __shared__ __align__(16) double buf[8 * 72];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G_[e];
  __syncthreads();
  long long t0 = clock64();
  int rk = which ? grp_sweep44<RMAX, G>(Gm, R, tol, buf, swept) : grp_sweep_inverse<RMAX, G>(Gm, R, tol, buf, swept);
  long long t1 = clock64();
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) out[e] = Gm[(e / R) * (R + 1) + e % R];
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = rk; }
}
template <int RMAX>
void run(int R, int dup) {
  std::vector<double> A(200 * R), Gh(R * R, 0.0);
  unsigned s = 1 + R;
  for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
  if (dup && R > 2) for (int r = 0; r < 200; ++r) A[r * R + R / 2] = A[r * R + 1] * 2.0;
  if (dup > 1 && R > 6) for (int r = 0; r < 200; ++r) A[r * R + 5] = A[r * R + 4] - A[r * R + 2];
  for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) Gh[i * R + j] += A[r * R + i] * A[r * R + j];
  double d0 = 0; for (int i = 0; i < R; ++i) d0 = fmax(d0, Gh[i * R + i]);
  double tol = R * 2.220446049250313e-16 * d0;
  double *dG, *dO; long long* dc; long long h0[2], h1[2];
  cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 16);
  cudaMemcpy(dG, Gh.data(), 8 * R * R, cudaMemcpyHostToDevice);
  std::vector<double> W0(R * R), W1(R * R);
  for (int rep = 0; rep < 5; ++rep) k<RMAX, 4><<<1, 256>>>(dG, R, tol, dO, dc, 0);
  cudaMemcpy(h0, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W0.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
  for (int rep = 0; rep < 5; ++rep) k<RMAX, 4><<<1, 256>>>(dG, R, tol, dO, dc, 1);
  cudaMemcpy(h1, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W1.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
  double dif = 0, nrm = 0;
  for (int e = 0; e < R * R; ++e) { dif = fmax(dif, fabs(W0[e] - W1[e])); nrm = fmax(nrm, fabs(W0[e])); }
  printf("dup=%d R=%2d: grp22 %6lld (rank %lld) | grp44 %6lld (rank %lld) | rel diff %.2e  err=%s\n", dup, R, h0[0], h0[1],
         h1[0], h1[1], dif / nrm, cudaGetErrorString(cudaGetLastError()));
  cudaFree(dG); cudaFree(dO); cudaFree(dc);
}
int main() {
  for (int dup : {0, 1, 2}) {
    run<8>(5, dup); run<8>(8, dup);
    run<24>(20, dup); run<24>(23, dup);
    run<32>(32, dup);
    run<56>(50, dup); run<56>(53, dup);
    run<64>(64, dup);
  }
  return 0;
}
