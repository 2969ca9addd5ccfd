// row-group sweep with static pivot positions (the pair loop unrolled over the owner group's rows:
// publish and pivot-row writes use static register indices, the update of every other entry is two
// DFMA with no selects).  Compared against cps::grp_sweep_inverse.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro/sweep_st tools/micro/sweep_st.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;

template <int RMAX, int G>
__device__ int grp_sweep_st(double* Gm, int R, double tol, double* rowbuf, int* swept) {
  constexpr int CW = (RMAX + 31) / 32, NT = 32 * CW * G, RPG = RMAX / G, RB = RMAX + 8;
  static_assert(RMAX % (2 * G) == 0, "RMAX: a multiple of 2G (pivot pairs never straddle two groups)");
  static_assert(4 * RB <= kSweepBuf, "sweep buffer");
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
    // one sweep step on pivot k = gk RPG + tk (d = M_kk > tol; rb = row k)
    auto single = [&](int gk, int k, int tk, const double* rb, double d) {
      const double dinv = __drcp_rn(d);
      const double f = (c == k) ? -dinv : rb[c] * dinv;
      if (c == k) {
#pragma unroll
        for (int t = 0; t < RPG; ++t) v[t] = 0.0;
      }
#pragma unroll
      for (int t = 0; t < RPG; ++t) v[t] = fma(-rb[g * RPG + t], f, v[t]);
      if (g == gk) v[tk] = f;
      if (tid == 0) swept[k] = 1;
    };
    int par = 0;
#pragma unroll 1
    for (int gk = 0; gk < G; ++gk) {
#pragma unroll
      for (int tk = 0; tk < RPG; tk += 2) {
        const int k = gk * RPG + tk, l = k + 1;  // l == R: the last pivot alone
        if (k < R) {
          double* rb1 = rowbuf + par * 2 * RB;
          double* rb2 = rb1 + RB;
          par ^= 1;
          if (g == gk && c < RMAX) {  // the owner group publishes rows k and l (= columns, by symmetry)
            rb1[c] = v[tk];
            rb2[c] = v[tk + 1];
          }
          named_bar_sync(1, NT);
          const double a = rb1[k], b = rb1[l], cc = rb2[l];  // l < RMAX: row l exists (identity past R)
          const double det = fma(a, cc, -b * b);
          if (l < R && a > tol && det > tol * a) {  // uniform
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
            if (c == k || c == l) {  // the pivot columns start from 0 (M_PP -> -B^{-1})
#pragma unroll
              for (int t = 0; t < RPG; ++t) v[t] = 0.0;
            }
#pragma unroll
            for (int t = 0; t < RPG; ++t) v[t] = fma(-rb1[g * RPG + t], f1, fma(-rb2[g * RPG + t], f2, v[t]));
            if (g == gk) {  // the pivot rows (static register indices)
              v[tk] = f1;
              v[tk + 1] = f2;
            }
            if (tid == 0) {
              swept[k] = 1;
              swept[l] = 1;
            }
          } else {
            if (a > tol) single(gk, k, tk, rb1, a);
            if (l < R) {  // pivot l on the values after step k: republish its row
              named_bar_sync(1, NT);  // every thread is done with rb2
              if (g == gk && c < RMAX) rb2[c] = v[tk + 1];
              named_bar_sync(1, NT);
              const double d = rb2[l];
              if (d > tol) single(gk, l, tk + 1, rb2, d);
            }
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
__device__ int grp_sweep_st2(double* Gm, int R, double tol, double* rowbuf, int* swept) {
  constexpr int CW = (RMAX + 31) / 32, NT = 32 * CW * G, RPG = RMAX / G, RB = RMAX + 8;
  static_assert(RMAX % (2 * G) == 0, "RMAX: a multiple of 2G (pivot pairs never straddle two groups)");
  static_assert(4 * RB <= kSweepBuf, "sweep buffer");
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
    // one sweep step on pivot k = gk RPG + tk (d = M_kk > tol); rb[2 i + o] = M_ki
    auto single = [&](int gk, int k, int tk, const double* rb, int o, double d) {
      const double dinv = __drcp_rn(d);
      const double f = (c == k) ? -dinv : rb[2 * c + o] * dinv;
      if (c == k) {
#pragma unroll
        for (int t = 0; t < RPG; ++t) v[t] = 0.0;
      }
#pragma unroll
      for (int t = 0; t < RPG; ++t) v[t] = fma(-rb[2 * (g * RPG + t) + o], f, v[t]);
      if (g == gk) v[tk] = f;
      if (tid == 0) swept[k] = 1;
    };
    int par = 0;
#pragma unroll 1
    for (int gk = 0; gk < G; ++gk) {
#pragma unroll
      for (int tk = 0; tk < RPG; tk += 2) {
        const int k = gk * RPG + tk, l = k + 1;  // l == R: the last pivot alone
        if (k < R) {
          // rows k and l interleaved: rb[2 i] = M_ki, rb[2 i + 1] = M_li (one 16-byte load per row i)
          double* rb = rowbuf + par * 2 * RB;
          double2* rb2 = reinterpret_cast<double2*>(rb);
          par ^= 1;
          if (g == gk && c < RMAX) rb2[c] = make_double2(v[tk], v[tk + 1]);  // owner group publishes
          named_bar_sync(1, NT);
          const double2 pk = rb2[k], pl = rb2[l];
          const double a = pk.x, b = pk.y, cc = pl.y;  // l < RMAX: row l exists (identity past R)
          const double det = fma(a, cc, -b * b);
          if (l < R && a > tol && det > tol * a) {  // uniform
            const double dinv = __drcp_rn(det);
            const double2 m = rb2[c];
            double f1, f2;
            if (c == k) {
              f1 = -cc * dinv;
              f2 = b * dinv;
            } else if (c == l) {
              f1 = b * dinv;
              f2 = -a * dinv;
            } else {
              f1 = fma(cc, m.x, -b * m.y) * dinv;
              f2 = fma(a, m.y, -b * m.x) * dinv;
            }
            if (c == k || c == l) {  // the pivot columns start from 0 (M_PP -> -B^{-1})
#pragma unroll
              for (int t = 0; t < RPG; ++t) v[t] = 0.0;
            }
#pragma unroll
            for (int t = 0; t < RPG; ++t) {
              const double2 q = rb2[g * RPG + t];
              v[t] = fma(-q.x, f1, fma(-q.y, f2, v[t]));
            }
            if (g == gk) {  // the pivot rows (static register indices)
              v[tk] = f1;
              v[tk + 1] = f2;
            }
            if (tid == 0) {
              swept[k] = 1;
              swept[l] = 1;
            }
          } else {
            if (a > tol) single(gk, k, tk, rb, 0, a);
            if (l < R) {  // pivot l on the values after step k: republish its row
              named_bar_sync(1, NT);  // every thread is done with rb
              if (g == gk && c < RMAX) rb[2 * c + 1] = v[tk + 1];
              named_bar_sync(1, NT);
              const double d = rb[2 * l + 1];
              if (d > tol) single(gk, l, tk + 1, rb, 1, d);
            }
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

// rcp_nr: cps::rcp_nr (kernels.cuh)
template <int RMAX, int G>
__device__ int grp_sweep_st3(double* Gm, int R, double tol, double* rowbuf, int* swept) {
  constexpr int CW = (RMAX + 31) / 32, NT = 32 * CW * G, RPG = RMAX / G, RB = RMAX + 8;
  static_assert(RMAX % (2 * G) == 0, "RMAX: a multiple of 2G (pivot pairs never straddle two groups)");
  static_assert(4 * RB <= kSweepBuf, "sweep buffer");
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
    // one sweep step on pivot k = gk RPG + tk (d = M_kk > tol); rb[2 i + o] = M_ki
    auto single = [&](int gk, int k, int tk, const double* rb, int o, double d) {
      const double dinv = rcp_nr(d);
      const double f = (c == k) ? -dinv : rb[2 * c + o] * dinv;
      if (c == k) {
#pragma unroll
        for (int t = 0; t < RPG; ++t) v[t] = 0.0;
      }
#pragma unroll
      for (int t = 0; t < RPG; ++t) v[t] = fma(-rb[2 * (g * RPG + t) + o], f, v[t]);
      if (g == gk) v[tk] = f;
      if (tid == 0) swept[k] = 1;
    };
    int par = 0;
#pragma unroll 1
    for (int gk = 0; gk < G; ++gk) {
#pragma unroll
      for (int tk = 0; tk < RPG; tk += 2) {
        const int k = gk * RPG + tk, l = k + 1;  // l == R: the last pivot alone
        if (k < R) {
          // rows k and l interleaved: rb[2 i] = M_ki, rb[2 i + 1] = M_li (one 16-byte load per row i)
          double* rb = rowbuf + par * 2 * RB;
          double2* rb2 = reinterpret_cast<double2*>(rb);
          par ^= 1;
          if (g == gk && c < RMAX) rb2[c] = make_double2(v[tk], v[tk + 1]);  // owner group publishes
          named_bar_sync(1, NT);
          const double2 pk = rb2[k], pl = rb2[l];
          const double a = pk.x, b = pk.y, cc = pl.y;  // l < RMAX: row l exists (identity past R)
          const double det = fma(a, cc, -b * b);
          const double2 m = rb2[c];
          const double dinv = rcp_nr(det);  // speculative: overlaps the pivot test
          if (l < R && a > tol && det > tol * a) {  // uniform
            // (f1, f2) = B^{-1} m with m = M_Pc, or m = -e_k / -e_l on the pivot columns (the negated
            // columns of B^{-1}); selects instead of a divergent branch
            const double mx = (c == k) ? -1.0 : (c == l) ? 0.0 : m.x;
            const double my = (c == k) ? 0.0 : (c == l) ? -1.0 : m.y;
            const double f1 = fma(cc, mx, -b * my) * dinv;
            const double f2 = fma(a, my, -b * mx) * dinv;
            if (c == k || c == l) {  // the pivot columns start from 0 (M_PP -> -B^{-1})
#pragma unroll
              for (int t = 0; t < RPG; ++t) v[t] = 0.0;
            }
#pragma unroll
            for (int t = 0; t < RPG; ++t) {
              const double2 q = rb2[g * RPG + t];
              v[t] = fma(-q.x, f1, fma(-q.y, f2, v[t]));
            }
            if (g == gk) {  // the pivot rows (static register indices)
              v[tk] = f1;
              v[tk + 1] = f2;
            }
            if (tid == 0) {
              swept[k] = 1;
              swept[l] = 1;
            }
          } else {
            if (a > tol) single(gk, k, tk, rb, 0, a);
            if (l < R) {  // pivot l on the values after step k: republish its row
              named_bar_sync(1, NT);  // every thread is done with rb
              if (g == gk && c < RMAX) rb[2 * c + 1] = v[tk + 1];
              named_bar_sync(1, NT);
              const double d = rb[2 * l + 1];
              if (d > tol) single(gk, l, tk + 1, rb, 1, d);
            }
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
  __shared__ __align__(16) double buf[8 * 72];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G_[e];
  __syncthreads();
  long long t0 = clock64();
  int rk = which == 3 ? grp_sweep_st3<RMAX, G>(Gm, R, tol, buf, swept) : which == 2 ? grp_sweep_st2<RMAX, G>(Gm, R, tol, buf, swept) : which ? grp_sweep_st<RMAX, G>(Gm, R, tol, buf, swept) : grp_sweep_inverse<RMAX, G>(Gm, R, tol, buf, swept);
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
  long long h2[2]; std::vector<double> W2(R * R);
  for (int rep = 0; rep < 5; ++rep) k<RMAX, 4><<<1, 256>>>(dG, R, tol, dO, dc, 2);
  cudaMemcpy(h2, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W2.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
  double dif2 = 0; for (int e = 0; e < R * R; ++e) dif2 = fmax(dif2, fabs(W0[e] - W2[e]));
  long long h3[2]; std::vector<double> W3(R * R);
  for (int rep = 0; rep < 5; ++rep) k<RMAX, 4><<<1, 256>>>(dG, R, tol, dO, dc, 3);
  cudaMemcpy(h3, dc, 16, cudaMemcpyDeviceToHost); cudaMemcpy(W3.data(), dO, 8 * R * R, cudaMemcpyDeviceToHost);
  double dif3 = 0; for (int e = 0; e < R * R; ++e) dif3 = fmax(dif3, fabs(W0[e] - W3[e]));
  double dif = 0, nrm = 0;
  for (int e = 0; e < R * R; ++e) { dif = fmax(dif, fabs(W0[e] - W1[e])); nrm = fmax(nrm, fabs(W0[e])); }
  printf("dup=%d R=%2d: grp22 %6lld (rank %lld) | grpst %6lld (rank %lld) | rel diff %.2e | st2 %6lld (rank %lld) diff %.2e | st3 %6lld (rank %lld) diff %.2e err=%s\n", dup, R, h0[0], h0[1],
         h1[0], h1[1], dif / nrm, h2[0], h2[1], dif2 / nrm, h3[0], h3[1], dif3 / nrm, cudaGetErrorString(cudaGetLastError()));
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
