#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "/root/repo/paper_2103_04081_b200/csrc/kernels.cuh"
using namespace cps;
__device__ int KS;
__device__ __forceinline__ long long stamp_dep(double x) {
  long long t;
  asm volatile("{\n\t.reg .f64 tmp;\n\tadd.f64 tmp, %1, 0d0000000000000000;\n\tmov.u64 %0, %%clock64;\n\t}" : "=l"(t) : "d"(x) : "memory");
  return t;
}
#define ST(i, x) if (k == KS && (tid == 0 || tid == NT - 1)) ts[(tid != 0) * 8 + (i)] = stamp_dep(x)
template <int RMAX, int G>
__device__ int grp_t(double* Gm, int R, double tol, double* rowbuf, int* swept, long long* ts) {
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
          ST(0, v[RPG - 1] + v[0]);
          if (g == gk && c < RMAX) rb2[c] = make_double2(v[tk], v[tk + 1]);  // owner group publishes
          named_bar_sync(1, NT);
          ST(1, 0.0);
          const double2 pk = rb2[k], pl = rb2[l];
          const double a = pk.x, b = pk.y, cc = pl.y;  // l < RMAX: row l exists (identity past R)
          const double det = fma(a, cc, -b * b);
          ST(2, det);
          if (l < R && a > tol && det > tol * a) {  // uniform
            const double dinv = __drcp_rn(det);
            ST(3, dinv);
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
            ST(4, f1 + f2);
            if (c == k || c == l) {  // the pivot columns start from 0 (M_PP -> -B^{-1})
#pragma unroll
              for (int t = 0; t < RPG; ++t) v[t] = 0.0;
            }
#pragma unroll
            for (int t = 0; t < RPG; ++t) {
              const double2 q = rb2[g * RPG + t];
              v[t] = fma(-q.x, f1, fma(-q.y, f2, v[t]));
            }
            ST(5, v[RPG - 1] + v[0]);
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

template <int RMAX>
__global__ void k(const double* G_, int R, double tol, double* out, long long* cyc) {
  __shared__ double Gm[64 * 65];
  __shared__ __align__(16) double buf[8 * 72];
  __shared__ int swept[64];
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) Gm[(e / R) * (R + 1) + e % R] = G_[e];
  __syncthreads();
  long long t0 = clock64();
  int rk = grp_t<RMAX, 4>(Gm, R, tol, buf, swept, cyc + 2);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = rk; }
}
template <int RMAX>
void run(int R, int ks) {
  cudaMemcpyToSymbol(KS, &ks, 4);
  std::vector<double> A(200 * R), Gh(R * R, 0.0);
  unsigned s = 1 + R;
  for (auto& a : A) { s = s * 1664525u + 1013904223u; a = (s >> 8) * (1.0 / 16777216.0) - 0.5; }
  for (int i = 0; i < R; ++i) for (int j = 0; j < R; ++j) for (int r = 0; r < 200; ++r) Gh[i * R + j] += A[r * R + i] * A[r * R + j];
  double d0 = 0; for (int i = 0; i < R; ++i) d0 = fmax(d0, Gh[i * R + i]);
  double tol = R * 2.220446049250313e-16 * d0;
  double *dG, *dO; long long* dc; long long h[26];
  cudaMalloc(&dG, 8 * R * R); cudaMalloc(&dO, 8 * R * R); cudaMalloc(&dc, 26 * 8);
  cudaMemcpy(dG, Gh.data(), 8 * R * R, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 5; ++rep) k<RMAX><<<1, 256>>>(dG, R, tol, dO, dc);
  cudaMemcpy(h, dc, 26 * 8, cudaMemcpyDeviceToHost);
  printf("R=%d k=%d total %lld\n", R, ks, h[0]);
  for (int w = 0; w < 2; ++w) {
    long long* q = h + 2 + 8 * w;
    printf(" thr %s: publish+bar %lld | ld+det %lld | rcp %lld | f %lld | update %lld | next publish start %s\n", w ? "last" : "0", q[1] - q[0], q[2] - q[1], q[3] - q[2], q[4] - q[3], q[5] - q[4], "");
  }
}
int main() { run<56>(50, 20); run<56>(50, 24); run<24>(20, 8); run<24>(20, 12); return 0; }
