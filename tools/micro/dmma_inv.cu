// Blocked symmetric sweep inverse on fp64 tensor cores (mma.sync m8n8k4 f64), one 448-thread CTA:
// the RMAX x RMAX matrix lives in DMMA accumulator fragments (8x8 tiles round-robin over the 14 warps); per
// 8-pivot block: the block row is published to shared memory, warps 0..NB-1 sweep the 8x8 pivot block in
// registers (shuffles; 2x2 sub-pivots) and form F = B^-1 M_P,: (one 8x8 column block each, 2 DMMA), then
// every warp updates its tiles: C -= M_:,P F (2 DMMA per tile), the pivot row / column blocks <- F / F^T,
// the pivot block <- -B^-1.  Compared with a host Gauss-Jordan inverse; cycles per call.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_inv dmma_inv.cu && ./dmma_inv
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

#ifndef TIMING_ONE_WARP
#define TIMING_ONE_WARP 0
#endif
constexpr int kThreads = 448, kWarps = 14;

template <int RMAX>
__global__ void __launch_bounds__(kThreads, 1) kinv(const double* G, int R, double tol, double* W, int* status,
                                                    long long* cyc) {
  constexpr int NB = RMAX / 8, NT = NB * NB, TPW = (NT + kWarps - 1) / kWarps, LD = RMAX + 2;
  __shared__ double Prow[2][8 * LD];  // published pivot rows: [p][c]
  __shared__ double Fb[8 * LD];       // F = B^-1 M_P,: : [p][c]
  __shared__ double NB_[64];          // -B^-1
  __shared__ int s_fail;
  __shared__ long long tacc[4];
  if (threadIdx.x < 4) tacc[threadIdx.x] = 0;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, gr = lane >> 2, gc = lane & 3;
  if (tid == 0) s_fail = 0;
  // accumulator fragments: tile t = w + kWarps * j -> (I = t / NB, J = t % NB); lane holds (8I + gr, 8J + 2gc + {0,1})
  double c0[TPW], c1[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int t = w + kWarps * j;
    const int I = t / NB, J = t % NB, r = 8 * I + gr, c = 8 * J + 2 * gc;
    auto at = [&](int rr, int cc) { return rr < R && cc < R ? G[rr * R + cc] : (rr == cc ? 1.0 : 0.0); };
    c0[j] = t < NT ? at(r, c) : 0.0;
    c1[j] = t < NT ? at(r, c + 1) : 0.0;
  }
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 1
  for (int kb = 0; kb < NB; ++kb) {
    double* P = Prow[kb & 1];
    // publish block row kb
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int t = w + kWarps * j;
      if (t < NT && t / NB == kb) {
        const int J = t % NB;
        P[gr * LD + 8 * J + 2 * gc] = c0[j];
        P[gr * LD + 8 * J + 2 * gc + 1] = c1[j];
      }
    }
    __syncthreads();
    long long ta = clock64();
    if (w == 0) {
      // the 8x8 pivot block B = P[:, 8kb..]: lane (gr, gc) holds B[gr][2gc], B[gr][2gc+1]; natural-order sweep
      double b0 = P[gr * LD + 8 * kb + 2 * gc], b1 = P[gr * LD + 8 * kb + 2 * gc + 1];
      bool bad = false;
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const int h = k >> 1;
        const double rk0 = __shfl_sync(0xffffffffu, b0, 4 * k + gc), rk1 = __shfl_sync(0xffffffffu, b1, 4 * k + gc);
        const double rl0 = __shfl_sync(0xffffffffu, b0, 4 * (k + 1) + gc), rl1 = __shfl_sync(0xffffffffu, b1, 4 * (k + 1) + gc);
        const double mk = __shfl_sync(0xffffffffu, b0, 4 * gr + h), ml = __shfl_sync(0xffffffffu, b1, 4 * gr + h);
        const double a = __shfl_sync(0xffffffffu, b0, 4 * k + h), bb = __shfl_sync(0xffffffffu, b1, 4 * k + h);
        const double cc = __shfl_sync(0xffffffffu, b1, 4 * (k + 1) + h);
        const double det = fma(a, cc, -bb * bb);
        if (8 * kb + k < R && !(a > tol && det > tol * a)) bad = true;
        const double dinv = rcp_nr(det);
        const double g1 = fma(cc, mk, -bb * ml) * dinv, g2 = fma(a, ml, -bb * mk) * dinv;
        const bool pr = (gr == k || gr == k + 1);
        // select-free: pivot-row values, pivot-column values, general values, then one select per entry
        const double adj0 = (gr == 2 * gc) ? ((2 * gc == k) ? cc : a) : -bb;
        const double adj1 = (gr == 2 * gc + 1) ? ((2 * gc + 1 == k) ? cc : a) : -bb;
        const double prow0 = (gr == k) ? fma(cc, rk0, -bb * rl0) * dinv : fma(a, rl0, -bb * rk0) * dinv;
        const double prow1 = (gr == k) ? fma(cc, rk1, -bb * rl1) * dinv : fma(a, rl1, -bb * rk1) * dinv;
        const double gen0 = fma(-g1, rk0, fma(-g2, rl0, b0)), gen1 = fma(-g1, rk1, fma(-g2, rl1, b1));
        const bool pc0 = (2 * gc == k || 2 * gc == k + 1), pc1 = (2 * gc + 1 == k || 2 * gc + 1 == k + 1);
        b0 = pc0 ? (pr ? -adj0 * dinv : (2 * gc == k ? g1 : g2)) : (pr ? prow0 : gen0);
        b1 = pc1 ? (pr ? -adj1 * dinv : (2 * gc + 1 == k ? g1 : g2)) : (pr ? prow1 : gen1);
      }
      if (bad && lane == 0) s_fail = 1;
      NB_[gr * 8 + 2 * gc] = b0;  // -B^-1
      NB_[gr * 8 + 2 * gc + 1] = b1;
      if (tid == 0) tacc[0] += clock64() - ta;
    }
    __syncthreads();
    if (w < NB) {
      // F_J for J = w: A = B^-1 row-major a[gr][gc + 4h], B operand b[k = gc + 4h][n = gr] = P[gc + 4h][8J + gr]
      const double a_lo = -NB_[gr * 8 + gc], a_hi = -NB_[gr * 8 + gc + 4];
      const int J = w;
      double f0 = 0.0, f1 = 0.0;
      dmma(f0, f1, a_lo, P[gc * LD + 8 * J + gr]);
      dmma(f0, f1, a_hi, P[(gc + 4) * LD + 8 * J + gr]);
      Fb[gr * LD + 8 * J + 2 * gc] = f0;
      Fb[gr * LD + 8 * J + 2 * gc + 1] = f1;
    }
    __syncthreads();
    if (tid == 0) tacc[1] += clock64() - ta;
    if (s_fail) break;
    long long tu = clock64();
    // tile updates
#pragma unroll
    for (int j = 0; j < TPW; ++j) {
      const int t = w + kWarps * j;
      if (t >= NT) continue;
      const int I = t / NB, J = t % NB;
      if (I == kb && J == kb) {
        c0[j] = NB_[gr * 8 + 2 * gc];
        c1[j] = NB_[gr * 8 + 2 * gc + 1];
      } else if (I == kb) {
        c0[j] = Fb[gr * LD + 8 * J + 2 * gc];
        c1[j] = Fb[gr * LD + 8 * J + 2 * gc + 1];
      } else if (J == kb) {  // (F_I)^T: element (r, p) = F[p][8I + r]
        c0[j] = Fb[(2 * gc) * LD + 8 * I + gr];
        c1[j] = Fb[(2 * gc + 1) * LD + 8 * I + gr];
      } else {  // C -= U_I F_J, U_I[r][p] = P[p][8I + r]; A = -U (row-major a[gr][gc + 4h]); B = F_J b[gc + 4h][gr]
        dmma(c0[j], c1[j], -P[gc * LD + 8 * I + gr], Fb[gc * LD + 8 * J + gr]);
        dmma(c0[j], c1[j], -P[(gc + 4) * LD + 8 * I + gr], Fb[(gc + 4) * LD + 8 * J + gr]);
      }
    }
    if (tid == 0) { double s = c0[0] + c1[0]; tacc[2] += clock64() - tu + (s == 12345.678 ? 1 : 0); }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 32 * 13) tacc[3] = 0;
  // W = -M on the first R rows / columns
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int t = w + kWarps * j;
    if (t >= NT) continue;
    const int I = t / NB, J = t % NB, r = 8 * I + gr, c = 8 * J + 2 * gc;
    if (r < R && c < R) W[r * R + c] = -c0[j];
    if (r < R && c + 1 < R) W[r * R + c + 1] = -c1[j];
  }
  if (tid == 0) {
    *status = s_fail;
    *cyc = t1 - t0;
    printf("per call: B sweep %lld, sweep+F+barrier %lld, updates (warp 0) %lld cycles\n", tacc[0], tacc[1], tacc[2]);
  }
}

int main() {
  const int R = 50, I = 2000;
  std::vector<double> A((size_t)I * R), G((size_t)R * R, 0.0);
  srand(1);
  auto nrm = [] {
    double u = (rand() + 1.0) / (RAND_MAX + 2.0), v = (rand() + 1.0) / (RAND_MAX + 2.0);
    return sqrt(-2 * log(u)) * cos(6.283185307179586 * v);
  };
  for (int i = 0; i < I; ++i) {
    const double s = exp(nrm());
    for (int r = 0; r < R; ++r) A[(size_t)i * R + r] = s * nrm();
  }
  for (int i = 0; i < I; ++i)
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) G[a * R + b] += A[(size_t)i * R + a] * A[(size_t)i * R + b];
  // host reference: Gauss-Jordan in long double
  std::vector<long double> M((size_t)R * 2 * R, 0.0L);
  for (int a = 0; a < R; ++a) {
    for (int b = 0; b < R; ++b) M[a * 2 * R + b] = G[a * R + b];
    M[a * 2 * R + R + a] = 1.0L;
  }
  for (int k = 0; k < R; ++k) {
    const long double d = M[k * 2 * R + k];
    for (int c = 0; c < 2 * R; ++c) M[k * 2 * R + c] /= d;
    for (int r = 0; r < R; ++r)
      if (r != k) {
        const long double f = M[r * 2 * R + k];
        for (int c = 0; c < 2 * R; ++c) M[r * 2 * R + c] -= f * M[k * 2 * R + c];
      }
  }
  double dmax = 0;
  for (int a = 0; a < R; ++a) dmax = fmax(dmax, G[a * R + a]);
  const double tol = I * 2.220446049250313e-16 * dmax;
  double *dG, *dW;
  int* dst;
  long long* dc;
  cudaMalloc(&dG, sizeof(double) * R * R);
  cudaMalloc(&dW, sizeof(double) * R * R);
  cudaMalloc(&dst, 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dG, G.data(), sizeof(double) * R * R, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 3; ++rep) kinv<56><<<1, kThreads>>>(dG, R, tol, dW, dst, dc);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> Wh((size_t)R * R);
  int st;
  long long cy;
  cudaMemcpy(Wh.data(), dW, sizeof(double) * R * R, cudaMemcpyDeviceToHost);
  cudaMemcpy(&st, dst, 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cy, dc, 8, cudaMemcpyDeviceToHost);
  double err = 0, ref = 0;
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < R; ++b) {
      const double x = (double)M[a * 2 * R + R + b];
      err = fmax(err, fabs(Wh[a * R + b] - x));
      ref = fmax(ref, fabs(x));
    }
  printf("%s status %d  max|W - W_ref| / max|W_ref| = %.3e  cycles %lld (%.2f us at 1.92 GHz)\n", cudaGetErrorString(e),
         st, err / ref, cy, cy / 1920.0);
  return 0;
}
