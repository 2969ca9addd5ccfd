// Look-ahead blocked sweep inverse on fp64 tensor cores (mma.sync m8n8k4 f64), one 448-thread CTA.
// Warp 0 (the pivot warp) owns the serial chain: sweep the 8x8 pivot block B_kb in registers (2x2 sub-pivots),
// publish -B^-1, then form the NEXT pivot block itself, B_kb+1 = D - Q^T B^-1 Q (Q = the published block row's
// next column block, D = the next diagonal tile as it was published), and sweep it -- while warps 1..13 (the
// owners of the upper-triangle 8x8 tiles) form F = B^-1 M_P,: and update their tiles (2 DMMA each), then publish
// the next block row.  Compared with a host Gauss-Jordan inverse; cycles per call.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_la dmma_la.cu && ./dmma_la
#include <cmath>
#include <cstdint>
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
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(su32(b)), "r"(par)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ void obar() { asm volatile("bar.sync 2, 416;" ::: "memory"); }  // the 13 owner warps

#ifndef SWEEP8
#define SWEEP8 sweep8
#endif
constexpr int kThreads = 448, kOwners = 13;

// sweep of the 8x8 block held as (b0, b1) = B[gr][2gc], B[gr][2gc+1]: 2x2 sub-pivots, select-free; returns false
// when a real pivot fails the single-pivot rule (a > tol, det > tol a)
__device__ __forceinline__ bool sweep8(double& b0, double& b1, int gr, int gc, int kbase, int R, double tol) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const int h = k >> 1;
    const double rk0 = __shfl_sync(0xffffffffu, b0, 4 * k + gc), rk1 = __shfl_sync(0xffffffffu, b1, 4 * k + gc);
    const double rl0 = __shfl_sync(0xffffffffu, b0, 4 * (k + 1) + gc), rl1 = __shfl_sync(0xffffffffu, b1, 4 * (k + 1) + gc);
    const double mk = __shfl_sync(0xffffffffu, b0, 4 * gr + h), ml = __shfl_sync(0xffffffffu, b1, 4 * gr + h);
    const double a = __shfl_sync(0xffffffffu, b0, 4 * k + h), bb = __shfl_sync(0xffffffffu, b1, 4 * k + h);
    const double cc = __shfl_sync(0xffffffffu, b1, 4 * (k + 1) + h);
    const double det = fma(a, cc, -bb * bb);
    if (kbase + k < R && !(a > tol && det > tol * a)) ok = false;
    const double dinv = rcp_nr(det);
    const double g1 = fma(cc, mk, -bb * ml) * dinv, g2 = fma(a, ml, -bb * mk) * dinv;
    const bool pr = (gr == k || gr == k + 1);
    const double adj0 = (gr == 2 * gc) ? ((2 * gc == k) ? cc : a) : -bb;
    const double adj1 = (gr == 2 * gc + 1) ? ((2 * gc + 1 == k) ? cc : a) : -bb;
    const double prow0 = (gr == k) ? fma(cc, rk0, -bb * rl0) * dinv : fma(a, rl0, -bb * rk0) * dinv;
    const double prow1 = (gr == k) ? fma(cc, rk1, -bb * rl1) * dinv : fma(a, rl1, -bb * rk1) * dinv;
    const double gen0 = fma(-g1, rk0, fma(-g2, rl0, b0)), gen1 = fma(-g1, rk1, fma(-g2, rl1, b1));
    const bool pc0 = (2 * gc == k || 2 * gc == k + 1), pc1 = (2 * gc + 1 == k || 2 * gc + 1 == k + 1);
    b0 = pc0 ? (pr ? -adj0 * dinv : (2 * gc == k ? g1 : g2)) : (pr ? prow0 : gen0);
    b1 = pc1 ? (pr ? -adj1 * dinv : (2 * gc + 1 == k ? g1 : g2)) : (pr ? prow1 : gen1);
  }
  return ok;
}

// one pivot per step (8 steps): lane (gr, gc) holds B[gr][2gc], B[gr][2gc+1]
__device__ __forceinline__ bool sweep8s(double& b0, double& b1, int gr, int gc, int kbase, int R, double tol) {
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double d = __shfl_sync(0xffffffffu, (k & 1) ? b1 : b0, 4 * k + (k >> 1));
    const double rk0 = __shfl_sync(0xffffffffu, b0, 4 * k + gc), rk1 = __shfl_sync(0xffffffffu, b1, 4 * k + gc);
    const double ck = __shfl_sync(0xffffffffu, (k & 1) ? b1 : b0, 4 * gr + (k >> 1));
    if (kbase + k < R && !(d > tol)) ok = false;
    const double dinv = rcp_nr(d);
    const double f = ck * dinv;
    const bool pr = (gr == k);
    const double n0 = pr ? rk0 * dinv : fma(-f, rk0, b0), n1 = pr ? rk1 * dinv : fma(-f, rk1, b1);
    b0 = (2 * gc == k) ? (pr ? -dinv : f) : n0;
    b1 = (2 * gc + 1 == k) ? (pr ? -dinv : f) : n1;
  }
  return ok;
}

template <int RMAX>
__global__ void __launch_bounds__(kThreads, 1) kinv(const double* G, int R, double tol, double* W, int* status,
                                                    long long* cyc) {
  constexpr int NB = RMAX / 8, NT = NB * (NB + 1) / 2, TPW = (NT + kOwners - 1) / kOwners, LD = RMAX + 2;
  __shared__ double Prow[NB][8 * LD];  // block row kb as published: [p][c]
  __shared__ double Dd[NB][64];        // diagonal tile kb + 1 as published with block row kb
  __shared__ double Sw[NB][64];        // -B_kb^-1
  __shared__ double Fb[8 * LD];        // F = B^-1 M_P,: of the current step
  __shared__ double scr[64];           // the pivot warp's scratch
  __shared__ __align__(8) uint64_t rows_b[NB], binv_b[NB];
  __shared__ int s_fail;
  __shared__ long long tacc[8];
  if (threadIdx.x < 8) tacc[threadIdx.x] = 0;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, gr = lane >> 2, gc = lane & 3;
  if (tid == 0) {
    s_fail = 0;
    for (int k = 0; k < NB; ++k) {
      mb_init(&rows_b[k], 32 * kOwners);
      mb_init(&binv_b[k], 32);
    }
  }
  // owner tiles: upper-triangle tile t (row-major over I <= J) -> warp 1 + t % 13, slot t / 13
  int tI[TPW], tJ[TPW];
  double c0[TPW], c1[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int t = (w - 1) + kOwners * j;
    int I = 0, rem = t;
    while (I < NB && rem >= NB - I) { rem -= NB - I; ++I; }
    tI[j] = (w >= 1 && t < NT) ? I : -1;
    tJ[j] = I + rem;
    const int r = 8 * I + gr, c = 8 * tJ[j] + 2 * gc;
    auto at = [&](int rr, int cc) { return rr < R && cc < R ? G[rr * R + cc] : (rr == cc ? 1.0 : 0.0); };
    c0[j] = tI[j] >= 0 ? at(r, c) : 0.0;
    c1[j] = tI[j] >= 0 ? at(r, c + 1) : 0.0;
  }
  __syncthreads();
  long long t0 = clock64();
  if (w == 0) {  // ---------------- the pivot warp
    mb_wait(&rows_b[0], 0);
    double b0 = Prow[0][gr * LD + 2 * gc], b1 = Prow[0][gr * LD + 2 * gc + 1];
#pragma unroll 1
    for (int kb = 0; kb < NB; ++kb) {
      long long ts0 = clock64();
      const bool ok = SWEEP8(b0, b1, gr, gc, 8 * kb, R, tol);
      if (lane == 0) tacc[0] += clock64() - ts0;
      if (!ok && lane == 0) s_fail = 1;
      Sw[kb][gr * 8 + 2 * gc] = b0;
      Sw[kb][gr * 8 + 2 * gc + 1] = b1;
      mb_arrive(&binv_b[kb]);
      if (!ok || kb + 1 == NB) break;
      // B_kb+1 = D - Q^T B^-1 Q, Q = Prow[kb][:, block kb+1]; the same DMMA sequence the owners apply to that tile
      long long tw0 = clock64();
      mb_wait(&rows_b[kb], 0);
      if (lane == 0) tacc[1] += clock64() - tw0;
      long long tsch = clock64();
      const double* P = Prow[kb];
      const int J = kb + 1;
      const double a_lo = -Sw[kb][gr * 8 + gc], a_hi = -Sw[kb][gr * 8 + gc + 4];
      double f0 = 0.0, f1 = 0.0;
      dmma(f0, f1, a_lo, P[gc * LD + 8 * J + gr]);
      dmma(f0, f1, a_hi, P[(gc + 4) * LD + 8 * J + gr]);
      scr[gr * 8 + 2 * gc] = f0;
      scr[gr * 8 + 2 * gc + 1] = f1;
      __syncwarp();
      double d0 = Dd[kb + 1][gr * 8 + 2 * gc], d1 = Dd[kb + 1][gr * 8 + 2 * gc + 1];
      dmma(d0, d1, -P[gc * LD + 8 * J + gr], scr[gc * 8 + gr]);
      dmma(d0, d1, -P[(gc + 4) * LD + 8 * J + gr], scr[(gc + 4) * 8 + gr]);
      __syncwarp();
      b0 = d0;
      b1 = d1;
      if (lane == 0) tacc[2] += clock64() - tsch;
    }
  } else {  // ---------------- the owners
#pragma unroll 1
    for (int kb = 0; kb < NB; ++kb) {
      double* P = Prow[kb];
      // publish block row kb (tiles (kb, J >= kb) as they are; tiles (I < kb, kb) transposed) and tile (kb+1, kb+1)
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int I = tI[j], J = tJ[j];
        if (I < 0) continue;
        if (I == kb) {
          P[gr * LD + 8 * J + 2 * gc] = c0[j];
          P[gr * LD + 8 * J + 2 * gc + 1] = c1[j];
        } else if (J == kb) {
          P[(2 * gc) * LD + 8 * I + gr] = c0[j];
          P[(2 * gc + 1) * LD + 8 * I + gr] = c1[j];
        }
        if (I == kb + 1 && J == kb + 1) {
          Dd[kb + 1][gr * 8 + 2 * gc] = c0[j];
          Dd[kb + 1][gr * 8 + 2 * gc + 1] = c1[j];
        }
      }
      long long q0 = clock64();
      mb_arrive(&rows_b[kb]);
      mb_wait(&rows_b[kb], 0);
      long long q1 = clock64();
      mb_wait(&binv_b[kb], 0);
      long long q2 = clock64();
      if (tid == 32) { tacc[3] += q1 - q0; tacc[4] += q2 - q1; }
      if (s_fail) break;
      if (w <= NB) {  // F_J = B^-1 P[:, block J], J = w - 1
        const int J = w - 1;
        const double a_lo = -Sw[kb][gr * 8 + gc], a_hi = -Sw[kb][gr * 8 + gc + 4];
        double f0 = 0.0, f1 = 0.0;
        dmma(f0, f1, a_lo, P[gc * LD + 8 * J + gr]);
        dmma(f0, f1, a_hi, P[(gc + 4) * LD + 8 * J + gr]);
        Fb[gr * LD + 8 * J + 2 * gc] = f0;
        Fb[gr * LD + 8 * J + 2 * gc + 1] = f1;
      }
      obar();
      long long q3 = clock64();
      if (tid == 32) tacc[5] += q3 - q2;
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int I = tI[j], J = tJ[j];
        if (I < 0) continue;
        if (I == kb && J == kb) {
          c0[j] = Sw[kb][gr * 8 + 2 * gc];
          c1[j] = Sw[kb][gr * 8 + 2 * gc + 1];
        } else if (I == kb) {
          c0[j] = Fb[gr * LD + 8 * J + 2 * gc];
          c1[j] = Fb[gr * LD + 8 * J + 2 * gc + 1];
        } else if (J == kb) {  // (F_I)^T
          c0[j] = Fb[(2 * gc) * LD + 8 * I + gr];
          c1[j] = Fb[(2 * gc + 1) * LD + 8 * I + gr];
        } else {
          dmma(c0[j], c1[j], -P[gc * LD + 8 * I + gr], Fb[gc * LD + 8 * J + gr]);
          dmma(c0[j], c1[j], -P[(gc + 4) * LD + 8 * I + gr], Fb[(gc + 4) * LD + 8 * J + gr]);
        }
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int I = tI[j], J = tJ[j];
    if (I < 0) continue;
    const int r = 8 * I + gr, c = 8 * J + 2 * gc;
    if (r < R && c < R) { W[r * R + c] = -c0[j]; W[c * R + r] = -c0[j]; }
    if (r < R && c + 1 < R) { W[r * R + c + 1] = -c1[j]; W[(c + 1) * R + r] = -c1[j]; }
  }
  if (tid == 0) {
    *status = s_fail;
    *cyc = t1 - t0;
    printf("pivot warp: sweeps %lld, waits for rows %lld, Schur %lld cycles; owner warp 1: rows barrier %lld, binv wait %lld, F+obar %lld\n", tacc[0], tacc[1], tacc[2], tacc[3], tacc[4], tacc[5]);
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
