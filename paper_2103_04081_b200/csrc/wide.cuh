// wide.cuh -- the single-GPU wide path after the gather kernel (k_gather_update[_tc]), one step =
//
//   k_gather_update[_tc]  (a4-a6)  chunk partials of M = X_F diag(w) Z_F            (all SMs)
//   k_update_wide         (a6-a8)  M = sum_c M_c (chunk order), G = A Gamma - M, fixed / adaptive
//                                  update; partial fp64 Grams (leverage) or row norms (Euclidean)
//                                  of the new rows -> the table kernel               (all SMs)
//   k_table_wide          (a1)     Gram -> symmetric-sweep inverse -> leverage scores, or the
//                                  Euclidean ratios; fixed-point quantisation; integer scan -> CDF
//                                  (one cluster: the R-pivot chain is inherently serial)
//   k_sample_wide         (a2-a4)  the next batch: draws, SKR rows, weighted rows / tcgen05 images,
//                                  Gamma = Z_F^T diag(w) Z_F (clusters of 8, last cluster sums)  (all SMs)
//
// Citations: PAPER.md:<lines> (<label>); R<k> = DESIGN.md readings.
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cps {

constexpr int kUWRows = 16;     // rows of A^(n) per k_update_wide CTA (divides the 128-row tiles)
constexpr int kWThreads = 256;
constexpr int kTWThreads = 256;  // k_table_wide (512 would cap registers at 128 and spill the sweep)
constexpr int kSWFibers = 32;   // fibers per k_sample_wide CTA
constexpr int kSWCluster = 8;
constexpr int kUWCluster = 8;   // k_update_wide CTAs per cluster (table partials summed over DSMEM)

template <typename T>
struct UWParams {
  int R, strategy, rule;
  int64_t In;
  const T* Mpart;     // [tiles][CK][R][128]
  int CK;
  const T* Gam;       // [R][R]
  T* A;               // A^(n), updated in place
  T* S;               // adaptive accumulator or NULL
  T* Gout;
  T* Gam_out;
  double alpha;
  const double* alpha_dev;
  double eta, b, eps;
  double* gpart;      // [clusters][R(R+1)/2] (leverage) or [clusters] (Euclidean)
  double* rownorm;    // [I_n] (Euclidean)
};

// (a6-a8) + the parallel half of (a1): grid = ceil(I_n / kUWRows); dynamic shared memory
__host__ __device__ inline size_t uw_smem_bytes(int R, size_t esz) {
  return (esz * (3 * (size_t)kUWRows * (R + 1) + (size_t)R * R) + 15) / 16 * 16 +
         sizeof(double) * (size_t)(R * (R + 1) / 2) + 16;
}
template <typename T>
__global__ void __launch_bounds__(kWThreads) k_update_wide(UWParams<T> p) {
  constexpr int UR = kUWRows, TI = 128;
  const int R = p.R, RS = R + 1, tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * UR;
  const int nr = (int)cmax64(0, cmin64(UR, p.In - r0));  // 0 for the CTAs rounding the grid up
  extern __shared__ __align__(16) unsigned char uw_sm[];
  T* sA = reinterpret_cast<T*>(uw_sm);  // [UR][R+1] each
  T* sS = sA + UR * RS;
  T* sM = sS + UR * RS;
  T* sG = sM + UR * RS;                 // [R][R]
  double* sgp = reinterpret_cast<double*>(uw_sm + ((sizeof(T) * (3 * UR * RS + R * R) + 15) / 16) * 16);  // [P]
  __shared__ double sred[kWThreads / 32];
  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  // rows of A and S, Gamma: every request in flight at once
  for (int e = tid; e < nr * R; e += kWThreads) {
    const int il = e / R, c = e % R;
    cp_async_small<sizeof(T)>(sA + il * RS + c, p.A + (r0 + il) * R + c, sizeof(T));
    if (p.rule != 0) cp_async_small<sizeof(T)>(sS + il * RS + c, p.S + (r0 + il) * R + c, sizeof(T));
  }
  for (int e = tid; e < R * R; e += kWThreads) cp_async_small<sizeof(T)>(sG + e, p.Gam + e, sizeof(T));
  cp_async_commit();
  // M = sum of the chunk partials, in chunk order (16-byte vectors of VW consecutive rows)
  {
    constexpr int VW = 16 / (int)sizeof(T);
    using V = typename Vec<T>::type;
    const int64_t tile = r0 / TI, lr0 = r0 % TI;
    const int ng = (nr + VW - 1) / VW;
    for (int t = tid; t < R * ng; t += kWThreads) {
      const int r = t / ng, gq = t % ng;
      const T* base = p.Mpart + ((tile * p.CK) * R + r) * TI + lr0 + gq * VW;
      T acc[VW];
#pragma unroll
      for (int w = 0; w < VW; ++w) acc[w] = T(0);
      for (int c0 = 0; c0 < p.CK; c0 += 8) {
        V ld[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (c0 + k < p.CK) ld[k] = __ldcg(reinterpret_cast<const V*>(base + (int64_t)(c0 + k) * R * TI));
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (c0 + k < p.CK) {
            const T* x = reinterpret_cast<const T*>(&ld[k]);
#pragma unroll
            for (int w = 0; w < VW; ++w) acc[w] += x[w];
          }
      }
#pragma unroll
      for (int w = 0; w < VW; ++w)
        if (gq * VW + w < nr) sM[(gq * VW + w) * RS + r] = acc[w];
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // G = A Gamma - M (each task owns its 4 x 4 block of M -> G in place)
  const int nb4 = (R + 3) >> 2;
  for (int t = tid; t < ((nr + 3) >> 2) * nb4; t += kWThreads) {
    const int a0 = 4 * (t / nb4), q0 = 4 * (t % nb4);
    T acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][c] = T(0);
    for (int k = 0; k < R; ++k) {
      T x[4], y[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) x[a] = (a0 + a < nr) ? sA[(a0 + a) * RS + k] : T(0);
#pragma unroll
      for (int c = 0; c < 4; ++c) y[c] = (q0 + c < R) ? sG[k * R + q0 + c] : T(0);
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = fma(x[a], y[c], acc[a][c]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (a0 + a < nr && q0 + c < R) sM[(a0 + a) * RS + q0 + c] = acc[a][c] - sM[(a0 + a) * RS + q0 + c];
  }
  __syncthreads();
  // fixed (eq:proposed) / adaptive (eq:etaada/eq:Aada, :531-537, R12) update
  const double alpha = p.alpha_dev ? *p.alpha_dev : p.alpha;
  for (int e = tid; e < nr * R; e += kWThreads) {
    const int il = e / R, r = e % R;
    const int64_t gi = (r0 + il) * R + r;
    const T g = sM[il * RS + r];
    p.Gout[gi] = g;
    const T a = sA[il * RS + r];
    T an = a;
    if (p.rule == 0) {
      an = a - (T)alpha * g;
    } else {
      const T sv = sS[il * RS + r] + g * g;
      p.S[gi] = sv;
      if (sv > T(0)) {
        T step;
        if (p.eps == 0.0) step = (T)p.eta / sqrt((T)p.b + sv);
        else step = (T)p.eta / (T)pow((double)((T)p.b + sv), 0.5 + p.eps);
        an = a - step * g;
      }
    }
    p.A[gi] = an;
    sA[il * RS + r] = an;
  }
  if (blockIdx.x == 0)
    for (int e = tid; e < R * R; e += kWThreads) p.Gam_out[e] = sG[e];
  __syncthreads();
  // table partials of the new rows (R9: the table of A^(n) is rebuilt after every update)
  if (p.strategy == 1 || p.strategy == 3) {  // leverage: partial fp64 Gram, packed upper triangle
    const int P = R * (R + 1) / 2;
    const int nblk = nb4 * (nb4 + 1) / 2;  // thread = 4 x 4 block (bi <= bj)
    for (int blk = tid; blk < nblk; blk += kWThreads) {
      int bi = 0, rem = blk;
      while (rem >= nb4 - bi) { rem -= nb4 - bi; ++bi; }
      const int bj = bi + rem;
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
      for (int il = 0; il < nr; ++il) {
        double x[4], y[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          x[a] = 4 * bi + a < R ? (double)sA[il * RS + 4 * bi + a] : 0.0;
          y[a] = 4 * bj + a < R ? (double)sA[il * RS + 4 * bj + a] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fma(x[a], y[c], acc[a][c]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int r1 = 4 * bi + a, r2 = 4 * bj + c;
          if (r1 < R && r2 < R && r1 <= r2)
            sgp[r1 * R - r1 * (r1 - 1) / 2 + (r2 - r1)] = acc[a][c];
        }
    }
    // cluster sum (rank order) of the CTA partials -> one partial per cluster of kUWCluster CTAs
    cluster.sync();
    const int CU = (int)cluster.num_blocks(), q = (int)cluster.block_rank();
    const int per = (P + CU - 1) / CU;
    for (int pair = q * per + tid; pair < min(P, (q + 1) * per); pair += kWThreads) {
      double v[kUWCluster], s = 0.0;
#pragma unroll
      for (int qq = 0; qq < kUWCluster; ++qq) v[qq] = qq < CU ? cluster.map_shared_rank(sgp, qq)[pair] : 0.0;
#pragma unroll
      for (int qq = 0; qq < kUWCluster; ++qq) s += v[qq];
      p.gpart[(int64_t)(blockIdx.x / CU) * P + pair] = s;
    }
    cluster.sync();
  } else if (p.strategy == 2 || p.strategy == 4) {  // Euclidean: row norms + the CTA's partial ||A||^2
    double acc = 0.0;
    for (int il = tid; il < nr; il += kWThreads) {
      double rs = 0.0;
      for (int c = 0; c < R; ++c) rs += (double)sA[il * RS + c] * (double)sA[il * RS + c];
      p.rownorm[r0 + il] = rs;
      acc += rs;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) sred[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kWThreads / 32; ++w) t += sred[w];
      sgp[0] = t;
    }
    cluster.sync();
    if (cluster.block_rank() == 0 && tid == 0) {
      double t = 0.0;
      for (int qq = 0; qq < (int)cluster.num_blocks(); ++qq) t += cluster.map_shared_rank(sgp, qq)[0];
      p.gpart[blockIdx.x / cluster.num_blocks()] = t;
    }
    cluster.sync();
  }
}

// ------------------------------------------------------------------------------------------
// (a1) the table of the updated A^(n): one cluster of CU CTAs (CTA q owns rows [q rows_per, ...))
// ------------------------------------------------------------------------------------------
struct TWParams {
  int R, strategy;
  int64_t In, rows_per;
  int nparts;               // k_update_wide CTAs
  const double* gpart;      // their partials
  const double* rownorm;    // Euclidean row norms (k_update_wide)
  const void* A;            // A^(n) (updated), T = float or double
  int esz;
  double* p_out;
  uint64_t* cdf;
  uint64_t* Tout;
  int* status;
  long long* dbg;
};

__host__ __device__ inline size_t tw_smem_bytes(int R, int64_t rows_per) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = (off + 15) / 16 * 16;
    off += bytes;
  };
  const int RD = ut_rd(R), P = R * (R + 1) / 2;
  take(sizeof(double) * rows_per * RD);      // Ad
  const size_t wk = ut_work_bytes(R, rows_per), st = sizeof(double) * rows_per * R;
  take(wk > st ? wk : st);                   // W + score partials | staged rows of A
  take(sizeof(double) * P);                  // this CTA's slice sums (read by peers)
  take(sizeof(double) * R * (R + 1));        // Gm
  take(sizeof(double) * 4 * kMaxRank);       // sweep buffers
  take(sizeof(int) * kMaxRank);              // swept
  take(sizeof(double) * rows_per);           // prow
  take(sizeof(unsigned long long) * rows_per);
  take(sizeof(unsigned long long) * 2);
  return off + 16;
}

template <typename T>
__device__ void table_wide_body(const TWParams& p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int CU = (int)cluster.num_blocks(), q = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int R = p.R, RD = ut_rd(R), nb4 = (R + 3) >> 2, P = R * (R + 1) / 2, RS = R + 1;
  const int64_t r_beg = cmin64((int64_t)q * p.rows_per, p.In), r_end = cmin64(r_beg + p.rows_per, p.In);
  const int nr = (int)(r_end - r_beg);
  extern __shared__ __align__(16) unsigned char tw_sm[];
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    off = (off + 15) / 16 * 16;
    unsigned char* ptr = tw_sm + off;
    off += bytes;
    return ptr;
  };
  double* Ad = reinterpret_cast<double*>(carve(sizeof(double) * p.rows_per * RD));
  double* work = reinterpret_cast<double*>(
      carve(ut_work_bytes(R, p.rows_per) > sizeof(double) * p.rows_per * R ? ut_work_bytes(R, p.rows_per)
                                                                             : sizeof(double) * p.rows_per * R));
  double* slice = reinterpret_cast<double*>(carve(sizeof(double) * P));
  double* Gm = reinterpret_cast<double*>(carve(sizeof(double) * R * (R + 1)));
  double* colbuf = reinterpret_cast<double*>(carve(sizeof(double) * 4 * kMaxRank));
  int* swept = reinterpret_cast<int*>(carve(sizeof(int) * kMaxRank));
  double* prow = reinterpret_cast<double*>(carve(sizeof(double) * p.rows_per));
  unsigned long long* qrow = reinterpret_cast<unsigned long long*>(carve(sizeof(unsigned long long) * p.rows_per));
  unsigned long long* qtot = reinterpret_cast<unsigned long long*>(carve(sizeof(unsigned long long) * 2));
  __shared__ int s_bad;
  __shared__ double s_red[kTWThreads / 32];
  __shared__ unsigned long long s_wtot[kTWThreads / 32];
  __shared__ double s_tol, s_fro;
  if (tid == 0) s_bad = 0;
  const bool lev = (p.strategy == 1 || p.strategy == 3);
  const T* A = reinterpret_cast<const T*>(p.A);
  if (p.dbg && q == 0 && tid == 0) p.dbg[0] = clock64();
  if (lev) {
    // rows of the new A^(n) for the scores: cp.async into the work area (all requests in flight,
    // overlapped with the slice sums), then fp64 (zero padded to RD)
    T* Ast = reinterpret_cast<T*>(work);
    for (int e = tid; e < nr * R; e += kTWThreads) cp_async_small<sizeof(T)>(Ast + e, A + r_beg * R + e, sizeof(T));
    cp_async_commit();
    // pair slice of this CTA: sum of the k_update_wide partials in CTA order
    const int per = (P + CU - 1) / CU, pb = q * per, pe = min(P, pb + per);
    for (int pair = pb + tid; pair < pe; pair += kTWThreads) {
      double v[8], s = 0.0;
      for (int c0 = 0; c0 < p.nparts; c0 += 8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = (c0 + k < p.nparts) ? __ldcg(p.gpart + (int64_t)(c0 + k) * P + pair) : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) s += v[k];  // zeros past nparts are exact
      }
      slice[pair - pb] = s;
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int e = tid; e < nr * RD; e += kTWThreads) {
      const int il = e / RD, c = e % RD;
      Ad[e] = c < R ? (double)Ast[il * R + c] : 0.0;
    }
    cluster.sync();  // #1 slices visible (and Ad complete; the work area is free again)
    for (int pair = tid; pair < P; pair += kTWThreads) {
      const int owner = pair / per;
      const double sum = cluster.map_shared_rank(slice, owner)[pair - owner * per];
      int r1 = 0, rem = pair;
      while (rem >= R - r1) { rem -= R - r1; ++r1; }
      const int r2 = r1 + rem;
      Gm[r1 * RS + r2] = sum;
      Gm[r2 * RS + r1] = sum;
    }
    __syncthreads();
    if (wid == 0) {
      double d0 = 0.0;
      bool fin = true;
      for (int j = lane; j < R; j += 32) {
        const double d = Gm[j * RS + j];
        d0 = fmax(d0, d);
        fin = fin && (d == d) && d < 1.7e308;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
      if (!__all_sync(0xffffffffu, fin) && lane == 0) s_bad |= 8;
      if (lane == 0) s_tol = (double)(p.In > R ? p.In : R) * 2.220446049250313e-16 * d0;
    }
    __syncthreads();
    if (p.dbg && q == 0 && tid == 0) p.dbg[1] = clock64();
    constexpr int EPT = (kMaxRank * kMaxRank + kTWThreads - 1) / kTWThreads;
    const int rank = (p.In < 2 * R) ? cta_sweep_inverse_pivoted<EPT>(Gm, R, s_tol, colbuf, swept, colbuf + R)
                                    : grp_sweep_dispatch(Gm, R, s_tol, colbuf, swept);
    if (tid == 0 && rank == 0) s_bad |= 2;
    if (p.dbg && q == 0 && tid == 0) p.dbg[2] = clock64();
    // scores l_i = sum_c (A W)_ic a_ic (4 rows x 4 columns per task; k in pairs)
    double* Wd = work;
    double* sc = work + R * RD;  // [nb4][rows_per]
    for (int e = tid; e < R * RD; e += kTWThreads) {
      const int r1 = e / RD, c = e % RD;
      Wd[e] = c < R ? Gm[r1 * RS + c] : 0.0;
    }
    __syncthreads();
    const int nrg = (nr + 3) >> 2, ntask = nrg * nb4;
    for (int t = tid; t < ntask; t += kTWThreads) {
      const int rg = t / nb4, cg2 = t % nb4;
      const int il0 = 4 * rg;
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
      const double* arow[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) arow[a] = Ad + (il0 + a < nr ? il0 + a : il0) * RD;
      for (int kk = 0; kk < R; kk += 2) {
        double2 av[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = *reinterpret_cast<const double2*>(arow[a] + kk);
        const int k1 = kk + 1 < R ? kk + 1 : kk;
        const double2 w00 = *reinterpret_cast<const double2*>(Wd + kk * RD + 4 * cg2);
        const double2 w01 = *reinterpret_cast<const double2*>(Wd + kk * RD + 4 * cg2 + 2);
        const double2 w10 = *reinterpret_cast<const double2*>(Wd + k1 * RD + 4 * cg2);
        const double2 w11 = *reinterpret_cast<const double2*>(Wd + k1 * RD + 4 * cg2 + 2);
        const double wk0[4] = {w00.x, w00.y, w01.x, w01.y};
        const double wk1[4] = {w10.x, w10.y, w11.x, w11.y};
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fma(av[a].y, wk1[c], fma(av[a].x, wk0[c], acc[a][c]));
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        if (il0 + a >= nr) continue;
        const double2 x0 = *reinterpret_cast<const double2*>(arow[a] + 4 * cg2);
        const double2 x1 = *reinterpret_cast<const double2*>(arow[a] + 4 * cg2 + 2);
        sc[cg2 * p.rows_per + il0 + a] = acc[a][0] * x0.x + acc[a][1] * x0.y + acc[a][2] * x1.x + acc[a][3] * x1.y;
      }
    }
    __syncthreads();
    for (int il = tid; il < nr; il += kTWThreads) {
      double l = 0.0;
      for (int cg2 = 0; cg2 < nb4; ++cg2) l += sc[cg2 * p.rows_per + il];
      prow[il] = rank > 0 ? fmax(l, 0.0) / (double)rank : 0.0;
    }
  } else {
    if (tid == 0) {
      double fro = 0.0;
      for (int c = 0; c < p.nparts; ++c) fro += __ldcg(p.gpart + c);
      s_fro = fro;
      if (!(fro == fro) || fro > 1.7e308) s_bad |= 8;
      else if (!(fro > 0.0)) s_bad |= 2;
    }
    __syncthreads();
    const double fro = s_fro;
    for (int il = tid; il < nr; il += kTWThreads) prow[il] = fro > 0.0 ? __ldcg(p.rownorm + r_beg + il) / fro : 0.0;
    cluster.sync();  // #1 (matches the leverage branch)
  }
  __syncthreads();
  if (p.dbg && q == 0 && tid == 0) p.dbg[3] = clock64();
  // quantise + CTA scan (contiguous segment per thread) + DSMEM prefix of the lower ranks
  const int seg = (nr + kTWThreads - 1) / kTWThreads;
  const int a0 = min(tid * seg, nr), a1 = min(a0 + seg, nr);
  unsigned long long local = 0;
  int bad = 0;
  for (int il = a0; il < a1; ++il) {
    const double pv = prow[il];
    unsigned long long qv = 0;
    if (!(pv == pv) || pv > 2.0) {
      bad = 1;
    } else if (pv > 0.0) {
      const double s = rint(pv * 4294967296.0);
      qv = (s < 1.0) ? 1ull : (unsigned long long)s;
    }
    p.p_out[r_beg + il] = pv;
    local += qv;
    qrow[il] = local;
  }
  if (bad) atomicOr(&s_bad, 8);
  unsigned long long incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_wtot[wid] = incl;
  __syncthreads();
  unsigned long long wpre = 0;
  for (int w = 0; w < wid; ++w) wpre += s_wtot[w];
  const unsigned long long seg_pre = wpre + incl - local;
  if (tid == kTWThreads - 1) qtot[0] = seg_pre + local;
  cluster.sync();  // #2 CTA totals visible
  unsigned long long cta_pre = 0, total = 0;
  for (int qq = 0; qq < CU; ++qq) {
    const unsigned long long t = cluster.map_shared_rank(qtot, qq)[0];
    if (qq < q) cta_pre += t;
    total += t;
  }
  for (int il = a0; il < a1; ++il) p.cdf[r_beg + il] = cta_pre + seg_pre + qrow[il];
  if (tid == 0) {
    if (q == 0) *p.Tout = total;
    int st = 0;
    if (s_bad & 8) st = -8;
    else if ((s_bad & 2) || (q == 0 && total == 0)) st = -3;
    if (st != 0) atomicCAS(p.status, 0, st);
  }
  cluster.sync();  // #3 peers done with this CTA's shared memory
  if (p.dbg && q == 0 && tid == 0) p.dbg[4] = clock64();
}

template <typename T>
__global__ void __launch_bounds__(kTWThreads, 1) k_table_wide(TWParams p) {
  table_wide_body<T>(p);
}

// ------------------------------------------------------------------------------------------
// (a2-a4) the next batch: clusters of kSWCluster CTAs of kSWFibers fibers each
// ------------------------------------------------------------------------------------------
struct SWParams {
  long long* dbg;
  SampleParams sp;          // batch of mode sp.n at the iteration in *sp.iter; zwp / gam_next set
  void* gcl;                // [clusters][R][R] cluster partials of Gamma (T)
  unsigned* cnt;            // arrival counter (zero between launches)
  int64_t cdf_elems;        // staged CDF entries (sum of I_k, k != n; 0 = uniform)
};

__host__ __device__ inline size_t sw_smem_bytes(int N, int R, int64_t cdf_elems, size_t esz) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = (off + 15) / 16 * 16;
    off += bytes;
  };
  take(sizeof(uint64_t) * cdf_elems);
  take(sizeof(int32_t) * kSWFibers * (N - 1));
  take(sizeof(double) * kSWFibers);
  take(esz * kSWFibers * zg_rp(R));
  take(esz * (size_t)zg_groups(R, kWThreads) * R * R);
  return off + 16;
}

#define SWM(slot)                                                                           \
  do {                                                                                      \
    if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0) P.dbg[100 + (slot)] = clock64();     \
  } while (0)
template <typename T>
__global__ void __launch_bounds__(kWThreads) k_sample_wide(SWParams P) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const SampleParams& sp = P.sp;
  const int tid = threadIdx.x;
  const int N = sp.N, NP = N - 1, R = sp.R, RP = zg_rp(R), nb4 = (R + 3) >> 2;
  extern __shared__ __align__(16) unsigned char sw_sm[];
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    off = (off + 15) / 16 * 16;
    unsigned char* ptr = sw_sm + off;
    off += bytes;
    return ptr;
  };
  uint64_t* cdfs = reinterpret_cast<uint64_t*>(carve(sizeof(uint64_t) * P.cdf_elems));
  int32_t* sidx = reinterpret_cast<int32_t*>(carve(sizeof(int32_t) * kSWFibers * NP));
  double* sw = reinterpret_cast<double*>(carve(sizeof(double) * kSWFibers));
  T* zs = reinterpret_cast<T*>(carve(sizeof(T) * kSWFibers * RP));
  T* red = reinterpret_cast<T*>(carve(sizeof(T) * (size_t)zg_groups(R, kWThreads) * R * R));
  __shared__ const uint64_t* s_cp[kMaxOrder];
  __shared__ int s_last;
  SWM(0);
  long long gt0 = 0;
  if (P.dbg && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
  {
    int64_t o = 0;
    for (int k = 0; k < N; ++k) {
      const uint64_t* src = sp.cdf[k];
      if (k != sp.n && sp.strategy != 0) {
        cp_async_u64(cdfs + o, src, sp.dims[k], tid, kWThreads);
        src = cdfs + o;
        o += sp.dims[k];
      }
      if (tid == 0) s_cp[k] = src;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  const uint64_t r_now = *sp.iter;  SWM(1);

  const int64_t b0 = cmin64((int64_t)blockIdx.x * kSWFibers, sp.bmax), b1 = cmin64(b0 + kSWFibers, sp.bmax);
  const int nf = (int)(b1 - b0);
  if (sp.strategy == 3 || sp.strategy == 4) {
    draw_rows(sp, s_cp, r_now, b0, b1, tid, kWThreads, sidx, sw);
  } else {
    // row-wise draws (eq:ik, R8): one thread per (fiber, position) -- the N-1 draws of a fiber run
    // in parallel -- then per fiber the exact weight (DESIGN.md section 4 order) and the offset
    double* spt = reinterpret_cast<double*>(zs);  // [kSWFibers][N-1] realised probabilities (scratch)
    for (int e = tid; e < nf * NP; e += kWThreads) {
      const int lb = e / NP, pos = e % NP;
      const int k = pos < sp.n ? pos : pos + 1;
      const uint64_t Tk = sp.strategy == 0 ? (uint64_t)sp.dims[k] : sp.Ttot[k];
      const uint64_t rr = scale_draw(draw_word(sp.seed, r_now, (uint32_t)(b0 + lb), kPurposeRow, (uint32_t)pos), Tk);
      int64_t i;
      uint64_t qk;
      if (sp.strategy == 0) {
        i = (int64_t)rr;
        qk = 1;
      } else {
        const uint64_t* c = s_cp[k];
        i = upper_bound_u64(c, sp.dims[k], rr);
        qk = c[i] - (i > 0 ? c[i - 1] : 0ull);
      }
      sidx[e] = (int32_t)i;
      spt[e] = __ddiv_rn((double)((uint64_t)sp.dims[k] * qk), (double)Tk);
    }
    __syncthreads();
    if (b0 == 0 && tid == 0) *sp.beff = sp.B;
    for (int lb = tid; lb < nf; lb += kWThreads) {
      const int64_t b = b0 + lb;
      double prod = spt[lb * NP];
      for (int pos = 1; pos < NP; ++pos) prod = __dmul_rn(prod, spt[lb * NP + pos]);
      const double wv = __ddiv_rn(1.0, __dmul_rn((double)sp.B, prod));
      sw[lb] = wv;
      sp.w[b] = wv;
      int64_t offn = 0, jrow = 0, jmul = 1;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == sp.n) continue;
        const int64_t ik = sidx[lb * NP + pos];
        sp.idx[b * NP + pos] = (int32_t)ik;
        ++pos;
        offn += ik * sp.lstride[k];
        jrow += ik * jmul;
        jmul *= sp.ldims[k];
      }
      sp.fbase[b] = sp.mode_major ? jrow * sp.pitch : offn;
    }
  }
  __syncthreads();
  SWM(2);
  // SKR rows (Alg. 1): z[lb][r] = prod_{k != n, ascending} A^(k)(i_k, r); every
  // factor load of a thread's elements is issued before the products (one round trip per mode)
  {
    constexpr int U = (kSWFibers * 64 + kWThreads - 1) / kWThreads;  // >= elements per thread
    int lbu[U], ru[U];
    T z[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = tid + u * kWThreads;
      lbu[u] = e / RP;
      ru[u] = e % RP;
      z[u] = (e < kSWFibers * RP && lbu[u] < nf && ru[u] < R) ? T(1) : T(0);
    }
    int pos = 0;
    for (int k = 0; k < N; ++k) {  // ascending modes (Alg. 1)
      if (k == sp.n) continue;
      const T* F = reinterpret_cast<const T*>(sp.factors[k]);
      T f[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        f[u] = z[u] != T(0) ? F[(int64_t)sidx[lbu[u] * NP + pos] * R + ru[u]] : T(0);
#pragma unroll
      for (int u = 0; u < U; ++u) z[u] = z[u] * f[u];
      ++pos;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (tid + u * kWThreads < kSWFibers * RP) zs[tid + u * kWThreads] = z[u];
  }
  __syncthreads();
  SWM(3);
  // weighted rows zw_b = w_b z_b for the gather kernels (row-contiguous, zero past R) and the
  // tcgen05 A-operand images (zh / zl rows of 128 B over the 32 fibers: lanes run over fibers)
  {
    T* zwp = reinterpret_cast<T*>(sp.zwp);
    for (int e = tid; e < nf * RP; e += kWThreads) {
      const int lb = e / RP, r = e % RP;
      zwp[(b0 + lb) * RP + r] = (T)sw[lb] * zs[e];
    }
    if constexpr (sizeof(T) == 4) {
      if (sp.zimg)
        for (int e = tid; e < R * kSWFibers; e += kWThreads) {
          const int r = e / kSWFibers, lb = e % kSWFibers;
          if (lb < nf) {
            const float zw = (float)((T)sw[lb] * zs[lb * RP + r]);
            const float h = __uint_as_float(__float_as_uint(zw) & 0xFFFFE000u);
            sp.zimg[zimg_off(b0 + lb, r) >> 2] = h;
            sp.zimg[zimg_off(b0 + lb, 64 + r) >> 2] = zw - h;
          }
        }
    }
  }
  SWM(4);
  // Gamma_q = sum_b zw_b z_b^T over this CTA's fibers (4x4 blocks bi <= bj, G fiber groups)
  {
    const int nblk = nb4 * (nb4 + 1) / 2, G = zg_groups(R, kWThreads);
    const int g = tid / nblk, blk = tid % nblk;
    if (g < G) {
      int bi = 0, rem = blk;
      while (rem >= nb4 - bi) { rem -= nb4 - bi; ++bi; }
      const int bj = bi + rem;
      T acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = T(0);
      for (int kk = g; kk < nf; kk += G) {
        const T wk = (T)sw[kk];
        T x[4], y[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          x[a] = wk * zs[kk * RP + 4 * bi + a];
          y[a] = zs[kk * RP + 4 * bj + a];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fma(x[a], y[c], acc[a][c]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int r1 = 4 * bi + a, r2 = 4 * bj + c;
          if (r1 < R && r2 < R) {
            red[(g * R + r1) * R + r2] = acc[a][c];
            if (bi != bj) red[(g * R + r2) * R + r1] = acc[a][c];
          }
        }
    }
    __syncthreads();
    for (int e = tid; e < R * R; e += kWThreads) {
      T s = red[e];
      for (int gg = 1; gg < G; ++gg) s += red[gg * R * R + e];
      red[e] = s;
    }
  }
  // cluster sum (rank order) -> this cluster's partial; the last cluster to arrive sums them
  SWM(5);
  const int CU = (int)cluster.num_blocks(), q = (int)cluster.block_rank();
  const int ncl = gridDim.x / CU, cl = blockIdx.x / CU;
  T* gcl = reinterpret_cast<T*>(P.gcl);
  cluster.sync();
  {
    const int E = R * R, per = (E + CU - 1) / CU;
    for (int e = q * per + tid; e < min(E, (q + 1) * per); e += kWThreads) {
      T s = T(0);
      for (int qq = 0; qq < CU; ++qq) s += cluster.map_shared_rank(red, qq)[e];
      gcl[(int64_t)cl * E + e] = s;
    }
  }
  SWM(6);
  __threadfence();
  cluster.sync();  // the whole cluster partial is written
  if (q == 0 && tid == 0) s_last = (atomicAdd(P.cnt, 1u) == (unsigned)(ncl - 1));
  cluster.sync();
  if (*cluster.map_shared_rank(&s_last, 0)) {  // this cluster arrived last: its CTAs sum all partials
    __threadfence();
    T* out = reinterpret_cast<T*>(sp.gam_next);
    const int E = R * R, per = (E + CU - 1) / CU;
    for (int e = q * per + tid; e < min(E, (q + 1) * per); e += kWThreads) {
      T v[16], s = T(0);
      for (int c0 = 0; c0 < ncl; c0 += 16) {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = (c0 + k < ncl) ? __ldcg(gcl + (int64_t)(c0 + k) * E + e) : T(0);
#pragma unroll
        for (int k = 0; k < 16; ++k) s += v[k];  // cluster order; zeros past ncl are exact
      }
      out[e] = s;
    }
    if (q == 0 && tid == 0) *P.cnt = 0u;
  }
  cluster.sync();  // rank 0's s_last read by the peers before it exits
  SWM(7);
  if (P.dbg && tid == 0 && blockIdx.x < 480) {
    long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    P.dbg[2048 + 2 * blockIdx.x] = gt0;
    P.dbg[2049 + 2 * blockIdx.x] = gt1;
  }
}

}  // namespace cps
