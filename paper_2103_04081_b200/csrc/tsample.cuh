// tsample.cuh -- k_table_sample: the second launch of a wide-path step (after k_gather_update).
// ONE thread-block cluster of CU <= 16 CTAs (CTA q owns rows [q*rows_per, ...) of A^(n) and
// fibers [q*fpc, ...) of the next batch):
//
//   (a1) importance table of the updated A^(n) (R9: rebuilt after every update):
//        leverage  -- fp64 partial Grams of the owned rows (4x4 register blocks), rank-ordered DSMEM
//                     sum, symmetric sweep inverse W = (A_S^T A_S)^{-1} (R4b), scores
//                     l_i = a_i^T W a_i = ||Q(i,:)||^2 (Def. 2.3), p = l / rank;
//        euclidean -- p_i = ||a_i||^2 / ||A||_F^2 (Def. 2.5);
//        q = rint(p 2^32) (>= 1 if p > 0), CDF = integer scan (CTA scan + DSMEM prefix).
//   (a2, a3) the next batch of mode n' at iteration r (contract DESIGN.md section 4), kept in shared
//        memory; (a4) its SKR rows z_b = (*)_{k != n'} A^(k)(i_k, :) (Alg. 1);
//        zw_b = w_b z_b -> p.sp.zwp (what k_gather_update streams); Gamma = sum_b zw_b z_b^T
//        (eq:gradient1/2), rank-ordered over the cluster -> p.sp.gam_next.
//
// Every phase is shared-memory resident: global memory is touched once per phase (factor rows,
// CDFs), never re-read after a barrier.
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cps {

constexpr int kTSThreads = 256;

template <typename T>
struct TSParams {
  int R, strategy;
  int64_t In;           // rows of A^(n)
  int64_t rows_per;     // rows per CTA
  const T* A;           // A^(n), updated by k_gather_update
  double* p_out;
  uint64_t* cdf;
  uint64_t* Tout;
  int* status;
  int sample_next;
  int64_t fpc;          // fibers of the next batch per CTA
  SampleParams sp;      // next batch (mode sp.n); sp.zwp / sp.gam_next set
  // stage U (wide path, p.Mpart != NULL): finish the step k_gather_update started
  const T* Mpart;       // [tiles][CK][R][128] chunk partials of M = X_F diag(w) Z_F
  int CK;
  const T* Gam;         // Gamma of this step's batch (R x R)
  T* Aw;                // A^(n), updated in place (== A)
  T* S;                 // adaptive accumulator of mode n, or NULL
  T* Gout;              // G (debug hook)
  int rule;
  double alpha;
  const double* alpha_dev;
  double eta, b, eps;
  long long* dbg;
};

struct TSLayout {
  size_t us, uss, ug, um;                                               // update phase (rows: stride R+1)
  size_t ad, work, gpart, gm, colbuf, swept, prow, qrow, qtot, tbytes;   // table phase
  size_t cdfs, sidx, sw, zs, red, sbytes;                               // sample phase (aliases)
  size_t total;
};

__host__ __device__ inline TSLayout ts_layout(int N, int R, int64_t rows_per, int64_t fpc, int64_t cdf_elems,
                                              size_t esz) {
  TSLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = (off + 15) / 16 * 16;
    const size_t at = off;
    off += bytes;
    return at;
  };
  const int RD = ut_rd(R);
  // table phase
  L.ad = take(sizeof(double) * rows_per * RD);
  const size_t ad_end = off;
  L.work = take(ut_work_bytes(R, rows_per));
  L.gpart = take(sizeof(double) * (R * (R + 1) / 2 + 1));
  L.gm = take(sizeof(double) * R * (R + 1));
  L.colbuf = take(sizeof(double) * 2 * kMaxRank);
  L.swept = take(sizeof(int) * kMaxRank);
  L.prow = take(sizeof(double) * rows_per);
  L.qrow = take(sizeof(unsigned long long) * rows_per);
  L.qtot = take(sizeof(unsigned long long) * 2);
  L.tbytes = off;
  // update phase (before the table; everything but `us` is dead once the rows are updated, and `us`
  // only until the fp64 copy `ad` is filled, so `us` must not overlap `ad`)
  off = 0;
  L.uss = take(esz * rows_per * (R + 1));    // S rows
  L.ug = take(esz * R * R);                  // Gamma
  L.um = take(esz * rows_per * (R + 1));     // M rows -> G rows
  if (off < ad_end) off = ad_end;
  L.us = take(esz * rows_per * (R + 1));     // rows of A^(n), updated
  const size_t ubytes = off;
  // sample phase
  off = 0;
  const int RP = zg_rp(R);
  L.cdfs = take(sizeof(uint64_t) * cdf_elems);
  L.sidx = take(sizeof(int32_t) * fpc * (N - 1));
  L.sw = take(sizeof(double) * fpc);
  L.zs = take(esz * fpc * RP);
  L.red = take(esz * (size_t)zg_groups(R, kTSThreads) * R * R);
  L.sbytes = off;
  size_t tot = L.tbytes > L.sbytes ? L.tbytes : L.sbytes;
  L.total = (tot > ubytes ? tot : ubytes) + 16;
  return L;
}

#define TS_MARK(slot)                                              \
  do {                                                             \
    if (p.dbg && q == 0 && tid == 0) p.dbg[slot] = clock64();      \
  } while (0)

template <typename T>
__global__ void __launch_bounds__(kTSThreads, 1) k_table_sample(TSParams<T> p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int CU = (int)cluster.num_blocks(), q = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int R = p.R, RD = ut_rd(R), nb4 = (R + 3) >> 2, P = R * (R + 1) / 2, RS = R + 1;
  const int64_t r_beg = cmin64((int64_t)q * p.rows_per, p.In), r_end = cmin64(r_beg + p.rows_per, p.In);
  const int nr = (int)(r_end - r_beg);
  const SampleParams& sp = p.sp;
  int64_t cdf_elems = 0;
  if (p.sample_next && sp.strategy != 0)
    for (int k = 0; k < sp.N; ++k)
      if (k != sp.n) cdf_elems += sp.dims[k];
  const TSLayout L = ts_layout(sp.N, R, p.rows_per, p.fpc, cdf_elems, sizeof(T));
  extern __shared__ __align__(16) unsigned char ts_sm[];
  double* Ad = reinterpret_cast<double*>(ts_sm + L.ad);
  double* work = reinterpret_cast<double*>(ts_sm + L.work);
  double* gpart = reinterpret_cast<double*>(ts_sm + L.gpart);
  double* Gm = reinterpret_cast<double*>(ts_sm + L.gm);
  double* colbuf = reinterpret_cast<double*>(ts_sm + L.colbuf);
  int* swept = reinterpret_cast<int*>(ts_sm + L.swept);
  double* prow = reinterpret_cast<double*>(ts_sm + L.prow);
  unsigned long long* qtot = reinterpret_cast<unsigned long long*>(ts_sm + L.qtot);
  __shared__ int s_bad;
  __shared__ double s_red[kTSThreads / 32];
  __shared__ unsigned long long s_wtot[kTSThreads / 32];
  __shared__ double s_tol, s_fro;
  if (tid == 0) s_bad = 0;
  TS_MARK(0);
  T* As = reinterpret_cast<T*>(ts_sm + L.us);  // rows of A^(n) owned by this CTA (stride R+1)
  if (p.Mpart) {
    // ======================= (a6-a8) finish the step: G = A Gamma - sum_c M_c, update =======================
    T* Ss = reinterpret_cast<T*>(ts_sm + L.uss);
    T* sG = reinterpret_cast<T*>(ts_sm + L.ug);
    T* Mf = reinterpret_cast<T*>(ts_sm + L.um);
    for (int e = tid; e < nr * R; e += kTSThreads) {
      const int il = e / R, c = e % R;
      cp_async_small<sizeof(T)>(As + il * RS + c, p.Aw + (r_beg + il) * R + c, sizeof(T));
      if (p.rule != 0) cp_async_small<sizeof(T)>(Ss + il * RS + c, p.S + (r_beg + il) * R + c, sizeof(T));
    }
    for (int e = tid; e < R * R; e += kTSThreads) cp_async_small<sizeof(T)>(sG + e, p.Gam + e, sizeof(T));
    cp_async_commit();
    // M rows: partials [tile][c][r][128 rows], 16-byte vectors of VW rows, chunks summed in order
    {
      constexpr int VW = 16 / (int)sizeof(T);
      using V = typename Vec<T>::type;
      const int ng = (nr + VW - 1) / VW;  // rows_per and r_beg are multiples of 4 (host)
      const int ntask = R * ng;
      constexpr int TU = 2;
      for (int t0 = tid; t0 < ntask; t0 += TU * kTSThreads) {
        T acc[TU][VW];
        int64_t off[TU];
#pragma unroll
        for (int u = 0; u < TU; ++u) {
          const int t = t0 + u * kTSThreads;
          const int r = t / ng, gq = t % ng;
          const int64_t row = r_beg + (int64_t)gq * VW;
          off[u] = t < ntask ? ((row / kGUTI) * p.CK * R + r) * kGUTI + (row % kGUTI) : -1;
#pragma unroll
          for (int w = 0; w < VW; ++w) acc[u][w] = T(0);
        }
        for (int c0 = 0; c0 < p.CK; c0 += 8) {
          V ld[TU][8];
#pragma unroll
          for (int u = 0; u < TU; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (off[u] >= 0 && c0 + k < p.CK)
                ld[u][k] = __ldcg(reinterpret_cast<const V*>(p.Mpart + off[u] + (int64_t)(c0 + k) * R * kGUTI));
#pragma unroll
          for (int u = 0; u < TU; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (off[u] >= 0 && c0 + k < p.CK) {
                const T* x = reinterpret_cast<const T*>(&ld[u][k]);
#pragma unroll
                for (int w = 0; w < VW; ++w) acc[u][w] += x[w];
              }
        }
#pragma unroll
        for (int u = 0; u < TU; ++u) {
          const int t = t0 + u * kTSThreads;
          if (t >= ntask) continue;
          const int r = t / ng, gq = t % ng;
#pragma unroll
          for (int w = 0; w < VW; ++w)
            if (gq * VW + w < nr) Mf[(gq * VW + w) * RS + r] = acc[u][w];
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    // G = A Gamma - M (4 rows x 4 columns per task), then the fixed / adaptive update in place
    T* Gf = Mf;
    {
      const int ntask = ((nr + 3) >> 2) * nb4;
      for (int t = tid; t < ntask; t += kTSThreads) {
        const int r0 = 4 * (t / nb4), q0 = 4 * (t % nb4);
        T acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = T(0);
        for (int k = 0; k < R; ++k) {
          T x[4], y[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) x[a] = (r0 + a < nr) ? As[(r0 + a) * RS + k] : T(0);
#pragma unroll
          for (int c = 0; c < 4; ++c) y[c] = (q0 + c < R) ? sG[k * R + q0 + c] : T(0);
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[a][c] = fma(x[a], y[c], acc[a][c]);
        }
        // each task reads and writes only its own 4x4 block of M -> G in place
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (r0 + a < nr && q0 + c < R) Gf[(r0 + a) * RS + q0 + c] = acc[a][c] - Mf[(r0 + a) * RS + q0 + c];
      }
    }
    __syncthreads();
    const double alpha = p.alpha_dev ? *p.alpha_dev : p.alpha;
    for (int e = tid; e < nr * R; e += kTSThreads) {
      const int il = e / R, r = e % R;
      const int64_t gi = (r_beg + il) * R + r;
      const T g = Gf[il * RS + r];
      p.Gout[gi] = g;
      const T a = As[il * RS + r];
      T an = a;
      if (p.rule == 0) {
        an = a - (T)alpha * g;
      } else {
        const T sv = Ss[il * RS + r] + g * g;
        p.S[gi] = sv;
        if (sv > T(0)) {
          T step;
          if (p.eps == 0.0) step = (T)p.eta / sqrt((T)p.b + sv);
          else step = (T)p.eta / (T)pow((double)((T)p.b + sv), 0.5 + p.eps);
          an = a - step * g;
        }
      }
      p.Aw[gi] = an;
      As[il * RS + r] = an;
    }
    __syncthreads();
    TS_MARK(7);
  }

  if (p.strategy != 0) {
    // ======================= (a1) table of the updated A^(n) =======================
    const bool lev = (p.strategy == 1 || p.strategy == 3);
#pragma unroll 8
    for (int e = tid; e < nr * RD; e += kTSThreads) {  // fp64 copy of the owned rows, zero padded to RD
      const int il = e / RD, c = e % RD;
      Ad[e] = c < R ? (double)(p.Mpart ? As[il * RS + c] : p.A[(r_beg + il) * R + c]) : 0.0;
    }
    __syncthreads();
    if (lev) {
      // partial Gram of the owned rows: thread = (row group g, 4x4 block bi <= bj)
      const int nblk = nb4 * (nb4 + 1) / 2, GG = ut_gram_groups(R);
      const int g = tid / nblk, blk = tid % nblk;
      if (g < GG) {
        int bi = 0, rem = blk;
        while (rem >= nb4 - bi) { rem -= nb4 - bi; ++bi; }
        const int bj = bi + rem;
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
        for (int il = g; il < nr; il += GG) {
          const double2 x0 = *reinterpret_cast<const double2*>(Ad + il * RD + 4 * bi);
          const double2 x1 = *reinterpret_cast<const double2*>(Ad + il * RD + 4 * bi + 2);
          const double2 y0 = *reinterpret_cast<const double2*>(Ad + il * RD + 4 * bj);
          const double2 y1 = *reinterpret_cast<const double2*>(Ad + il * RD + 4 * bj + 2);
          const double x[4] = {x0.x, x0.y, x1.x, x1.y}, y[4] = {y0.x, y0.y, y1.x, y1.y};
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
            if (r1 < R && r2 < R && r1 <= r2) work[g * P + r1 * R - r1 * (r1 - 1) / 2 + (r2 - r1)] = acc[a][c];
          }
      }
      __syncthreads();
      for (int pair = tid; pair < P; pair += kTSThreads) {
        double s = work[pair];
        for (int gg = 1; gg < GG; ++gg) s += work[gg * P + pair];
        gpart[pair] = s;
      }
    } else {
      double acc = 0.0;
      for (int il = tid; il < nr; il += kTSThreads) {  // ||a_i||^2
        double rs = 0.0;
        for (int c = 0; c < R; ++c) rs += Ad[il * RD + c] * Ad[il * RD + c];
        prow[il] = rs;
      }
      __syncthreads();
      for (int il = tid; il < nr; il += kTSThreads) acc += prow[il];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
      if (lane == 0) s_red[wid] = acc;
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < kTSThreads / 32; ++w) t += s_red[w];
        gpart[0] = t;
      }
    }
    cluster.sync();  // #1 partial Grams / norms visible
    TS_MARK(1);
    int rank = 0;
    if (lev) {
      for (int pair = tid; pair < P; pair += kTSThreads) {
        double v[16];
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) v[qq] = (qq < CU) ? cluster.map_shared_rank(gpart, qq)[pair] : 0.0;
        double sum = 0.0;
#pragma unroll
        for (int qq = 0; qq < 16; ++qq) sum += v[qq];  // rank order (zeros past CU are exact)
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
      constexpr int EPT = (kMaxRank * kMaxRank + kTSThreads - 1) / kTSThreads;
      rank = (p.In < 2 * R) ? cta_sweep_inverse_pivoted<EPT>(Gm, R, s_tol, colbuf, swept, colbuf + R)
                            : lc_sweep_dispatch(Gm, R, s_tol, colbuf, swept);
      if (tid == 0 && rank == 0) s_bad |= 2;
      TS_MARK(2);
      // scores l_i = sum_c (A W)_ic a_ic (4 rows x 4 columns per task; k in pairs)
      double* Wd = work;
      double* sc = work + R * RD;  // [nb4][rows_per]
      for (int e = tid; e < R * RD; e += kTSThreads) {
        const int r1 = e / RD, c = e % RD;
        Wd[e] = c < R ? Gm[r1 * RS + c] : 0.0;
      }
      __syncthreads();
      const int nrg = (nr + 3) >> 2, ntask = nrg * nb4;
      for (int t = tid; t < ntask; t += kTSThreads) {
        const int rg = t / nb4, cg = t % nb4;
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
          const double2 w00 = *reinterpret_cast<const double2*>(Wd + kk * RD + 4 * cg);
          const double2 w01 = *reinterpret_cast<const double2*>(Wd + kk * RD + 4 * cg + 2);
          const double2 w10 = *reinterpret_cast<const double2*>(Wd + k1 * RD + 4 * cg);
          const double2 w11 = *reinterpret_cast<const double2*>(Wd + k1 * RD + 4 * cg + 2);
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
          const double2 x0 = *reinterpret_cast<const double2*>(arow[a] + 4 * cg);
          const double2 x1 = *reinterpret_cast<const double2*>(arow[a] + 4 * cg + 2);
          sc[cg * p.rows_per + il0 + a] = acc[a][0] * x0.x + acc[a][1] * x0.y + acc[a][2] * x1.x + acc[a][3] * x1.y;
        }
      }
      __syncthreads();
      for (int il = tid; il < nr; il += kTSThreads) {
        double l = 0.0;
        for (int cg = 0; cg < nb4; ++cg) l += sc[cg * p.rows_per + il];
        prow[il] = rank > 0 ? fmax(l, 0.0) / (double)rank : 0.0;
      }
    } else {
      if (tid == 0) {
        double fro = 0.0;
        for (int qq = 0; qq < CU; ++qq) fro += cluster.map_shared_rank(gpart, qq)[0];
        s_fro = fro;
        if (!(fro == fro) || fro > 1.7e308) s_bad |= 8;
        else if (!(fro > 0.0)) s_bad |= 2;
      }
      __syncthreads();
      const double fro = s_fro;
      for (int il = tid; il < nr; il += kTSThreads) prow[il] = fro > 0.0 ? prow[il] / fro : 0.0;
    }
    __syncthreads();
    TS_MARK(3);
    // quantise + CTA scan (contiguous segment per thread) + DSMEM prefix of the lower ranks
    unsigned long long* qrow = reinterpret_cast<unsigned long long*>(ts_sm + L.qrow);
    const int seg = (nr + kTSThreads - 1) / kTSThreads;
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
    if (tid == kTSThreads - 1) qtot[0] = seg_pre + local;
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
    __threadfence();
    cluster.sync();  // #3 CDF / T of mode n visible cluster-wide; peers done with this CTA's table smem
    TS_MARK(4);
  }
  if (!p.sample_next) return;

  // ======================= (a2-a4) the next batch + zw rows + Gamma =======================
  const int N = sp.N, NP = N - 1, RP = zg_rp(R);
  uint64_t* cdfs = reinterpret_cast<uint64_t*>(ts_sm + L.cdfs);
  int32_t* sidx = reinterpret_cast<int32_t*>(ts_sm + L.sidx);
  double* sw = reinterpret_cast<double*>(ts_sm + L.sw);
  T* zs = reinterpret_cast<T*>(ts_sm + L.zs);
  T* red = reinterpret_cast<T*>(ts_sm + L.red);
  __shared__ const uint64_t* s_cp[kMaxOrder];
  {
    int64_t off = 0;
    for (int k = 0; k < N; ++k) {
      const uint64_t* src = sp.cdf[k];
      if (k != sp.n && sp.strategy != 0) {
        cp_async_u64(cdfs + off, src, sp.dims[k], tid, kTSThreads);
        src = cdfs + off;
        off += sp.dims[k];
      }
      if (tid == 0) s_cp[k] = src;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  const uint64_t r_now = *sp.iter;  // already advanced by k_gather_update
  const int64_t b0 = cmin64((int64_t)q * p.fpc, sp.bmax), b1 = cmin64(b0 + p.fpc, sp.bmax);
  const int nf = (int)(b1 - b0);
  draw_rows(sp, s_cp, r_now, b0, b1, tid, kTSThreads, sidx, sw);
  __syncthreads();
  TS_MARK(5);
  // SKR rows into shared memory: z[lb][r], all factor loads of a batch of elements in flight
  {
    const int cnt = nf * RP;
    constexpr int U = 8;
    for (int base = 0; base < cnt; base += kTSThreads * U) {
      T z[U];
      int lbu[U], ru[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * kTSThreads + tid;
        lbu[u] = e < cnt ? e / RP : -1;
        ru[u] = e % RP;
        z[u] = T(1);
      }
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == sp.n) continue;
        const T* F = reinterpret_cast<const T*>(sp.factors[k]);
        T f[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          f[u] = (lbu[u] >= 0 && ru[u] < R) ? F[(int64_t)sidx[lbu[u] * NP + pos] * R + ru[u]] : T(0);
#pragma unroll
        for (int u = 0; u < U; ++u) z[u] = z[u] * f[u];
        ++pos;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (lbu[u] >= 0) zs[lbu[u] * RP + ru[u]] = z[u];
    }
  }
  __syncthreads();
  // zw rows for k_gather_update (coalesced), Gamma partial from shared memory
  {
    T* zwp = reinterpret_cast<T*>(sp.zwp);
    for (int e = tid; e < nf * RP; e += kTSThreads) {
      const int lb = e / RP, r = e % RP;
      const T zw = (T)sw[lb] * zs[e];
      zwp[(b0 + lb) * RP + r] = zw;
      if constexpr (sizeof(T) == 4) {
        if (sp.zhi && r < R) write_zw_images(sp, b0 + lb, r, (float)zw);
      }
    }
    const int nblk = nb4 * (nb4 + 1) / 2, G = zg_groups(R, kTSThreads);
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
    for (int e = tid; e < R * R; e += kTSThreads) {
      T s = red[e];
      for (int gg = 1; gg < G; ++gg) s += red[gg * R * R + e];
      red[e] = s;
    }
    gamma_cluster_reduce<T>(cluster, red, R, reinterpret_cast<T*>(sp.gam_next), tid, kTSThreads);
  }
  TS_MARK(6);
}

}  // namespace cps
