// fused.cuh -- persistent single-cluster sweep kernel for problems whose whole step fits one
// thread-block cluster (C1-C3 of BASELINE.json): one launch runs `nsteps` SGD iterations.
//
// CTA q of the 16-CTA cluster owns
//   * fibers [q*BPC, (q+1)*BPC) of every batch: it samples them (Alg. 3/4 + contract), keeps
//     their SKR rows (Alg. 1), weights and offsets in shared memory, gathers them (Alg. 5) and
//     forms the partial M_q = X_F,q diag(w) Z_F,q and Gamma_q (eq:gradient1/2);
//   * rows [q*RPC, (q+1)*RPC) of the factor being updated: it reduces M and Gamma over the
//     cluster through DSMEM in rank order (deterministic), updates its rows (eq:proposed /
//     eq:Aada), and contributes its rows to the importance table of the new factor.
// Phases are separated by cluster barriers only -- no kernel boundary, no host round trip.
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cps {

constexpr int kFThreads = 256;
constexpr int kFChunk = 16;  // fibers whose values are loaded per round

template <typename T>
struct FusedParams {
  int N, R, strategy, rule, CU;
  int64_t dims[kMaxOrder];
  int64_t stride[kMaxOrder];       // first-index-fastest strides of the native tensor
  const T* Xg[kMaxOrder];          // gather base of mode n: mode-major copy or the native tensor
  int64_t estride[kMaxOrder];      // element stride along the fiber in that layout
  int64_t pitch[kMaxOrder];        // row pitch of the mode-major copy (0: native)
  T* factors[kMaxOrder];
  T* S[kMaxOrder];
  uint64_t* cdf[kMaxOrder];
  double* pprob[kMaxOrder];
  uint64_t* Ttot;
  int* status;
  uint64_t* iter;
  uint64_t seed;
  int64_t B;
  int32_t window[kMaxOrder][kMaxOrder];
  int64_t bmax[kMaxOrder];
  double alpha, eta, b, eps;
  const double* alpha_dev;
  int nsteps, first_mode, order;   // order: 0 cyclic, 1 random
  T* Gout;
  T* Gam_out;
  int* last_mode;                  // out
  int BPC;                         // fibers per CTA (max over modes)
  int RPC;                         // factor rows per CTA (max over modes)
  int64_t Imax;
  long long* dbg;
};

// shared memory layout (bytes) -- mirrored by the host
struct FusedLayout {
  size_t zw, zu, fb, wt, ix, mp, gp, gam, aold, anew, gpart, gm, prow, qrow, qtot, cdfs, total;
};
__host__ __device__ inline FusedLayout fused_layout(int N, int R, int BPC, int RPC, int64_t Imax, int64_t cdf_elems,
                                                    size_t esz) {
  FusedLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    off = (off + 15) / 16 * 16;
    size_t at = off;
    off += bytes;
    return at;
  };
  L.zw = take(esz * BPC * R);
  L.zu = take(esz * BPC * R);
  L.fb = take(sizeof(int64_t) * BPC);
  L.wt = take(sizeof(double) * BPC);
  L.ix = take(sizeof(int32_t) * BPC * (N - 1));
  L.mp = take(esz * Imax * R);
  L.gp = take(esz * R * R);
  L.gam = take(esz * R * R);
  L.aold = take(esz * RPC * (R + 1));
  L.anew = take(esz * RPC * (R + 1));
  L.gpart = take(sizeof(double) * (R * (R + 1) / 2 + 2));
  L.gm = take(sizeof(double) * R * (R + 1));
  L.prow = take(sizeof(double) * RPC);
  L.qrow = take(sizeof(unsigned long long) * RPC);
  L.qtot = take(sizeof(unsigned long long) * 2);
  L.cdfs = take(sizeof(uint64_t) * cdf_elems);
  L.total = off + 16;
  return L;
}

// ------------------------------------------------------------------------------------------
// single-warp register-resident symmetric sweep (Gauss-Jordan on the SPD Gram, natural pivot
// order, pivots with Schur diagonal <= tol skipped -- reading R4(b)); lane j owns column j.
// On exit Gm (stride R+1) holds W = (G_SS)^{-1} on the swept set S and 0 elsewhere; returns |S|.
// ------------------------------------------------------------------------------------------
template <int RMAX>
__device__ int warp_sweep_inverse(double* Gm, int R, double tol) {
  const int lane = threadIdx.x & 31;
  const int RS = R + 1;
  double col[RMAX];
#pragma unroll
  for (int i = 0; i < RMAX; ++i) col[i] = (lane < R && i < R) ? Gm[i * RS + lane] : 0.0;
  bool swept = false;
  int rank = 0;
#pragma unroll 1
  for (int k = 0; k < R; ++k) {
    // diagonal of column k lives in lane k: M[k][k] = col_k[k]
    double mine = 0.0;
#pragma unroll
    for (int i = 0; i < RMAX; ++i)
      if (i == k) mine = col[i];
    const double d = __shfl_sync(0xffffffffu, mine, k);
    if (!(d > tol)) continue;  // numerically dependent column: leave unswept
    ++rank;
    const double dinv = __drcp_rn(d);
    // my entry in row k (= M[k][lane]) and the pivot column entries M[i][k] (broadcast from lane k)
    double mkj = 0.0;
#pragma unroll
    for (int i = 0; i < RMAX; ++i)
      if (i == k) mkj = col[i];
#pragma unroll
    for (int i = 0; i < RMAX; ++i) {
      const double mik = __shfl_sync(0xffffffffu, col[i], k);
      if (i < R) {
        if (lane == k) {
          col[i] = (i == k) ? -dinv : col[i] * dinv;
        } else {
          col[i] = (i == k) ? mkj * dinv : col[i] - mik * (mkj * dinv);
        }
      }
    }
    if (lane == k) swept = true;
  }
  // W = -M on S x S
  const unsigned sm = __ballot_sync(0xffffffffu, swept);
#pragma unroll
  for (int i = 0; i < RMAX; ++i)
    if (lane < R && i < R) Gm[i * RS + lane] = (swept && ((sm >> i) & 1u)) ? -col[i] : 0.0;
  __syncwarp();
  return rank;
}

// ------------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------------
template <typename T, int RMAX, int ROWS>
__global__ void __launch_bounds__(kFThreads, 1) k_sweep_fused(FusedParams<T> p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int CU = p.CU;
  const int q = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int N = p.N, R = p.R, RS = R + 1;
  extern __shared__ __align__(16) unsigned char f_sm[];
  int64_t cdf_elems = 0;
  {
    int64_t mx = 0;
    for (int n = 0; n < N; ++n) {
      int64_t s = 0;
      for (int k = 0; k < N; ++k)
        if (k != n) s += p.dims[k];
      mx = max(mx, s);
    }
    cdf_elems = (p.strategy == 0) ? 0 : mx;
  }
  const FusedLayout L = fused_layout(N, R, p.BPC, p.RPC, p.Imax, cdf_elems, sizeof(T));
  T* zw = reinterpret_cast<T*>(f_sm + L.zw);
  T* zu = reinterpret_cast<T*>(f_sm + L.zu);
  int64_t* fb = reinterpret_cast<int64_t*>(f_sm + L.fb);
  double* wt = reinterpret_cast<double*>(f_sm + L.wt);
  int32_t* ix = reinterpret_cast<int32_t*>(f_sm + L.ix);
  T* Mp = reinterpret_cast<T*>(f_sm + L.mp);
  T* Gp = reinterpret_cast<T*>(f_sm + L.gp);
  T* Gam = reinterpret_cast<T*>(f_sm + L.gam);
  T* Aold = reinterpret_cast<T*>(f_sm + L.aold);
  T* Anew = reinterpret_cast<T*>(f_sm + L.anew);
  double* gpart = reinterpret_cast<double*>(f_sm + L.gpart);
  double* Gm = reinterpret_cast<double*>(f_sm + L.gm);
  double* prow = reinterpret_cast<double*>(f_sm + L.prow);
  unsigned long long* qrow = reinterpret_cast<unsigned long long*>(f_sm + L.qrow);
  unsigned long long* qtot = reinterpret_cast<unsigned long long*>(f_sm + L.qtot);
  uint64_t* cdfs = reinterpret_cast<uint64_t*>(f_sm + L.cdfs);
  __shared__ int64_t s_beff;
  __shared__ int s_bad;
  __shared__ double s_red[kFThreads / 32];
  __shared__ unsigned long long s_wtot[kFThreads / 32];
  __shared__ const uint64_t* s_cp[kMaxOrder];
  if (tid == 0) s_bad = 0;

  uint64_t r = *p.iter;
  const bool block = (p.strategy == 3 || p.strategy == 4);
  auto mode_of = [&](uint64_t it, int s) -> int {
    return p.order == 1 ? random_mode(p.seed, it, N) : (p.first_mode + s) % N;
  };

  // ---- sample this CTA's fibers of the batch of mode n at iteration it (contract §8c.2) ----
  auto sample_own = [&](int n, uint64_t it) {
    // stage the CDFs of the modes k != n
    int64_t off = 0;
    if (tid < kMaxOrder) s_cp[tid] = nullptr;
    __syncthreads();
    for (int k = 0; k < N; ++k) {
      if (k == n || p.strategy == 0) continue;
      for (int64_t i = tid; i < p.dims[k]; i += kFThreads) cdfs[off + i] = p.cdf[k][i];
      if (tid == 0) s_cp[k] = cdfs + off;
      off += p.dims[k];
    }
    __syncthreads();
    const int64_t bmax = p.bmax[n];
    const int64_t b0 = (int64_t)q * p.BPC;
    // block strategies: the window draws are common to the whole batch
    int32_t start[kMaxOrder], len[kMaxOrder];
    double wblk = 0.0;
    int64_t beff = p.B;
    if (block) {
      double prod = 1.0;
      beff = 1;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == n) continue;
        const int64_t bk = p.window[n][pos];
        const uint64_t Tk = p.Ttot[k];
        const uint64_t rr = scale_draw(draw_word(p.seed, it, 0u, kPurposeWindow, (uint32_t)pos), Tk);
        const uint64_t* c = s_cp[k];
        const int64_t istar = upper_bound_u64(c, p.dims[k], rr);
        const int64_t s0 = (istar / bk) * bk, e0 = min(s0 + bk, p.dims[k]);
        const uint64_t Q = c[e0 - 1] - (s0 > 0 ? c[s0 - 1] : 0ull);
        start[pos] = (int32_t)s0;
        len[pos] = (int32_t)(e0 - s0);
        const double pt = __ddiv_rn((double)((uint64_t)p.dims[k] * Q), (double)Tk);
        prod = (pos == 0) ? pt : __dmul_rn(prod, pt);
        beff *= (e0 - s0);
        ++pos;
      }
      wblk = __ddiv_rn(1.0, prod);
    }
    if (tid == 0) s_beff = beff;
    for (int lb = tid; lb < p.BPC; lb += kFThreads) {
      const int64_t b = b0 + lb;
      int32_t* ib = ix + lb * (N - 1);
      if (b >= bmax || b >= beff) {
        fb[lb] = -1;
        wt[lb] = 0.0;
        continue;
      }
      if (!block) {
        double prod = 1.0;
        int pos = 0;
        for (int k = 0; k < N; ++k) {
          if (k == n) continue;
          const uint64_t Tk = (p.strategy == 0) ? (uint64_t)p.dims[k] : p.Ttot[k];
          const uint64_t rr = scale_draw(draw_word(p.seed, it, (uint32_t)b, kPurposeRow, (uint32_t)pos), Tk);
          int64_t i;
          uint64_t qk;
          if (p.strategy == 0) {
            i = (int64_t)rr;
            qk = 1;
          } else {
            const uint64_t* c = s_cp[k];
            i = upper_bound_u64(c, p.dims[k], rr);
            qk = c[i] - (i > 0 ? c[i - 1] : 0ull);
          }
          ib[pos] = (int32_t)i;
          const double pt = __ddiv_rn((double)((uint64_t)p.dims[k] * qk), (double)Tk);
          prod = (pos == 0) ? pt : __dmul_rn(prod, pt);
          ++pos;
        }
        wt[lb] = __ddiv_rn(1.0, __dmul_rn((double)p.B, prod));
      } else {
        int64_t rem = b;
        for (int qq = 0; qq < N - 1; ++qq) {
          ib[qq] = start[qq] + (int32_t)(rem % len[qq]);
          rem /= len[qq];
        }
        wt[lb] = wblk;
      }
      int64_t offn = 0, jrow = 0, jmul = 1;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == n) continue;
        const int64_t ik = ib[pos++];
        offn += ik * p.stride[k];
        jrow += ik * jmul;
        jmul *= p.dims[k];
      }
      fb[lb] = p.pitch[n] ? jrow * p.pitch[n] : offn;
    }
    __syncthreads();
    // SKR rows (Alg. 1): z = (*)_{k != n} A^(k)(i_k, :); zw = w z
    for (int e = tid; e < p.BPC * R; e += kFThreads) {
      const int lb = e / R, rr = e % R;
      T z = T(0), zwv = T(0);
      if (fb[lb] >= 0) {
        const int32_t* ib = ix + lb * (N - 1);
        z = T(1);
        int pos = 0;
        for (int k = 0; k < N; ++k) {
          if (k == n) continue;
          z = z * p.factors[k][(int64_t)ib[pos++] * R + rr];
        }
        zwv = (T)wt[lb] * z;
      }
      zu[e] = z;
      zw[e] = zwv;
    }
    __syncthreads();
  };

  int n = mode_of(r, 0);
  int n_done = n;
  sample_own(n, r);

#pragma unroll 1
  for (int s = 0; s < p.nsteps; ++s) {
    const int64_t In = p.dims[n];
    const int64_t rpc = (In + CU - 1) / CU;
    const int64_t r_beg = min((int64_t)q * rpc, In), r_end = min(r_beg + rpc, In);
    const int nr = (int)(r_end - r_beg);
    // ------------------------------------------------ (1) gather + partial contractions
    {
      T acc[ROWS][RMAX];
#pragma unroll
      for (int u = 0; u < ROWS; ++u)
#pragma unroll
        for (int j = 0; j < RMAX; ++j) acc[u][j] = T(0);
      const T* Xn = p.Xg[n];
      const int64_t es = p.estride[n];
      for (int c0 = 0; c0 < p.BPC; c0 += kFChunk) {
        T xv[kFChunk][ROWS];
#pragma unroll
        for (int c = 0; c < kFChunk; ++c) {
          const int lb = c0 + c;
          const int64_t f = (lb < p.BPC) ? fb[lb] : -1;
#pragma unroll
          for (int u = 0; u < ROWS; ++u) {
            const int64_t i = tid + (int64_t)u * kFThreads;
            xv[c][u] = (f >= 0 && i < In) ? __ldg(Xn + f + i * es) : T(0);
          }
        }
#pragma unroll
        for (int c = 0; c < kFChunk; ++c) {
          const int lb = c0 + c;
          if (lb < p.BPC) {
#pragma unroll
            for (int j = 0; j < RMAX; ++j) {
              const T z = (j < R) ? zw[lb * R + j] : T(0);
#pragma unroll
              for (int u = 0; u < ROWS; ++u) acc[u][j] += xv[c][u] * z;
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < ROWS; ++u) {
        const int64_t i = tid + (int64_t)u * kFThreads;
        if (i < In)
#pragma unroll
          for (int j = 0; j < RMAX; ++j)
            if (j < R) Mp[i * R + j] = acc[u][j];
      }
      for (int e = tid; e < R * R; e += kFThreads) {
        const int r1 = e / R, r2 = e % R;
        T g = T(0);
        for (int lb = 0; lb < p.BPC; ++lb) g += zw[lb * R + r1] * zu[lb * R + r2];
        Gp[e] = g;
      }
    }
    cluster.sync();  // #1: partials visible
    // ------------------------------------------------ (2) cluster reduction (rank order) + update
    for (int e = tid; e < R * R; e += kFThreads) {
      T g = T(0);
      for (int qq = 0; qq < CU; ++qq) g += cluster.map_shared_rank(Gp, qq)[e];
      Gam[e] = g;
    }
    for (int e = tid; e < nr * R; e += kFThreads) {
      const int il = e / R, c = e % R;
      Aold[il * RS + c] = p.factors[n][(r_beg + il) * R + c];
    }
    __syncthreads();
    if (q == 0 && s == p.nsteps - 1)
      for (int e = tid; e < R * R; e += kFThreads) p.Gam_out[e] = Gam[e];
    const double alpha = p.alpha_dev ? *p.alpha_dev : p.alpha;
    for (int e = tid; e < nr * R; e += kFThreads) {
      const int il = e / R, rr = e % R;
      const int64_t i = r_beg + il;
      T m = T(0);
      for (int qq = 0; qq < CU; ++qq) m += cluster.map_shared_rank(Mp, qq)[i * R + rr];
      T ag = T(0);
      for (int c = 0; c < R; ++c) ag += Aold[il * RS + c] * Gam[c * R + rr];
      const T g = ag - m;
      const int64_t gi = i * R + rr;
      p.Gout[gi] = g;
      const T a = Aold[il * RS + rr];
      T an = a;
      if (p.rule == 0) {
        an = a - (T)alpha * g;
      } else {
        const T sv = p.S[n][gi] + g * g;
        p.S[n][gi] = sv;
        if (sv > T(0)) {
          T step;
          if (p.eps == 0.0) step = (T)p.eta / sqrt((T)p.b + sv);
          else step = (T)p.eta / (T)pow((double)((T)p.b + sv), 0.5 + p.eps);
          an = a - step * g;
        }
      }
      p.factors[n][gi] = an;
      Anew[il * RS + rr] = an;
    }
    __syncthreads();
    // ------------------------------------------------ (3) importance table of the new A^(n)
    if (p.strategy != 0) {
      const bool lev = (p.strategy == 1 || p.strategy == 3);
      const int P = R * (R + 1) / 2;
      if (lev) {
        for (int pair = tid; pair < P; pair += kFThreads) {
          int r1 = 0, rem = pair;
          while (rem >= R - r1) { rem -= R - r1; ++r1; }
          const int r2 = r1 + rem;
          double a2 = 0.0;
          for (int il = 0; il < nr; ++il) a2 += (double)Anew[il * RS + r1] * (double)Anew[il * RS + r2];
          gpart[pair] = a2;
        }
      } else {
        double a2 = 0.0;
        for (int il = tid; il < nr; il += kFThreads) {
          double rs = 0.0;
          for (int c = 0; c < R; ++c) rs += (double)Anew[il * RS + c] * (double)Anew[il * RS + c];
          prow[il] = rs;
          a2 += rs;
        }
        for (int o = 16; o > 0; o >>= 1) a2 += __shfl_down_sync(0xffffffffu, a2, o);
        if (lane == 0) s_red[wid] = a2;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
          for (int w = 0; w < kFThreads / 32; ++w) t += s_red[w];
          gpart[0] = t;
        }
      }
      cluster.sync();  // #2: partial Grams / norms visible
      int rank = 1;
      double fro = 1.0;
      if (lev) {
        for (int pair = tid; pair < P; pair += kFThreads) {
          double sum = 0.0;
          for (int qq = 0; qq < CU; ++qq) sum += cluster.map_shared_rank(gpart, qq)[pair];
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
          for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
          if (!__all_sync(0xffffffffu, fin) && lane == 0) s_bad |= 8;
          const double tol = (double)(In > R ? In : R) * 2.220446049250313e-16 * d0;
          const int rk = warp_sweep_inverse<RMAX>(Gm, R, tol);
          if (lane == 0) s_red[0] = (double)rk;
        }
        __syncthreads();
        rank = (int)s_red[0];
        if (tid == 0 && rank == 0) s_bad |= 2;
        // scores: l = a^T W a, one warp per row, lanes over the R^2 products
        for (int il = wid; il < nr; il += kFThreads / 32) {
          const T* a = Anew + il * RS;
          double part = 0.0;
          for (int e = lane; e < R * R; e += 32) {
            const int i = e / R, j = e % R;
            part += (double)a[i] * Gm[i * RS + j] * (double)a[j];
          }
          for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
          if (lane == 0) prow[il] = rank > 0 ? fmax(part, 0.0) / (double)rank : 0.0;
        }
      } else {
        if (tid == 0) {
          double t = 0.0;
          for (int qq = 0; qq < CU; ++qq) t += cluster.map_shared_rank(gpart, qq)[0];
          s_red[0] = t;
          if (!(t == t) || t > 1.7e308) s_bad |= 8;
          else if (!(t > 0.0)) s_bad |= 2;
        }
        __syncthreads();
        fro = s_red[0];
        for (int il = tid; il < nr; il += kFThreads) prow[il] = prow[il] / fro;
      }
      __syncthreads();
      // quantise + scan (thread per row; rows per CTA <= kFThreads)
      unsigned long long qv = 0;
      if (tid < nr) {
        const double pv = prow[tid];
        if (!(pv == pv) || pv > 2.0) {
          atomicOr(&s_bad, 8);
        } else if (pv > 0.0) {
          const double sc = rint(pv * 4294967296.0);
          qv = (sc < 1.0) ? 1ull : (unsigned long long)sc;
        }
        p.pprob[n][r_beg + tid] = pv;
      }
      unsigned long long incl = qv;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) s_wtot[wid] = incl;
      __syncthreads();
      unsigned long long wpre = 0;
      for (int w = 0; w < wid; ++w) wpre += s_wtot[w];
      if (tid == kFThreads - 1) qtot[0] = wpre + incl;
      __syncthreads();
      cluster.sync();  // #3: CTA totals visible
      unsigned long long cpre = 0, total = 0;
      for (int qq = 0; qq < CU; ++qq) {
        const unsigned long long t = cluster.map_shared_rank(qtot, qq)[0];
        if (qq < q) cpre += t;
        total += t;
      }
      if (tid < nr) p.cdf[n][r_beg + tid] = cpre + wpre + incl;
      if (tid == 0) {
        if (q == 0) p.Ttot[n] = total;
        int st = 0;
        if (s_bad & 8) st = -8;
        else if ((s_bad & 2) || (q == 0 && total == 0)) st = -3;
        if (st) atomicCAS(p.status, 0, st);
      }
    }
    ++r;
    n_done = n;
    const int n_next = mode_of(r, s + 1);
    __threadfence();
    cluster.sync();  // #4: factors, CDF and T of mode n visible cluster-wide; peers done with our smem
    if (s + 1 < p.nsteps) {
      sample_own(n_next, r);
    }
    n = n_next;
  }
  if (q == 0 && tid == 0) {
    *p.iter = r;
    *p.last_mode = n_done;
  }
}

}  // namespace cps
