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
  int rebuild;                     // 1: factors staged in fstage (host input): every mode whose factor differs
                                   // from the device copy is replaced and its table rebuilt before step 0
  const T* fstage[kMaxOrder];
  T* Gout;
  T* Gam_out;
  int* last_mode;                  // out
  int BPC;                         // fibers per CTA (max over modes)
  int RPC;                         // factor rows per CTA (max over modes)
  int64_t Imax;
  TraceParams tr;                  // cp_sgd_trace (debug): consumed batches and resulting states
  long long* dbg;
};

// shared memory layout (bytes) -- mirrored by the host
struct FusedLayout {
  size_t zw, zu, fb, wt, ix, pt, mp, gp, gam, aold, anew, sold, gpart, gm, prow, sc, rowbuf, swept, qtot, qpre, cdfs, xs, total;
};
// row pitch (elements) of the staged fiber segments: I_max rounded up to a 16-byte multiple
__host__ __device__ inline int64_t fused_xpitch(int64_t Imax, size_t esz) {
  const int64_t VE = 16 / (int64_t)esz;
  return (Imax + VE - 1) / VE * VE;
}
__host__ __device__ inline int fused_rp(int R, size_t esz) {
  const int W = esz == 8 ? 2 : 4;
  return (R + W - 1) / W * W;
}
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
  const int RP = fused_rp(R, esz);
  L.zw = take(esz * BPC * RP);
  L.zu = take(esz * BPC * RP);
  L.fb = take(sizeof(int64_t) * BPC);
  L.wt = take(sizeof(double) * BPC);
  L.ix = take(sizeof(int32_t) * BPC * (N - 1));
  L.pt = take(sizeof(double) * BPC * (N - 1));
  L.mp = take(esz * Imax * (R + 1));
  L.gp = take(esz * R * R);
  L.gam = take(esz * R * R);
  L.aold = take(esz * RPC * (R + 1));
  L.anew = take(esz * RPC * (R + 1));
  L.sold = take(esz * RPC * (R + 1));
  L.gpart = take(sizeof(double) * (R * (R + 1) / 2 + 2));
  L.gm = take(sizeof(double) * R * (R + 1));
  L.prow = take(sizeof(double) * RPC);
  L.sc = take(sizeof(double) * RPC * R);
  L.rowbuf = take(sizeof(double) * kSweepBuf);
  L.swept = take(sizeof(int) * R);
  L.qtot = take(sizeof(unsigned long long) * 2);
  L.qpre = take(sizeof(unsigned long long) * RPC);
  L.cdfs = take(sizeof(uint64_t) * cdf_elems);
  L.xs = take(esz * (size_t)BPC * fused_xpitch(Imax, esz));
  L.total = off + 16;
  return L;
}



// fiber gather + contraction for ROWS rows per thread and RV vector groups of columns:
// acc[u][g] += x(row u) * zw[lb][g]; zw rows padded to RV * W with zeros (stride RP).
template <typename T, int ROWS, int RV>
__device__ __forceinline__ void gather_contract(const T* xs, int64_t Ip, int64_t In, const int64_t* fb,
                                                const T* zw, int RP, int BPC, T* Mp, int R, long long* dbg = nullptr) {
  using V = typename Vec<T>::type;
  constexpr int W = Vec<T>::W;
  const int tid = threadIdx.x;
  V acc[ROWS][RV];
#pragma unroll
  for (int u = 0; u < ROWS; ++u)
#pragma unroll
    for (int g = 0; g < RV; ++g) {
      T* a = reinterpret_cast<T*>(&acc[u][g]);
#pragma unroll
      for (int c = 0; c < W; ++c) a[c] = T(0);
    }
  constexpr int CH = 16;
  if (dbg) dbg[16] = clock64();
  for (int c0 = 0; c0 < BPC; c0 += CH) {
    T xv[CH][ROWS];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int lb = c0 + c;
#pragma unroll
      for (int u = 0; u < ROWS; ++u) {
        const int i = tid + u * kFThreads;
        // clamped unconditional load, then select (a conditional load compiles to a branch per load);
        // padding fibers are staged as zeros
        const T t = xs[(lb < BPC ? lb : BPC - 1) * Ip + (i < In ? i : In - 1)];
        xv[c][u] = (lb < BPC && i < In) ? t : T(0);
      }
    }
    if (dbg && c0 < 2 * CH) {
      if (xv[CH - 1][ROWS - 1] == T(-12345)) xv[0][0] = T(0);
      dbg[17 + 2 * (c0 / CH)] = clock64();
    }
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int lb = c0 + c;
      if (lb >= BPC) break;
      const V* z = reinterpret_cast<const V*>(zw + lb * RP);
      if constexpr (sizeof(T) == 4) {
        // packed fp32x2 FMA (FFMA2): two independent round-to-nearest FMAs per instruction, the same
        // values as the scalar form with half the issue slots
        uint64_t xx[ROWS];
#pragma unroll
        for (int u = 0; u < ROWS; ++u) asm("mov.b64 %0, {%1, %1};" : "=l"(xx[u]) : "f"((float)xv[c][u]));
#pragma unroll
        for (int g = 0; g < RV; ++g) {
          const V zg = z[g];
          const uint64_t* z2 = reinterpret_cast<const uint64_t*>(&zg);
#pragma unroll
          for (int u = 0; u < ROWS; ++u) {
            uint64_t* a2 = reinterpret_cast<uint64_t*>(&acc[u][g]);
#pragma unroll
            for (int h = 0; h < 2; ++h) asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a2[h]) : "l"(xx[u]), "l"(z2[h]));
          }
        }
      } else {
#pragma unroll
        for (int g = 0; g < RV; ++g) {
          const V zg = z[g];
          const T* zt = reinterpret_cast<const T*>(&zg);
#pragma unroll
          for (int u = 0; u < ROWS; ++u) {
            T* a = reinterpret_cast<T*>(&acc[u][g]);
#pragma unroll
            for (int cc = 0; cc < W; ++cc) a[cc] += xv[c][u] * zt[cc];
          }
        }
      }
    }
    if (dbg && c0 < 2 * CH) {
      if (reinterpret_cast<T*>(&acc[ROWS - 1][RV - 1])[W - 1] == T(-12345)) xv[0][0] = T(1);
      dbg[18 + 2 * (c0 / CH)] = clock64();
    }
  }
#pragma unroll
  for (int u = 0; u < ROWS; ++u) {
    const int64_t i = tid + (int64_t)u * kFThreads;
    if (i < In) {
#pragma unroll
      for (int g = 0; g < RV; ++g) {
        const T* a = reinterpret_cast<const T*>(&acc[u][g]);
#pragma unroll
        for (int cc = 0; cc < W; ++cc) {
          const int j = g * W + cc;
          if (j < R) Mp[i * (R + 1) + j] = a[cc];  // row pitch R + 1: conflict-free across lanes
        }
      }
    }
  }
}

template <typename T, int ROWS>
__device__ __forceinline__ void gather_dispatch(const T* xs, int64_t Ip, int64_t In, const int64_t* fb, const T* zw,
                                                int RP, int BPC, T* Mp, int R, long long* dbg = nullptr) {
  switch (RP / Vec<T>::W) {
    case 1: gather_contract<T, ROWS, 1>(xs, Ip, In, fb, zw, RP, BPC, Mp, R, dbg); break;
    case 2: gather_contract<T, ROWS, 2>(xs, Ip, In, fb, zw, RP, BPC, Mp, R, dbg); break;
    case 3: gather_contract<T, ROWS, 3>(xs, Ip, In, fb, zw, RP, BPC, Mp, R, dbg); break;
    case 4: gather_contract<T, ROWS, 4>(xs, Ip, In, fb, zw, RP, BPC, Mp, R, dbg); break;
    case 5: gather_contract<T, ROWS, 5>(xs, Ip, In, fb, zw, RP, BPC, Mp, R, dbg); break;
    case 6: gather_contract<T, ROWS, 6>(xs, Ip, In, fb, zw, RP, BPC, Mp, R, dbg); break;
    case 7: gather_contract<T, ROWS, 7>(xs, Ip, In, fb, zw, RP, BPC, Mp, R, dbg); break;
    default: gather_contract<T, ROWS, 8>(xs, Ip, In, fb, zw, RP, BPC, Mp, R, dbg); break;
  }
}

template <typename T>
__device__ __forceinline__ bool bits_equal(T a, T b) {
  if constexpr (sizeof(T) == 8) return __double_as_longlong(a) == __double_as_longlong(b);
  else return __float_as_uint(a) == __float_as_uint(b);
}

// ------------------------------------------------------------------------------------------
// the kernel
// ------------------------------------------------------------------------------------------
#define F_MARK(slot)                                                          \
  do {                                                                        \
    if (p.dbg && q == 0 && tid == 0 && s == 1) p.dbg[slot] = clock64();       \
  } while (0)

template <typename T, int ROWS>
__device__ __forceinline__ void fused_body(const FusedParams<T>& p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int CU = p.CU;
  const int q = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int N = p.N, R = p.R, RS = R + 1, NP = N - 1;
  const int RP = fused_rp(R, sizeof(T));
  extern __shared__ __align__(16) unsigned char f_sm[];
  int64_t cdf_elems = 0;  // resident CDFs of every mode
  if (p.strategy != 0)
    for (int k = 0; k < N; ++k) cdf_elems += p.dims[k];
  const FusedLayout L = fused_layout(N, R, p.BPC, p.RPC, p.Imax, cdf_elems, sizeof(T));
  T* zw = reinterpret_cast<T*>(f_sm + L.zw);
  T* zu = reinterpret_cast<T*>(f_sm + L.zu);
  int64_t* fb = reinterpret_cast<int64_t*>(f_sm + L.fb);
  double* wt = reinterpret_cast<double*>(f_sm + L.wt);
  int32_t* ix = reinterpret_cast<int32_t*>(f_sm + L.ix);
  double* ptm = reinterpret_cast<double*>(f_sm + L.pt);
  T* Mp = reinterpret_cast<T*>(f_sm + L.mp);
  T* Gp = reinterpret_cast<T*>(f_sm + L.gp);
  T* Gam = reinterpret_cast<T*>(f_sm + L.gam);
  T* Aold = reinterpret_cast<T*>(f_sm + L.aold);
  T* Sold = reinterpret_cast<T*>(f_sm + L.sold);
  T* Anew = reinterpret_cast<T*>(f_sm + L.anew);
  double* gpart = reinterpret_cast<double*>(f_sm + L.gpart);
  double* Gm = reinterpret_cast<double*>(f_sm + L.gm);
  double* prow = reinterpret_cast<double*>(f_sm + L.prow);
  double* sc = reinterpret_cast<double*>(f_sm + L.sc);
  double* rowbuf = reinterpret_cast<double*>(f_sm + L.rowbuf);
  int* swept = reinterpret_cast<int*>(f_sm + L.swept);
  unsigned long long* qtot = reinterpret_cast<unsigned long long*>(f_sm + L.qtot);
  uint64_t* cdfs = reinterpret_cast<uint64_t*>(f_sm + L.cdfs);  // resident CDFs, mode k at cdf_off[k]
  unsigned long long* qpre = reinterpret_cast<unsigned long long*>(f_sm + L.qpre);  // CTA-inclusive prefix of q
  T* xs = reinterpret_cast<T*>(f_sm + L.xs);
  const int64_t Ip = fused_xpitch(p.Imax, sizeof(T));
  __shared__ int s_bad;
  __shared__ double s_red[kFThreads / 32];
  __shared__ unsigned long long s_wtot[kFThreads / 32];
  __shared__ const uint64_t* s_cp[kMaxOrder];
  __shared__ uint64_t s_T[kMaxOrder];
  __shared__ unsigned long long s_off[17];
  __shared__ double s_tol_als;
  __shared__ int32_t s_start[kMaxOrder], s_len[kMaxOrder];
  __shared__ double s_wblk;
  __shared__ int64_t s_beff;
  if (tid == 0) s_bad = 0;

  uint64_t r = *p.iter;
  const bool block = (p.strategy == 3 || p.strategy == 4);
  auto mode_of = [&](uint64_t it, int st) -> int {
    return p.order == 1 ? random_mode(p.seed, it, N) : (p.first_mode + st) % N;
  };

  // ---- this CTA's fibers [q*BPC, (q+1)*BPC) of the batch of mode n at iteration it (contract §8c.2)
  // the CDFs of every mode stay resident in shared memory: staged once here, then each table
  // rebuild assembles the new CDF of its mode from the cluster's CTA prefixes over DSMEM
  if (tid < kMaxOrder) s_cp[tid] = nullptr;
  __syncthreads();
  if (p.strategy != 0) {
    int64_t off = 0;
    for (int k = 0; k < N; ++k) {
      cp_async_u64(cdfs + off, p.cdf[k], p.dims[k], tid, kFThreads);
      if (tid == 0) {
        s_cp[k] = cdfs + off;
        s_T[k] = p.Ttot[k];
      }
      off += p.dims[k];
    }
    cp_async_commit();
    cp_async_wait<0>();
  }
  __syncthreads();

  long long* sdbg = nullptr;  // debug phase marks of one sample_own call
  auto sample_own = [&](int n, uint64_t it) {
    if (sdbg && tid == 0) sdbg[23] = clock64();
    if (block && tid == 0) {  // window draws (eq:bik, R2): common to the whole batch
      double prod = 1.0;
      int64_t beff = 1;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == n) continue;
        const int64_t bk = p.window[n][pos];
        const uint64_t Tk = s_T[k];
        const uint64_t rr = scale_draw(draw_word(p.seed, it, 0u, kPurposeWindow, (uint32_t)pos), Tk);
        const uint64_t* c = s_cp[k];
        const int64_t istar = upper_bound_u64(c, p.dims[k], rr);
        const int64_t s0 = (istar / bk) * bk, e0 = min(s0 + bk, p.dims[k]);
        const uint64_t cprev = c[s0 > 0 ? s0 - 1 : 0];  // unconditional load, then select
        const uint64_t Q = c[e0 - 1] - (s0 > 0 ? cprev : 0ull);
        s_start[pos] = (int32_t)s0;
        s_len[pos] = (int32_t)(e0 - s0);
        const double pt = __ddiv_rn((double)((uint64_t)p.dims[k] * Q), (double)Tk);
        prod = (pos == 0) ? pt : __dmul_rn(prod, pt);
        beff *= (e0 - s0);
        ++pos;
      }
      s_wblk = __ddiv_rn(1.0, prod);
      s_beff = beff;
    } else if (tid == 0) {
      s_beff = p.B;
    }
    __syncthreads();
    const int64_t bmax = p.bmax[n], b0 = (int64_t)q * p.BPC, beff = s_beff;
    if (!block) {  // one thread per (fiber, position) draw (eq:ik)
      for (int e = tid; e < p.BPC * NP; e += kFThreads) {
        const int lb = e / NP, pos = e % NP;
        const int64_t b = b0 + lb;
        if (b >= bmax) continue;
        int k = pos < n ? pos : pos + 1;
        const uint64_t Tk = (p.strategy == 0) ? (uint64_t)p.dims[k] : s_T[k];
        const uint64_t rr = scale_draw(draw_word(p.seed, it, (uint32_t)b, kPurposeRow, (uint32_t)pos), Tk);
        int64_t i;
        uint64_t qk;
        if (p.strategy == 0) {
          i = (int64_t)rr;
          qk = 1;
        } else {
          const uint64_t* c = s_cp[k];
          i = upper_bound_u64(c, p.dims[k], rr);
          const uint64_t cprev = c[i > 0 ? i - 1 : 0];  // unconditional load, then select
          qk = c[i] - (i > 0 ? cprev : 0ull);
        }
        ix[e] = (int32_t)i;
        ptm[e] = __ddiv_rn((double)((uint64_t)p.dims[k] * qk), (double)Tk);
      }
      __syncthreads();
    }
    if (sdbg && tid == 0) sdbg[24] = clock64();
    for (int lb = tid; lb < p.BPC; lb += kFThreads) {
      const int64_t b = b0 + lb;
      int32_t* ib = ix + lb * NP;
      if (b >= bmax || b >= beff) {
        fb[lb] = -1;
        wt[lb] = 0.0;
        continue;
      }
      if (!block) {
        double prod = ptm[lb * NP];
        for (int pos = 1; pos < NP; ++pos) prod = __dmul_rn(prod, ptm[lb * NP + pos]);
        wt[lb] = __ddiv_rn(1.0, __dmul_rn((double)p.B, prod));
      } else {
        int64_t rem = b;
        for (int qq = 0; qq < NP; ++qq) {
          ib[qq] = s_start[qq] + (int32_t)(rem % s_len[qq]);
          rem /= s_len[qq];
        }
        wt[lb] = s_wblk;
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
    if (sdbg && tid == 0) sdbg[25] = clock64();
    // TensorSamp (Alg. 5) issue: this CTA's fiber segments -> shared memory (xs[lb][i], pitch Ip) by
    // cp.async, completed at the gather.  The copies overlap the SKR rows and, for the next step's
    // batch, the whole tail of the current step.  (Direct loads at the gather were bound by the
    // SM's outstanding-miss limit: ~4.6k cycles per 16-fiber round, tools/micro/gat_lat.cu.)
    {
      const T* Xn = p.Xg[n];
      const int64_t In = p.dims[n], es = p.estride[n];
      constexpr int VE = 16 / (int)sizeof(T);
      const int nv = (int)((In + VE - 1) / VE);
      for (int e = tid; e < p.BPC * nv; e += kFThreads) {
        const int lb = e / nv, v = e % nv;
        const int64_t f = fb[lb];
        const int64_t i0 = (int64_t)v * VE;
        T* dst = xs + lb * Ip + i0;
        if (f < 0) {  // padding fiber: zeros, so the contraction needs no per-fiber test
#pragma unroll
          for (int j = 0; j < VE; ++j) dst[j] = T(0);
        } else if (es == 1 && (f % VE) == 0) {
          cp_async16(dst, Xn + f + i0, (int)(cmin64(VE, In - i0) * (int64_t)sizeof(T)));
        } else {
#pragma unroll
          for (int j = 0; j < VE; ++j)
            if (i0 + j < In) cp_async_small<sizeof(T)>(dst + j, Xn + f + (i0 + j) * es, (int)sizeof(T));
        }
      }
      cp_async_commit();
    }
    if (sdbg && tid == 0) sdbg[26] = clock64();
    // SKR rows (Alg. 1): z = (*)_{k != n} A^(k)(i_k, :); zw = w z; padded to RP with zeros.  kSU
    // entries per thread and two modes per round: their factor loads are issued together (one L2
    // round trip per two modes instead of one per mode and entry); the products keep the mode order.
    // The loads are coherent: rows of the mode updated in the previous step were written by peer CTAs
    // inside this kernel (ordered by the cluster barriers); the non-coherent path may not see them.
    {
      constexpr int kSU = 4;
      for (int e0 = 0; e0 < p.BPC * RP; e0 += kSU * kFThreads) {
        T z[kSU];
        bool act[kSU];
        int lbu[kSU];
#pragma unroll
        for (int u = 0; u < kSU; ++u) {
          const int e = e0 + u * kFThreads + tid;
          const int lb = e / RP, rr = e % RP;
          lbu[u] = lb;
          act[u] = e < p.BPC * RP && rr < R && fb[lb] >= 0;
          z[u] = act[u] ? T(1) : T(0);
        }
        for (int pos = 0; pos < NP; pos += 2) {
          const int k0 = pos < n ? pos : pos + 1, k1 = pos + 1 < n ? pos + 1 : pos + 2;
          const bool two = pos + 1 < NP;
          T f0[kSU], f1[kSU];
#pragma unroll
          for (int u = 0; u < kSU; ++u) {
            const int e = e0 + u * kFThreads + tid, rr = e % RP;
            // every load issued (a valid address: row 0 for inactive entries), then selected: a
            // conditional load compiles to a branch per load
            const int32_t* ibs = ix + (lbu[u] < p.BPC ? lbu[u] : p.BPC - 1) * NP;
            const int rc = rr < R ? rr : R - 1;
            const int32_t i0 = ibs[pos], i1 = two ? ibs[pos + 1] : 0;
            const T t0 = p.factors[k0][(int64_t)(act[u] ? i0 : 0) * R + rc];
            const T t1 = p.factors[two ? k1 : k0][(int64_t)((act[u] && two) ? i1 : 0) * R + rc];
            f0[u] = act[u] ? t0 : T(0);
            f1[u] = (act[u] && two) ? t1 : T(0);
          }
#pragma unroll
          for (int u = 0; u < kSU; ++u) {
            if (!act[u]) continue;
            z[u] = z[u] * f0[u];
            if (two) z[u] = z[u] * f1[u];
          }
        }
#pragma unroll
        for (int u = 0; u < kSU; ++u) {
          const int e = e0 + u * kFThreads + tid;
          if (e < p.BPC * RP) {
            zu[e] = z[u];
            zw[e] = act[u] ? (T)wt[lbu[u]] * z[u] : T(0);
          }
        }
      }
    }
    __syncthreads();
    if (sdbg && tid == 0) sdbg[27] = clock64();
  };

  // (a1) the table of the new A^(n) from this CTA's rows Anew (Gram / norm partials, cluster sums,
  // sweep inverse, scores, quantisation, scan, resident CDF); s: the step index (phase marks), -1 for
  // the rebuild prologue
  auto build_table = [&](int n, int64_t In, int64_t rpc, int64_t r_beg, int nr, int s) {
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
        __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
        for (int o = 16; o > 0; o >>= 1) a2 += __shfl_down_sync(0xffffffffu, a2, o);
        if (lane == 0) s_red[wid] = a2;
        __syncthreads();
        if (tid == 0) {
          double t = 0.0;
          for (int w = 0; w < kFThreads / 32; ++w) t += s_red[w];
          gpart[0] = t;
        }
      }
      F_MARK(4);
      cluster.sync();  // #2: partial Grams / norms visible
      F_MARK(5);
      if (lev) {
        for (int pair = tid; pair < P; pair += kFThreads) {
          const double sum = cluster_sum(cluster, gpart, pair, CU);
          int r1 = 0, rem = pair;
          while (rem >= R - r1) { rem -= R - r1; ++r1; }
          const int r2 = r1 + rem;
          Gm[r1 * RS + r2] = sum;
          Gm[r2 * RS + r1] = sum;
        }
        __syncthreads();
        F_MARK(13);
        if (wid == 0) {
          double d0 = 0.0;
          bool fin = true;
          for (int j = lane; j < R; j += 32) {
            const double d = Gm[j * RS + j];
            d0 = fmax(d0, d);
            fin = fin && (d == d) && d < 1.7e308;
          }
          __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
          for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
          if (!__all_sync(0xffffffffu, fin) && lane == 0) s_bad |= 8;
          if (lane == 0) s_red[0] = (double)(In > R ? In : R) * 2.220446049250313e-16 * d0;
        }
        __syncthreads();
        constexpr int EPT = (32 * 32 + kFThreads - 1) / kFThreads;
        const int rank = (In < 2 * R) ? cta_sweep_inverse_pivoted<EPT>(Gm, R, s_red[0], rowbuf, swept, rowbuf + R)
                                      : grp_sweep_dispatch<32>(Gm, R, s_red[0], rowbuf, swept);
        F_MARK(6);
        if (tid == 0 && rank == 0) s_bad |= 2;
        // scores l = a^T W a: thread per (row, i) forms a_i * (W a)_i; rows summed in order
        for (int e = tid; e < nr * R; e += kFThreads) {
          const int il = e / R, i = e % R;
          const T* a = Anew + il * RS;
          double t = 0.0;
          for (int j = 0; j < R; ++j) t += Gm[i * RS + j] * (double)a[j];
          sc[e] = (double)a[i] * t;
        }
        __syncthreads();
        for (int il = tid; il < nr; il += kFThreads) {
          double l = 0.0;
          for (int i = 0; i < R; ++i) l += sc[il * R + i];
          prow[il] = rank > 0 ? fmax(l, 0.0) / (double)rank : 0.0;
        }
      } else {
        if (tid == 0) {
          const double t = cluster_sum(cluster, gpart, 0, CU);
          s_red[0] = t;
          if (!(t == t) || t > 1.7e308) s_bad |= 8;
          else if (!(t > 0.0)) s_bad |= 2;
        }
        __syncthreads();
        const double fro = s_red[0];
        for (int il = tid; il < nr; il += kFThreads) prow[il] = fro > 0.0 ? prow[il] / fro : 0.0;
      }
      __syncthreads();
      F_MARK(7);
      // quantise + scan (thread per row; rows per CTA <= kFThreads)
      unsigned long long qv = 0;
      if (tid < nr) {
        const double pv = prow[tid];
        if (!(pv == pv) || pv > 2.0) {
          atomicOr(&s_bad, 8);
        } else if (pv > 0.0) {
          const double scv = rint(pv * 4294967296.0);
          qv = (scv < 1.0) ? 1ull : (unsigned long long)scv;
        }
        p.pprob[n][r_beg + tid] = pv;
      }
      unsigned long long incl = qv;
      __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) s_wtot[wid] = incl;
      __syncthreads();
      unsigned long long wpre = 0;
      for (int w = 0; w < wid; ++w) wpre += s_wtot[w];
      if (tid < nr) qpre[tid] = wpre + incl;
      if (tid == kFThreads - 1) qtot[0] = wpre + incl;
      F_MARK(8);
      cluster.sync();  // #3: CTA totals visible
      F_MARK(9);
      // CTA totals -> exclusive offsets (16 DSMEM loads, once per CTA)
      if (tid < 16) s_off[tid] = tid < CU ? cluster.map_shared_rank(qtot, tid)[0] : 0ull;
      __syncthreads();
      if (tid == 0) {
        unsigned long long acc = 0;
        for (int qq = 0; qq < 16; ++qq) {
          const unsigned long long v = s_off[qq];
          s_off[qq] = acc;
          acc += v;
        }
        s_off[16] = acc;
      }
      __syncthreads();
      const unsigned long long cpre = s_off[q], total = s_off[16];
      if (tid < nr) p.cdf[n][r_beg + tid] = cpre + wpre + incl;  // for the host / later launches
      {  // the new CDF of mode n in every CTA's resident copy: the peers' prefixes over DSMEM
        uint64_t* cn = const_cast<uint64_t*>(s_cp[n]);
        constexpr int U = 2;  // rows per thread per round, loads issued together
        for (int64_t r0 = tid; r0 < In; r0 += U * kFThreads) {
          unsigned long long v[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t row = r0 + u * kFThreads;
            const int owner = row < In ? (int)(row / rpc) : 0;
            v[u] = row < In ? cluster.map_shared_rank(qpre, owner)[row - owner * rpc] + s_off[owner] : 0ull;
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (r0 + u * kFThreads < In) cn[r0 + u * kFThreads] = v[u];
        }
      }
      if (tid == 0) {
        s_T[n] = total;
        if (q == 0) p.Ttot[n] = total;
        int st = 0;
        if (s_bad & 8) st = -8;
        else if ((s_bad & 2) || (q == 0 && total == 0)) st = -3;
        if (st) atomicCAS(p.status, 0, st);
      }
    }
  };

  if (p.rebuild) {
    // host input (cp_sgd_steps_host): each CTA compares its row block of every staged factor with the
    // device copy; a mode with any difference anywhere is taken over and its table rebuilt (the
    // tables are a function of the factors: an unchanged factor keeps its table)
    __shared__ unsigned s_chg;
    if (tid == 0) s_chg = 0u;
    __syncthreads();
    for (int k = 0; k < N; ++k) {
      const int64_t In = p.dims[k];
      const int64_t rpc = (In + CU - 1) / CU;
      const int64_t r_beg = min((int64_t)q * rpc, In);
      const int nr = (int)(min(r_beg + rpc, In) - r_beg);
      bool diff = false;
      for (int e = tid; e < nr * R; e += kFThreads)
        diff |= !bits_equal(p.fstage[k][r_beg * R + e], p.factors[k][r_beg * R + e]);
      if (__syncthreads_or(diff) && tid == 0) s_chg |= 1u << k;
    }
    cluster.sync();
    unsigned chg = 0u;
    for (int qq = 0; qq < CU; ++qq) chg |= *cluster.map_shared_rank(&s_chg, qq);
    cluster.sync();  // every peer has read this CTA's flags
    for (int k = 0; k < N; ++k) {
      if (!((chg >> k) & 1u)) continue;
      const int64_t In = p.dims[k];
      const int64_t rpc = (In + CU - 1) / CU;
      const int64_t r_beg = min((int64_t)q * rpc, In);
      const int nr = (int)(min(r_beg + rpc, In) - r_beg);
      for (int e = tid; e < nr * R; e += kFThreads) {
        const T v = p.fstage[k][r_beg * R + e];
        p.factors[k][r_beg * R + e] = v;
        Anew[(e / R) * RS + e % R] = v;
      }
      __syncthreads();
      if (p.strategy != 0) build_table(k, In, rpc, r_beg, nr, -1);
      cluster.sync();  // new rows visible; the peers are done with this build's prefixes
    }
  }
  int n = mode_of(r, 0);
  int n_done = n;
  sample_own(n, r);

#pragma unroll 1
  for (int s = 0; s < p.nsteps; ++s) {
    F_MARK(0);
    const int64_t In = p.dims[n];
    const int64_t rpc = (In + CU - 1) / CU;
    const int64_t r_beg = min((int64_t)q * rpc, In), r_end = min(r_beg + rpc, In);
    const int nr = (int)(r_end - r_beg);
    // ------------------------------------------------ (1) gather (Alg. 5) + partial contractions
    cp_async_wait<0>();  // this batch's fiber segments (issued by sample_own)
    __syncthreads();
    // old rows (and adaptive accumulators) of the block this CTA updates: in flight during the gather
    for (int e = tid; e < nr * R; e += kFThreads) {
      const int il = e / R, c = e % R;
      cp_async_small<sizeof(T)>(Aold + il * RS + c, p.factors[n] + (r_beg + il) * R + c, sizeof(T));
      if (p.rule == 1) cp_async_small<sizeof(T)>(Sold + il * RS + c, p.S[n] + (r_beg + il) * R + c, sizeof(T));
    }
    cp_async_commit();
    const bool trace = p.tr.base && p.tr.first + s < p.tr.cap;
    unsigned char* tb = trace ? p.tr.base + (p.tr.first + s) * p.tr.stride : nullptr;
    if (trace) {  // the batch this step consumes: this CTA's fibers (debug trace)
      int32_t* ti = reinterpret_cast<int32_t*>(tb + p.tr.o_idx);
      double* tw = reinterpret_cast<double*>(tb + p.tr.o_w);
      const int64_t bm = p.bmax[n], b0 = (int64_t)q * p.BPC;
      for (int e = tid; e < p.BPC * NP; e += kFThreads) {
        const int64_t b = b0 + e / NP;
        if (b < bm) ti[b * NP + e % NP] = b < s_beff ? ix[e] : 0;
      }
      for (int lb = tid; lb < p.BPC; lb += kFThreads)
        if (b0 + lb < bm) tw[b0 + lb] = wt[lb];
      if (q == 0 && tid == 0) {
        int64_t* tm = reinterpret_cast<int64_t*>(tb + p.tr.o_meta);
        tm[0] = n;
        tm[1] = (int64_t)r;
        tm[2] = s_beff;
        tm[3] = 0;
      }
    }
    const double alpha = p.alpha_dev ? *p.alpha_dev : p.alpha;
    gather_dispatch<T, ROWS>(xs, Ip, In, fb, zw, RP, p.BPC, Mp, R,
                             (p.dbg && q == 0 && tid == 0 && s == 1) ? p.dbg : nullptr);
    F_MARK(14);
    {  // Gamma partial: 2 x 2 blocks (each entry still summed over the CTA's fibers in order)
      const int h2 = (R + 1) >> 1;
      for (int e = tid; e < h2 * h2; e += kFThreads) {
        const int r1 = 2 * (e / h2), r2 = 2 * (e % h2);
        const int r1b = r1 + 1 < R ? r1 + 1 : r1, r2b = r2 + 1 < R ? r2 + 1 : r2;
        T g00 = T(0), g01 = T(0), g10 = T(0), g11 = T(0);
        for (int lb = 0; lb < p.BPC; ++lb) {
          const T w0 = zw[lb * RP + r1], w1 = zw[lb * RP + r1b], u0 = zu[lb * RP + r2], u1 = zu[lb * RP + r2b];
          g00 += w0 * u0;
          g01 += w0 * u1;
          g10 += w1 * u0;
          g11 += w1 * u1;
        }
        Gp[r1 * R + r2] = g00;
        if (r2 + 1 < R) Gp[r1 * R + r2 + 1] = g01;
        if (r1 + 1 < R) Gp[(r1 + 1) * R + r2] = g10;
        if (r1 + 1 < R && r2 + 1 < R) Gp[(r1 + 1) * R + r2 + 1] = g11;
      }
    }
    F_MARK(15);
    cp_async_wait<0>();  // old rows / accumulators
    F_MARK(1);
    cluster.sync();  // #1: partials visible
    F_MARK(2);
    // ------------------------------------------------ (2) cluster reduction (rank order) + update
    // Gamma is symmetric: the upper triangle of the partials (the remote reads are the cost: the
    // SM's DSMEM read rate, ~14 B/clk), mirrored
    for (int pair = tid; pair < R * (R + 1) / 2; pair += kFThreads) {
      int r1 = 0, rem = pair;
      while (rem >= R - r1) { rem -= R - r1; ++r1; }
      const int r2 = r1 + rem;
      const T v = cluster_sum(cluster, Gp, r1 * R + r2, CU);
      Gam[r1 * R + r2] = v;
      Gam[r2 * R + r1] = v;
    }
    __syncthreads();
    if (q == 0 && s == p.nsteps - 1)
      for (int e = tid; e < R * R; e += kFThreads) p.Gam_out[e] = Gam[e];
    if (p.rule == 2) {
      // sampled least squares (eq:lsq_krp; R25): W = Gamma^+ in fp64 by the
      // natural-order sweep (tol R eps max diag), every CTA; the rows follow as A = M W below
      for (int e = tid; e < R * R; e += kFThreads) Gm[(e / R) * RS + e % R] = (double)Gam[e];
      __syncthreads();
      if (wid == 0) {
        double d0 = 0.0;
        for (int j = lane; j < R; j += 32) d0 = fmax(d0, Gm[j * RS + j]);
        __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
        for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
        if (lane == 0) s_tol_als = (double)R * 2.220446049250313e-16 * d0;
      }
      __syncthreads();
      grp_sweep_dispatch<32>(Gm, R, s_tol_als, rowbuf, swept);
    }
    for (int e = tid; e < nr * R; e += kFThreads) {
      const int il = e / R, rr = e % R;
      const int64_t i = r_beg + il;
      const T m = cluster_sum(cluster, Mp, (int)(i * (R + 1) + rr), CU);
      T ag = T(0);
      for (int c = 0; c < R; ++c) ag += Aold[il * RS + c] * Gam[c * R + rr];
      const T g = ag - m;
      const int64_t gi = i * R + rr;
      p.Gout[gi] = g;
      const T a = Aold[il * RS + rr];
      T an = a;
      if (p.rule == 2) {
        Sold[il * RS + rr] = m;  // the M rows (the accumulator buffer is unused by this rule)
        continue;
      }
      if (p.rule == 0) {
        an = a - (T)alpha * g;
      } else {
        const T sv = Sold[il * RS + rr] + g * g;
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
    if (p.rule == 2) {
      __syncthreads();
      for (int e = tid; e < nr * R; e += kFThreads) {
        const int il = e / R, rr = e % R;
        double an = 0.0;
        for (int c = 0; c < R; ++c) an = fma((double)Sold[il * RS + c], Gm[c * RS + rr], an);
        p.factors[n][(r_beg + il) * R + rr] = (T)an;
        Anew[il * RS + rr] = (T)an;
      }
    }
    __syncthreads();
    F_MARK(3);
    // ------------------------------------------------ (3) importance table of the new A^(n)
    build_table(n, In, rpc, r_beg, nr, s);
    if (trace) {  // this CTA's rows of the updated factor, accumulator and CDF (debug trace)
      __syncthreads();
      T* tA = reinterpret_cast<T*>(tb + p.tr.o_A);
      T* tS = reinterpret_cast<T*>(tb + p.tr.o_S);
      uint64_t* tc = reinterpret_cast<uint64_t*>(tb + p.tr.o_cdf);
      for (int e = tid; e < nr * R; e += kFThreads) {
        tA[r_beg * R + e] = Anew[(e / R) * RS + e % R];
        if (p.rule == 1) tS[r_beg * R + e] = p.S[n][r_beg * R + e];
      }
      for (int il = tid; il < nr; il += kFThreads) tc[r_beg + il] = p.cdf[n][r_beg + il];
    }
    ++r;
    n_done = n;
    const int n_next = mode_of(r, s + 1);
    F_MARK(10);
    // the resident CDF / T of mode n are complete; the peers' prefixes and totals are not rewritten
    // before the next step's barrier #1, and the new factor rows are visible cluster-wide since
    // barrier #2.  Uniform sampling has no table (no barriers #2, #3): a cluster barrier orders the
    // peers' reads of this CTA's partials before the next step's gather rewrites them, and makes the
    // new factor rows visible to the next batch's SKR rows.
    if (p.strategy == 0) cluster.sync();
    else __syncthreads();
    F_MARK(11);
    sdbg = (p.dbg && q == 0 && s == 1) ? p.dbg : nullptr;
    if (s + 1 < p.nsteps) sample_own(n_next, r);
    sdbg = nullptr;
    F_MARK(12);
    n = n_next;
  }
  // no CTA may exit while a peer still reads its shared memory over DSMEM (the last step's CDF
  // assembly reads every peer's prefixes after barrier #3 and ends with a CTA-local barrier only)
  cluster.sync();
  if (q == 0 && tid == 0) {
    *p.iter = r;
    *p.last_mode = n_done;
  }
}

// one chain: the whole call in one cluster
template <typename T, int ROWS>
__global__ void __launch_bounds__(kFThreads, 1) k_sweep_fused(FusedParams<T> p) {
  fused_body<T, ROWS>(p);
}

// many independent chains: cluster c runs the call of chain c with its own
// parameters (ps[c]: factors, tables, accumulators, seed, ...; one geometry for all)
template <typename T, int ROWS>
__global__ void __launch_bounds__(kFThreads, 1) k_sweep_fused_multi(const FusedParams<T>* ps, int cu) {
  __shared__ __align__(16) FusedParams<T> sp;
  const FusedParams<T>* src = ps + blockIdx.x / cu;
  constexpr int W = (int)(sizeof(FusedParams<T>) / sizeof(int));
  static_assert(sizeof(FusedParams<T>) % sizeof(int) == 0, "param copy");
  for (int i = threadIdx.x; i < W; i += blockDim.x)
    reinterpret_cast<int*>(&sp)[i] = reinterpret_cast<const int*>(src)[i];
  __syncthreads();
  fused_body<T, ROWS>(sp);
}

}  // namespace cps
