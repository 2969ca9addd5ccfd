// wide.cuh -- the single-GPU wide path after the gather kernel (k_gather_update[_tc]), one step =
//
//   k_gather_update[_tc]  (a4-a6)  chunk partials of M = X_F diag(w) Z_F            (all SMs)
//   k_update_wide         (a6-a8)  M = sum_c M_c (chunk order), G = A Gamma - M, fixed / adaptive
//                    + (a1)        update; partial fp64 Grams (leverage) or row norms (Euclidean) of
//                                  the new rows; the LAST cluster sums the cluster partials and its
//                                  rank 0 inverts the Gram by the symmetric sweep -> W, |S| (the
//                                  R-pivot chain is inherently serial: one CTA) while every other CTA
//                                  waits (one resident wave, cooperative launch); then every CTA
//                                  scores and quantises its own rows, the LAST CTA scans -> CDF, T
//                                                                                     (all SMs)
//   k_sample_wide         (a2-a4)  the next batch: draws, SKR rows, weighted rows / tcgen05 images,
//                                  Gamma = Z_F^T diag(w) Z_F (clusters of 8, last cluster sums)  (all SMs)
//
// Citations: PAPER.md:<lines> (<label>); R<k> = DESIGN.md readings.
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cps {

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define WMARK(cond, slot)                                   \
  do {                                                      \
    if (p.dbg && (cond) && threadIdx.x == 0) p.dbg[slot] = gtimer(); \
  } while (0)

constexpr int kUWRows = 16;     // rows of A^(n) per k_update_wide CTA (divides the 128-row tiles)
constexpr int kWThreads = 256;
constexpr int kSWFibers = 32;   // fibers per k_sample_wide CTA
constexpr int kSWCluster = 8;
constexpr int kUWCluster = 8;   // k_update_wide CTAs per cluster (table partials summed over DSMEM)

// ---- replicas exchanging M over peer memory (CP_FLAG_P2P, NVLink / NVSwitch) ----------------------------
// Every rank owns a symmetric buffer: 64-bit flags (ready epoch at word 0; done[r] at word 16 + 16 r, each
// on its own 128-byte line, written by reader r into the owner's buffer) and, from byte kP2PHead, two parity
// copies of its chunk sum of M.  Exchange e (a device-side epoch, advanced in lockstep on every rank):
// the chunk-sum kernel waits until every reader has finished epoch e - 2 of this parity, writes the sum,
// and its last CTA publishes ready = e (release, system scope); k_update_wide waits for every peer's
// ready >= e (acquire, system scope), sums the P copies in rank order straight from peer memory (the
// collective fused into its consumer: bitwise identical M on every rank), and its last CTA writes
// done[rank] = e into every peer's buffer.
constexpr int kP2PHead = 4096;
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__host__ __device__ inline unsigned long long* p2p_done_flag(void* buf, int reader) {
  return reinterpret_cast<unsigned long long*>(buf) + 16 + 16 * reader;
}

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
  double* W;          // out (last CTA): leverage: the swept inverse W [R][R]; Euclidean: W[0] = ||A||_F^2
  int* tstat;         // out (last CTA): [0] rank |S| (leverage), [1] bad bits (2 degenerate, 8 non-finite)
  unsigned* cnt;      // cluster arrival counter (zero between launches)
  unsigned* flag;     // W-ready epoch: incremented once per launch by the sweeping CTA (never reset)
  unsigned* cnt2;     // CTA arrival counter of the scores (zero between launches)
  unsigned long long* qbuf;  // [I_n] quantised weights
  double* p_out;      // table: probabilities, CDF, T, status
  uint64_t* cdf;
  uint64_t* Tout;
  int* status;
  int64_t qch;        // last CTA's scan: q entries staged per round
  int table_only;     // 1: no step; take over the staged rows fstage (if *chg) and rebuild the table
  int update_only;    // 1: the step of rows [0, In) of a row block (A, S, Gout offset by the caller), no table
  const T* fstage;
  const int* chg;
  long long* dbg;
  // CP_FLAG_P2P (npeer > 0): M = sum over the peers' symmetric buffers (rank order) instead of Mpart
  int npeer, rank;
  void* peer[kMaxStrata];
  int64_t p2p_msz;                  // elements of one parity copy
  unsigned long long* p2p_epoch;    // device epoch of the last completed exchange
  unsigned* p2p_cnt;                // CTA arrivals after the peer reads (zero between launches)
};

// cp_sgd_steps_host (wide path): every mode in one launch (blockIdx.y = mode): chg[k] |= 1 when staged host factor k differs bitwise
template <typename T>
struct TakeAll {
  const T* fstage[kMaxOrder];
  const T* A[kMaxOrder];
  int64_t n[kMaxOrder];
};
template <typename T>
__global__ void k_take_compare_all(TakeAll<T> a, int* chg) {
  const int k = blockIdx.y;
  bool d = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.n[k]; e += (int64_t)gridDim.x * blockDim.x) {
    if constexpr (sizeof(T) == 8) d |= __double_as_longlong(a.fstage[k][e]) != __double_as_longlong(a.A[k][e]);
    else d |= __float_as_uint(a.fstage[k][e]) != __float_as_uint(a.A[k][e]);
  }
  if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(chg + k, 1);
}

// (a6-a8) + (a1) up to the inverse: grid = ceil(I_n / kUWRows); dynamic shared memory = the step's
// working set, or the last CTA's sweep workspace (Gram, sweep buffers), whichever is larger
__host__ __device__ inline size_t uw_sweep_ws_bytes(int R) {  // Gram + sweep buffers + swept flags
  return sizeof(double) * ((size_t)R * (R + 1) + kSweepBuf + kMaxRank) + sizeof(int) * kMaxRank + 64;
}
// dynamic shared memory: [step area: A, S, M rows, Gamma, Gram partial] [ext area: the last
// cluster's Gram slice + sweep workspace | W + score partials | the scan's q staging]
__host__ __device__ inline size_t uw_step_bytes(int R, size_t esz) {
  return ((esz * (3 * (size_t)kUWRows * (R + 1) + (size_t)R * R) + 15) / 16) * 16 +
         (sizeof(double) * (size_t)(R * (R + 1) / 2) + 15) / 16 * 16;
}
__host__ __device__ inline size_t uw_ext_bytes(int R, int64_t qch) {
  const size_t tail = (uw_sweep_ws_bytes(R) + 15) / 16 * 16 +
                      sizeof(double) * (size_t)((R * (R + 1) / 2 + kUWCluster - 1) / kUWCluster);
  const size_t sc = sizeof(double) * ((size_t)R * ut_rd(R) + (size_t)kUWRows * ut_rd(R) + (size_t)kUWRows * ((R + 3) / 4)) + 64;
  const size_t qs = sizeof(unsigned long long) * (size_t)qch;
  size_t m = tail > sc ? tail : sc;
  return m > qs ? m : qs;
}
__host__ __device__ inline size_t uw_smem_bytes(int R, size_t esz, int64_t qch) {
  return uw_step_bytes(R, esz) + uw_ext_bytes(R, qch);
}

// The last k_update_wide cluster to finish: the Gram of the new A^(n) as the cluster-ordered sum of
// the cluster partials (each CTA sums a slice of the pairs, every load of a pair in flight at
// once, and stores it into rank 0's Gram over DSMEM), then rank 0 inverts it by the symmetric sweep on the
// numerically full-rank pivot set (R4(b)) -> W, |S| in global memory.  Euclidean: ||A||_F^2.
// (Def. 2.3 / eq:lev, reading R4.)
template <typename T>
__device__ void uw_table_tail(const UWParams<T>& p, unsigned char* sm, const cooperative_groups::cluster_group& cluster) {
  const int tid = threadIdx.x, lane = tid & 31, R = p.R, RS = R + 1, P = R * (R + 1) / 2;
  const int CU = (int)cluster.num_blocks(), q = (int)cluster.block_rank(), ncl = (int)(gridDim.x / CU);
  __shared__ int s_bad;
  __shared__ double s_tol;
  if (p.strategy == 1 || p.strategy == 3) {
    double* Gm = reinterpret_cast<double*>(sm);
    double* rowbuf = Gm + R * RS;
    double* diag = rowbuf + kSweepBuf;
    int* swept = reinterpret_cast<int*>(diag + kMaxRank);
    // each CTA of the cluster sums a slice of the pairs and stores it straight into rank 0's Gram
    // (DSMEM stores), one cluster barrier
    double* Gm0 = cluster.map_shared_rank(Gm, 0);
    const int per = (P + CU - 1) / CU;
    for (int pair = q * per + tid; pair < min(P, (q + 1) * per); pair += kWThreads) {
      double v[16], s = 0.0;
      for (int c0 = 0; c0 < ncl; c0 += 16) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {  // clamped unconditional loads, then masked (no branch per load)
          const double t = __ldcg(p.gpart + (int64_t)(c0 + k < ncl ? c0 + k : ncl - 1) * P + pair);
          v[k] = (c0 + k < ncl) ? t : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) s += v[k];  // cluster order; zeros past ncl are exact
      }
      int r1 = 0, rem = pair;
      while (rem >= R - r1) { rem -= R - r1; ++r1; }
      Gm0[r1 * RS + r1 + rem] = s;
      Gm0[(r1 + rem) * RS + r1] = s;
    }
    cluster.sync();  // rank 0's Gram complete
    if (q != 0) return;
    if (tid == 0) s_bad = 0;
    WMARK(true, 313);
    if (tid < 32) {
      double d0 = 0.0;
      bool fin = true;
      for (int j = lane; j < R; j += 32) {
        const double d = Gm[j * RS + j];
        d0 = fmax(d0, d);
        fin = fin && (d == d) && d < 1.7e308;
      }
      __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
      if (lane == 0) {
        s_bad = __all_sync(0xffffffffu, fin) ? 0 : 8;
        s_tol = (double)(p.In > R ? p.In : R) * 2.220446049250313e-16 * d0;
      }
      if (lane != 0) __all_sync(0xffffffffu, fin);
    }
    __syncthreads();
    constexpr int EPT = (kMaxRank * kMaxRank + kWThreads - 1) / kWThreads;
    const int rank = (p.In < 2 * R) ? cta_sweep_inverse_pivoted<EPT>(Gm, R, s_tol, rowbuf, swept, diag)
                                    : grp_sweep_dispatch(Gm, R, s_tol, rowbuf, swept);
    WMARK(true, 314);
    for (int e = tid; e < R * R; e += kWThreads) p.W[e] = Gm[(e / R) * RS + e % R];
    if (tid == 0) {
      p.tstat[0] = rank;
      p.tstat[1] = s_bad | (rank == 0 ? 2 : 0);
      *p.cnt = 0u;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicAdd(p.flag, 1u);  // W ready (release: the fence above)
  } else {  // Euclidean
    if (q == 0 && tid == 0) {
      double fro = 0.0;
      for (int c = 0; c < ncl; ++c) fro += __ldcg(p.gpart + c);
      int bad = 0;
      if (!(fro == fro) || fro > 1.7e308) bad = 8;
      else if (!(fro > 0.0)) bad = 2;
      p.W[0] = fro;
      p.tstat[0] = 0;
      p.tstat[1] = bad;
      *p.cnt = 0u;
      __threadfence();
      atomicAdd(p.flag, 1u);
    }
  }
}

// (a1) the rows [r0, r0 + nr) of the new table: l_i = a_i^T W a_i / |S| (leverage) or
// ||a_i||^2 / ||A||_F^2 (Euclidean), quantised to the sampling contract's 2^-32 fixed point
// (Def. 2.3); then the last CTA to finish scans q -> CDF, T, status.
// Task (row il, column group cg) accumulates (A W)_{i, 4cg..4cg+3} over k in order and dots it
// with a_{i, 4cg..}; the nb4 partials of a row are summed in cg order.
template <typename T>
__device__ void uw_scores(const UWParams<T>& p, const T* sA, unsigned char* ext, int64_t r0, int nr) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int R = p.R, RS = R + 1, RD = ut_rd(R), nb4 = (R + 3) >> 2;
  const bool lev = (p.strategy == 1 || p.strategy == 3);
  __shared__ double s_p[kUWRows];
  __shared__ int s_last;
  __shared__ unsigned long long s_wtot[kWThreads / 32];
  __shared__ unsigned long long s_carry;
  if (lev) {
    double* Wd = reinterpret_cast<double*>(ext);  // [R][RD]
    double* Ad = Wd + R * RD;                     // [kUWRows][RD] fp64 copy of the new rows
    double* part = Ad + kUWRows * RD;             // [kUWRows][nb4]
    for (int e = tid; e < R * R; e += kWThreads) cp_async_small<8>(Wd + (e / R) * RD + e % R, p.W + e, 8);
    cp_async_commit();
    for (int e = tid; e < R * (RD - R); e += kWThreads) Wd[(e / (RD - R)) * RD + R + e % (RD - R)] = 0.0;
    for (int e = tid; e < kUWRows * RD; e += kWThreads) {
      const int il = e / RD, c = e % RD;
      Ad[e] = (il < nr && c < R) ? (double)sA[il * RS + c] : 0.0;
    }
    const int rank = __ldcg(p.tstat);
    cp_async_wait<0>();
    __syncthreads();
    // task = 2 rows x 4 columns: per k two row values, two 16-byte W loads, eight DFMA
    const int nrp = (nr + 1) >> 1;
    for (int t = tid; t < nrp * nb4; t += kWThreads) {
      const int il = 2 * (t / nb4), cg = t % nb4;
      const double* a0 = Ad + il * RD;
      const double* a1 = a0 + RD;  // row il + 1 (zeros past nr)
      double acc0[4] = {0.0, 0.0, 0.0, 0.0}, acc1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
      for (int k = 0; k < R; ++k) {
        const double x0 = a0[k], x1 = a1[k];
        const double2 w0 = *reinterpret_cast<const double2*>(Wd + k * RD + 4 * cg);
        const double2 w1 = *reinterpret_cast<const double2*>(Wd + k * RD + 4 * cg + 2);
        acc0[0] = fma(x0, w0.x, acc0[0]);
        acc0[1] = fma(x0, w0.y, acc0[1]);
        acc0[2] = fma(x0, w1.x, acc0[2]);
        acc0[3] = fma(x0, w1.y, acc0[3]);
        acc1[0] = fma(x1, w0.x, acc1[0]);
        acc1[1] = fma(x1, w0.y, acc1[1]);
        acc1[2] = fma(x1, w1.x, acc1[2]);
        acc1[3] = fma(x1, w1.y, acc1[3]);
      }
      part[il * nb4 + cg] = acc0[0] * a0[4 * cg] + acc0[1] * a0[4 * cg + 1] + acc0[2] * a0[4 * cg + 2] + acc0[3] * a0[4 * cg + 3];
      if (il + 1 < kUWRows)
        part[(il + 1) * nb4 + cg] =
            acc1[0] * a1[4 * cg] + acc1[1] * a1[4 * cg + 1] + acc1[2] * a1[4 * cg + 2] + acc1[3] * a1[4 * cg + 3];
    }
    __syncthreads();
    if (tid < nr) {
      double l = 0.0;
      for (int cg = 0; cg < nb4; ++cg) l += part[tid * nb4 + cg];
      s_p[tid] = rank > 0 ? fmax(l, 0.0) / (double)rank : 0.0;
    }
  } else if (tid < nr) {
    const double fro = __ldcg(p.W);
    s_p[tid] = fro > 0.0 ? __ldcg(p.rownorm + r0 + tid) / fro : 0.0;
  }
  __syncthreads();
  if (tid < nr) {
    const double pv = s_p[tid];
    unsigned long long qv = 0;
    if (!(pv == pv) || pv > 2.0) {
      atomicOr(p.tstat + 1, 8);
    } else if (pv > 0.0) {
      const double s = rint(pv * 4294967296.0);
      qv = (s < 1.0) ? 1ull : (unsigned long long)s;
    }
    p.p_out[r0 + tid] = pv;
    p.qbuf[r0 + tid] = qv;
  }
  // the last CTA: CDF = inclusive integer prefix of q over all rows (exact in any order), T, status
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (atomicAdd(p.cnt2, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t In = p.In;
  unsigned long long* qs = reinterpret_cast<unsigned long long*>(ext);
  if (tid == 0) s_carry = 0;
  for (int64_t c0 = 0; c0 < In; c0 += p.qch) {
    const int64_t n = cmin64(p.qch, In - c0);
    __syncthreads();
    for (int64_t i = tid; i < n; i += kWThreads) cp_async_small<8>(qs + i, p.qbuf + c0 + i, 8);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    const int64_t seg = (n + kWThreads - 1) / kWThreads;
    const int64_t a0 = cmin64((int64_t)tid * seg, n), a1 = cmin64(a0 + seg, n);
    unsigned long long local = 0;
    for (int64_t i = a0; i < a1; ++i) local += qs[i];
    unsigned long long incl = local;
    __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) s_wtot[wid] = incl;
    __syncthreads();
    unsigned long long pre = s_carry + incl - local;
    for (int w = 0; w < wid; ++w) pre += s_wtot[w];
    for (int64_t i = a0; i < a1; ++i) {
      pre += qs[i];
      p.cdf[c0 + i] = pre;
    }
    __syncthreads();
    if (tid == kWThreads - 1) s_carry = pre;  // the last thread's inclusive prefix = the running total
    __syncthreads();
  }
  if (tid == 0) {
    const unsigned long long total = s_carry;
    *p.Tout = total;
    const int bad = __ldcg(p.tstat + 1);
    int st = 0;
    if (bad & 8) st = -8;
    else if ((bad & 2) || total == 0) st = -3;
    if (st != 0) atomicCAS(p.status, 0, st);
    *p.cnt2 = 0u;
  }
}

template <typename T>
__global__ void __launch_bounds__(kWThreads) k_update_wide(UWParams<T> p) {
  constexpr int UR = kUWRows, TI = 128;
  const int R = p.R, RS = R + 1, tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * UR;
  const int nr = (int)cmax64(0, cmin64(UR, p.In - r0));  // 0 for the CTAs rounding the grid up
  WMARK(blockIdx.x == 0, 310);
  pdl_wait();  // partial tiles and Gamma come from the previous kernels
  __shared__ unsigned s_epoch0;
  if (tid == 0) s_epoch0 = *reinterpret_cast<volatile unsigned*>(p.flag);  // before any arrival below
  extern __shared__ __align__(16) unsigned char uw_sm[];
  T* sA = reinterpret_cast<T*>(uw_sm);  // [UR][R+1] each
  T* sS = sA + UR * RS;
  T* sM = sS + UR * RS;
  T* sG = sM + UR * RS;                 // [R][R]
  double* sgp = reinterpret_cast<double*>(uw_sm + ((sizeof(T) * (3 * UR * RS + R * R) + 15) / 16) * 16);  // [P]
  __shared__ double sred[kWThreads / 32];
  cooperative_groups::cluster_group cluster = cooperative_groups::this_cluster();
  const int nb4 = (R + 3) >> 2;
  if (p.table_only) {
    // cp_sgd_steps_host: the staged host rows replace the factor when any of them differs (the
    // flag set by k_take_compare_all); an unchanged factor keeps its table: every CTA leaves here
    if (__ldcg(p.chg) == 0) return;
    for (int e = tid; e < nr * R; e += kWThreads) {
      const int il = e / R, c = e % R;
      const T v = p.fstage[(r0 + il) * R + c];
      sA[il * RS + c] = v;
      p.A[(r0 + il) * R + c] = v;
    }
    __syncthreads();
  } else {
    // rows of A and S, Gamma: every request in flight at once
    for (int e = tid; e < nr * R; e += kWThreads) {
      const int il = e / R, c = e % R;
      cp_async_small<sizeof(T)>(sA + il * RS + c, p.A + (r0 + il) * R + c, sizeof(T));
      if (p.rule == 1) cp_async_small<sizeof(T)>(sS + il * RS + c, p.S + (r0 + il) * R + c, sizeof(T));
    }
    for (int e = tid; e < R * R; e += kWThreads) cp_async_small<sizeof(T)>(sG + e, p.Gam + e, sizeof(T));
    cp_async_commit();
    __shared__ unsigned long long s_pe;
    if (p.npeer > 0) {  // peer-memory exchange: every peer's copy of epoch e published
      if (tid == 0) {
        const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(p.p2p_epoch) + 1;
        s_pe = e;
        for (int g = 0; g < p.npeer; ++g)
          while (ld_acquire_sys_u64(reinterpret_cast<const unsigned long long*>(p.peer[g])) < e) {
          }
      }
      __syncthreads();
    }
    // M = sum of the chunk partials, in chunk order (16-byte vectors of VW consecutive rows); P2P: the
    // sum of the peers' chunk sums, in rank order, loaded from their memory
    if (p.npeer > 0) {
      constexpr int VW = 16 / (int)sizeof(T);
      using V = typename Vec<T>::type;
      const int64_t tile = r0 / TI, lr0 = r0 % TI;
      const int ng = (nr + VW - 1) / VW;
      const int64_t off = (int64_t)(s_pe & 1ull) * p.p2p_msz + tile * R * TI + lr0;
      for (int t = tid; t < R * ng; t += kWThreads) {
        const int r = t / ng, gq = t % ng;
        T acc[VW];
  #pragma unroll
        for (int w = 0; w < VW; ++w) acc[w] = T(0);
        V ld[kMaxStrata];
  #pragma unroll
        for (int g = 0; g < kMaxStrata; ++g)  // every peer's load in flight, then summed in rank order
          if (g < p.npeer)
            ld[g] = __ldcg(reinterpret_cast<const V*>(reinterpret_cast<const T*>(
                                                          reinterpret_cast<const unsigned char*>(p.peer[g]) + kP2PHead) +
                                                      off + (int64_t)r * TI + gq * VW));
  #pragma unroll
        for (int g = 0; g < kMaxStrata; ++g)
          if (g < p.npeer) {
            const T* x = reinterpret_cast<const T*>(&ld[g]);
  #pragma unroll
            for (int w = 0; w < VW; ++w) acc[w] += x[w];
          }
  #pragma unroll
        for (int w = 0; w < VW; ++w)
          if (gq * VW + w < nr) sM[(gq * VW + w) * RS + r] = acc[w];
      }
    } else {
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
    if (p.npeer > 0 && tid == 0) {  // this CTA's peer reads are complete; the last CTA signals every peer
      if (atomicAdd(p.p2p_cnt, 1u) == gridDim.x - 1) {
        *p.p2p_cnt = 0;
        for (int g = 0; g < p.npeer; ++g) st_release_sys_u64(p2p_done_flag(p.peer[g], p.rank), s_pe);
        *reinterpret_cast<volatile unsigned long long*>(p.p2p_epoch) = s_pe;  // every CTA read it at its start
      }
    }
    if (p.rule == 2) {
      // sampled least squares (eq:lsq_krp; R25): W = Gamma^+ in fp64 by the
      // natural-order sweep (tol R eps max diag) in every CTA, then this CTA's rows A = M W (into
      // sS, unused by this rule) before M is overwritten by G below
      double* Gm = reinterpret_cast<double*>(uw_sm + uw_step_bytes(R, sizeof(T)));
      double* rowbuf = Gm + R * RS;
      int* swept = reinterpret_cast<int*>(rowbuf + kSweepBuf + kMaxRank);
      __shared__ double s_tol_als;
      for (int e = tid; e < R * R; e += kWThreads) Gm[(e / R) * RS + e % R] = (double)sG[e];
      __syncthreads();
      if (tid < 32) {
        double d0 = 0.0;
        for (int j = tid; j < R; j += 32) d0 = fmax(d0, Gm[j * RS + j]);
        __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
  #pragma unroll
        for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
        if (tid == 0) s_tol_als = (double)R * 2.220446049250313e-16 * d0;
      }
      __syncthreads();
      grp_sweep_dispatch(Gm, R, s_tol_als, rowbuf, swept);
      for (int e = tid; e < nr * R; e += kWThreads) {
        const int il = e / R, r = e % R;
        double an = 0.0;
        for (int c = 0; c < R; ++c) an = fma((double)sM[il * RS + c], Gm[c * RS + r], an);
        sS[il * RS + r] = (T)an;
      }
      __syncthreads();
    }
    // G = A Gamma - M (each task owns its 4 x 4 block of M -> G in place)
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
        for (int a = 0; a < 4; ++a) {
          const T t = sA[(a0 + a) * RS + k];  // rows < kUWRows: inside the buffer; load, then select
          x[a] = (a0 + a < nr) ? t : T(0);
        }
  #pragma unroll
        for (int c = 0; c < 4; ++c) {
          const T t = sG[k * R + (q0 + c < R ? q0 + c : R - 1)];
          y[c] = (q0 + c < R) ? t : T(0);
        }
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
      if (p.rule == 2) {
        an = sS[il * RS + r];
      } else if (p.rule == 0) {
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
  }
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
          const T tx = sA[il * RS + (4 * bi + a < R ? 4 * bi + a : R - 1)];  // clamped, then select
          const T ty = sA[il * RS + (4 * bj + a < R ? 4 * bj + a : R - 1)];
          x[a] = 4 * bi + a < R ? (double)tx : 0.0;
          y[a] = 4 * bj + a < R ? (double)ty : 0.0;
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
    __threadfence();
    cluster.sync();
  } else if (p.strategy == 2 || p.strategy == 4) {  // Euclidean: row norms + the CTA's partial ||A||^2
    double acc = 0.0;
    for (int il = tid; il < nr; il += kWThreads) {
      double rs = 0.0;
      for (int c = 0; c < R; ++c) rs += (double)sA[il * RS + c] * (double)sA[il * RS + c];
      p.rownorm[r0 + il] = rs;
      acc += rs;
    }
    __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
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
      __threadfence();
    }
    cluster.sync();
  }
  WMARK(blockIdx.x == 0, 311);
  if (p.strategy == 0 || p.update_only) return;  // uniform tables are constant; row blocks: no table here
  unsigned char* ext = uw_sm + uw_step_bytes(R, sizeof(T));
  {  // the last cluster: the inverse (leverage) / the Frobenius norm (Euclidean)
    __shared__ int s_last;
    const int ncl = (int)(gridDim.x / cluster.num_blocks());
    if (cluster.block_rank() == 0 && tid == 0) s_last = (atomicAdd(p.cnt, 1u) == (unsigned)(ncl - 1));
    cluster.sync();
    const bool last = *cluster.map_shared_rank(&s_last, 0) != 0;
    cluster.sync();  // rank 0's flag read by every peer
    if (last) {
      __threadfence();
      WMARK(cluster.block_rank() == 0, 312);
      uw_table_tail<T>(p, ext, cluster);
      WMARK(cluster.block_rank() == 0, 315);
    }
  }
  // every CTA (all resident: one wave, cooperative launch) waits for W, then scores its own rows
  if (tid == 0) {
    unsigned f;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(f) : "l"(p.flag) : "memory");
      if (f == s_epoch0) __nanosleep(128);
    } while (f == s_epoch0);
  }
  __syncthreads();
  pdl_trigger();  // W is ready: the sampler may start its launch
  WMARK(blockIdx.x == 0, 316);
  uw_scores<T>(p, sA, ext, r0, nr);
  WMARK(blockIdx.x == 0, 317);
}

// ------------------------------------------------------------------------------------------
// (a2-a4) the next batch: clusters of kSWCluster CTAs of kSWFibers fibers each
// ------------------------------------------------------------------------------------------
struct SWParams {
  long long* dbg;
  SampleParams sp;          // batch of mode sp.n at the iteration in *sp.iter; zwp / gam_next set
  void* gcl;                // [clusters][R][R] cluster partials of Gamma (T)
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
__global__ void __launch_bounds__(kWThreads, 1) k_sample_wide(SWParams P) {
  pdl_wait();  // the tables and factors come from the previous kernel
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
  // block windows, stratified draws and slab shards (owned fibers, local offsets): the general draw_rows; the
  // single-GPU row-wise case below draws the N-1 positions of a fiber in parallel
  if (sp.strategy == 3 || sp.strategy == 4 || sp.strat_P > 1 || sp.ldims[N - 1] != sp.dims[N - 1] || sp.lo_last != 0) {
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
        const uint64_t cprev = c[i > 0 ? i - 1 : 0];  // unconditional load, then select
        qk = c[i] - (i > 0 ? cprev : 0ull);
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
    // ascending modes (Alg. 1), two per round: both modes' loads are issued before the products
    for (int pos = 0; pos < NP; pos += 2) {
      const int k0 = pos < sp.n ? pos : pos + 1, k1 = pos + 1 < sp.n ? pos + 1 : pos + 2;
      const bool two = pos + 1 < NP;
      const T* F0 = reinterpret_cast<const T*>(sp.factors[k0]);
      const T* F1 = reinterpret_cast<const T*>(sp.factors[two ? k1 : k0]);
      T f0[U], f1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool on = z[u] != T(0);
        f0[u] = on ? F0[(int64_t)sidx[lbu[u] * NP + pos] * R + ru[u]] : T(0);
        f1[u] = (on && two) ? F1[(int64_t)sidx[lbu[u] * NP + pos + 1] * R + ru[u]] : T(0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        z[u] = z[u] * f0[u];
        if (two) z[u] = z[u] * f1[u];
      }
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
    SWM(8);
    __syncthreads();
    SWM(9);
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
  // the cross-cluster sum of the partials (cluster order) is done by idle lanes of the next
  // kernel, the gather (gu_gamma_sum): it does not read Gamma, k_update_wide after it does
  cluster.sync();  // peers are done reading this CTA's partial
  SWM(7);
  if (P.dbg && tid == 0 && blockIdx.x < 480) {
    long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    P.dbg[2048 + 2 * blockIdx.x] = gt0;
    P.dbg[2049 + 2 * blockIdx.x] = gt1;
  }
}

}  // namespace cps
