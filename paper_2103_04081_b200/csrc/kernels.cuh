// kernels.cuh -- sm_100a kernels of the sampled SGD step (arXiv 2103.04081, BrawsCPD/AdawsCPD).
//
//   k_table    (a1)  per-mode importance table: fp64 Gram -> pivoted Cholesky -> leverage, or
//                    row norms (Euclidean), or uniform; fixed-point quantisation; integer scan
//   k_sample   (a2,a3) Philox draws -> upper_bound on the integer CDF (staged in shared memory)
//                    -> idx and the exact fp64 weights omega
//   k_gather   (a4,a5,a6) SKR rows (Alg. 1) x fiber gather (Alg. 5) -> per-chunk partial
//                    M = X_F diag(omega) Z_F and Gamma = Z_F^T diag(omega) Z_F
//   k_update   (a6,a7,a8) deterministic chunk reduction, G = A Gamma - M, fixed / adaptive update
//   k_fit             fit = 1 - ||X - [[A]]|| / ||X|| (per-block fp64 partials)
//   k_transpose       mode-major copies X_(n)^T (layout option)
//
// Citations: PAPER.md:<lines> (<label>); R<k> = DESIGN.md readings.
#pragma once
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "philox.cuh"

namespace cps {

constexpr int kMaxOrder = 16;
constexpr int kMaxRank = 64;
constexpr int kMaxStrata = 16;
// debug timers (CPSGD_DEBUG_TIMERS): 4096 kernel-specific slots, then k_sweep_wide's per-CTA marks
// [8 iterations][160 CTAs][32 slots]
constexpr int kDbgEntries = 4096 + 8 * 160 * 32;  // slabs of the stratified sampler (ranks of one box)
constexpr int kSweepBuf = 5 * kMaxRank;  // doubles of pivot-row buffer the sweep inverses need

// ------------------------------------------------------------------------------------------
// Parameters (passed by value; < 1 KB)
// ------------------------------------------------------------------------------------------
struct SampleParams {
  int N, n, strategy, R;
  int64_t B;                       // nominal batch
  int64_t dims[kMaxOrder];         // global dims
  int32_t window[kMaxOrder];       // per remaining position (block strategies), clamped to I_k
  const uint64_t* cdf[kMaxOrder];  // inclusive CDF per mode (device)
  const uint64_t* Ttot;            // [N] totals (device)
  uint64_t seed;
  const uint64_t* iter;            // device pointer to the iteration counter r
  uint64_t iter_add;               // draws use r + iter_add
  int32_t* idx;                    // out [B_max][N-1]
  double* w;                       // out [B_max]
  int64_t* beff;                   // out (device scalar)
  int64_t bmax;                    // rows the launch covers
  int stage_smem;                  // stage the CDFs of the N-1 sampled modes in shared memory
  // prefetch for k_gather (optional): unweighted SKR rows and fiber offsets of mode n
  const void* factors[kMaxOrder];
  void* zrow;                      // T [B_max][R] or NULL
  int64_t* fbase;                  // [B_max] element offset of fiber b in the gather's layout (-1: not owned)
  int64_t ldims[kMaxOrder];        // local dims (slab)
  int64_t lstride[kMaxOrder];
  int64_t lo_last;
  int mode_major;
  int64_t pitch;
  // wide path (k_gather_update): weighted padded SKR rows and Gamma of the batch (or NULL)
  void* zwp;                       // T [B_max][ceil8(R)]
  void* gam_next;                  // T [R][R]
  float* zimg;                     // tcgen05 path: 3xTF32 A-operand images of zw (or NULL)
  // stratified per-slab sampling (CP_FLAG_STRATIFIED; reading R26): strat_P > 1 strata, stratum g = batch
  // rows [off_g, off_g + B_g), B_g = B/P (+1 for g < B mod P), drawing the last mode from slab
  // [strat_lo[g], strat_lo[g + 1]) (modes n < N-1 only; 0 = off)
  int strat_P;
  int64_t strat_lo[kMaxStrata + 1];
};

// debug trace of the consumed batches and the states they lead to (cp_sgd_trace; persistent kernels
// k_sweep_wide and k_sweep_fused): per SGD iteration s of a launch, slot first + s (< cap) holds idx
// [bmax][N-1], w [bmax], the updated A^(n) [I_n][R], S^(n) [I_n][R] (adaptive rule), the new CDF of
// mode n [I_n] and meta {n, r, B_eff, 0}
struct TraceParams {
  unsigned char* base;
  int64_t stride, o_idx, o_w, o_A, o_S, o_cdf, o_meta;
  int64_t first, cap;
};

// byte offset of zh_r (part 0) / zl_r (part 1) of fiber b in the tcgen05 A-operand images
// (gupdate_tc.cuh): per stage of 32 fibers one 128-row x 128-byte tile (rows 0-63 zh, 64-127 zl),
// K-major with the 128-byte swizzle (16-byte chunk c of row m at chunk c ^ (m & 7))
__host__ __device__ __forceinline__ uint32_t zimg_off(int64_t b, int m) {
  const int kk = (int)(b & 31), rr = m & 7, c = (kk >> 2) & 7;
  return (uint32_t)((b >> 5) * 16384 + (m >> 3) * 1024 + rr * 128 + ((c ^ rr) << 4) + ((kk & 3) << 2));
}

template <typename T>
struct GatherParams {
  int N, n, R;
  int64_t ldims[kMaxOrder];    // local dims (last mode = slab length when sharded)
  int64_t lstride[kMaxOrder];  // first-index-fastest strides of the local tensor
  int64_t lo_last;             // slab begin on the last mode (0 if not sharded)
  const T* X;                  // native local tensor, or the mode-major copy of mode n
  int mode_major;              // 1: X is [J_n_local][pitch] (fiber-contiguous)
  int64_t pitch;               // row pitch of the mode-major copy (elements)
  const int64_t* fbase;        // [B_max] fiber offsets from the sampler (-1: not owned / padding)
  const T* zrow;               // [B_max][R] unweighted SKR rows from the sampler
  const double* w;             // [B_max]
  const int64_t* beff;         // device scalar
  int64_t TB;                  // fibers per chunk
  int64_t In_local;            // rows of M handled (local slab rows for the last mode)
  T* Mp;                       // out [chunks][R][In_local]
  T* Gp;                       // out [chunks][R][R]
};

template <typename T>
struct UpdateParams {
  int R;
  int64_t In_local;   // rows handled
  int64_t row0;       // global row of local row 0 (slab begin for the sharded mode)
  int nchunks;
  const T* Mp;        // [chunks][R][In_local] partials, or NULL when Msum is given
  const T* Gp;        // [chunks][R][R]
  const T* Msum;      // [R][In_local] reduced M (sharded path), or NULL
  const T* Gsum;      // [R][R] reduced Gamma, or NULL
  T* A;               // factor A^(n), row-major I_n x R (global rows)
  T* S;               // adaptive accumulator (same layout), NULL for the fixed rule
  T* Gout;            // last gradient (debug), row-major I_n x R (global rows)
  T* Gam_out;         // reduced Gamma (debug), R x R
  int rule;
  double alpha;       // fixed step (used when alpha_dev == NULL)
  const double* alpha_dev;
  double eta, b, eps;
  uint64_t* iter;     // incremented once per step (block 0), or NULL
};

// ------------------------------------------------------------------------------------------
// small helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ int64_t upper_bound_u64(const uint64_t* __restrict__ cdf, int64_t n, uint64_t r) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (cdf[mid] <= r) lo = mid + 1;
    else hi = mid;
  }
  return lo;  // #{i : cdf[i] <= r}
}

template <typename T>
struct Vec;
template <>
struct Vec<float> {
  using type = float4;
  static constexpr int W = 4;
};
template <>
struct Vec<double> {
  using type = double2;
  static constexpr int W = 2;
};

__host__ __device__ __forceinline__ int64_t cmin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t cmax64(int64_t a, int64_t b) { return a > b ? a : b; }

template <typename T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes) : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* dst, const void* src, int src_bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(d), "l"(src), "n"(BYTES), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// global -> shared copy of n 8-byte elements, every request in flight at once (one commit group);
// the caller waits (cp_async_wait<0>) and synchronises
__device__ __forceinline__ void cp_async_u64(uint64_t* dst, const uint64_t* src, int64_t n, int tid, int nth) {
  for (int64_t i = tid; i < n; i += nth) cp_async_small<8>(dst + i, src + i, 8);
  cp_async_commit();
}

// ==========================================================================================
// (a1) importance table of one mode -- single CTA of 1024 threads.
//   leverage : l_i = ||L^{-1} a_{i,piv}||^2 with A_piv^T A_piv = L L^T (pivoted Cholesky of the
//              fp64 Gram; Def. 2.3), p_i = l_i / rank (R4)
//   euclidean: p_i = ||A(i,:)||^2 / ||A||_F^2 (Def. 2.5)
//   uniform  : q_i = 1
//   q_i = p_i > 0 ? max(1, rint(p_i 2^32)) : 0; cdf = inclusive integer scan; T = cdf[I-1]
// status: 0 ok, -3 degenerate (T = 0), -8 non-finite.
// ==========================================================================================
constexpr int kTableThreads = 1024;

template <typename T>
__global__ void __launch_bounds__(kTableThreads) k_table(const T* __restrict__ A, int64_t I, int R, int strategy,
                                                         double* __restrict__ p_out, uint64_t* __restrict__ cdf,
                                                         uint64_t* __restrict__ Tout, int* __restrict__ status) {
  extern __shared__ double sm[];
  double* Gm = sm;                              // R x R
  double* red = Gm + kMaxRank * kMaxRank;       // max(kTableThreads, R(R+1)/2 * groups) scratch
  __shared__ int piv[kMaxRank];
  __shared__ int s_rank, s_stop, s_bad;
  __shared__ unsigned long long warp_tot[32];
  __shared__ double s_fro;
  const int tid = threadIdx.x;
  const bool lev = (strategy == 1 || strategy == 3);
  const bool euc = (strategy == 2 || strategy == 4);
  if (tid == 0) { s_bad = 0; s_rank = R; }

  if (lev) {
    // Gram in fp64: pairs (r1 <= r2); rows split over `groups` thread groups when the pairs
    // leave threads idle; partial sums reduced in a fixed order (deterministic).
    const int P = R * (R + 1) / 2;
    const int groups = max(1, kTableThreads / P);
    for (int e = tid; e < P * groups; e += kTableThreads) {
      const int pair = e % P, g = e / P;
      int r1 = 0, rem = pair;
      while (rem >= R - r1) { rem -= R - r1; ++r1; }
      const int r2 = r1 + rem;
      double s = 0.0;
      for (int64_t i = g; i < I; i += groups) s += (double)A[i * R + r1] * (double)A[i * R + r2];
      red[e] = s;
    }
    __syncthreads();
    for (int pair = tid; pair < P; pair += kTableThreads) {
      double s = 0.0;
      for (int g = 0; g < groups; ++g) s += red[g * P + pair];
      int r1 = 0, rem = pair;
      while (rem >= R - r1) { rem -= R - r1; ++r1; }
      const int r2 = r1 + rem;
      Gm[r1 * R + r2] = s;
      Gm[r2 * R + r1] = s;
    }
    __syncthreads();
    // pivoted Cholesky, right-looking, full symmetric storage; tolerance R4(b):
    // stop when the largest remaining Schur diagonal <= max(I,R) * eps * d0.
    if (tid < R) piv[tid] = tid;
    if (tid == 0) {
      double d0 = 0.0;
      for (int j = 0; j < R; ++j) d0 = fmax(d0, Gm[j * R + j]);
      red[0] = d0;
      s_stop = 0;
      if (!(d0 == d0) || d0 > 1.7e308) s_bad = 8;
    }
    __syncthreads();
    const double tol = (double)(I > R ? I : R) * 2.220446049250313e-16 * red[0];
    int k = 0;
    for (; k < R; ++k) {
      if (tid == 0) {
        int jm = k;
        double dm = Gm[k * R + k];
        for (int j = k + 1; j < R; ++j)
          if (Gm[j * R + j] > dm) { dm = Gm[j * R + j]; jm = j; }
        if (!(dm > tol)) {
          s_stop = 1;
        } else if (jm != k) {
          int t = piv[k]; piv[k] = piv[jm]; piv[jm] = t;
        }
        red[1] = (double)jm;
      }
      __syncthreads();
      if (s_stop) break;
      const int jm = (int)red[1];
      if (jm != k) {  // swap rows and columns k <-> jm of the full matrix
        for (int c = tid; c < R; c += kTableThreads) {
          double t = Gm[k * R + c]; Gm[k * R + c] = Gm[jm * R + c]; Gm[jm * R + c] = t;
        }
        __syncthreads();
        for (int rr = tid; rr < R; rr += kTableThreads) {
          double t = Gm[rr * R + k]; Gm[rr * R + k] = Gm[rr * R + jm]; Gm[rr * R + jm] = t;
        }
        __syncthreads();
      }
      const double lkk = sqrt(Gm[k * R + k]);
      __syncthreads();
      for (int i = k + 1 + tid; i < R; i += kTableThreads) Gm[i * R + k] = Gm[i * R + k] / lkk;
      if (tid == 0) Gm[k * R + k] = lkk;
      __syncthreads();
      const int m = R - k - 1;
      for (int e = tid; e < m * m; e += kTableThreads) {
        const int i = k + 1 + e / m, j = k + 1 + e % m;
        Gm[i * R + j] -= Gm[i * R + k] * Gm[j * R + k];
      }
      __syncthreads();
    }
    if (tid == 0) s_rank = k;
    __syncthreads();
  } else if (euc) {
    // ||A||_F^2 by a fixed-order tree reduction of per-thread row sums
    double s = 0.0;
    for (int64_t i = tid; i < I; i += kTableThreads) {
      double rs = 0.0;
      for (int r = 0; r < R; ++r) rs += (double)A[i * R + r] * (double)A[i * R + r];
      s += rs;
    }
    red[tid] = s;
    __syncthreads();
    for (int st = kTableThreads / 2; st > 0; st >>= 1) {
      if (tid < st) red[tid] += red[tid + st];
      __syncthreads();
    }
    if (tid == 0) s_fro = red[0];
    __syncthreads();
  }
  __syncthreads();
  const int rank = s_rank;
  const double fro = euc ? s_fro : 1.0;
  if (tid == 0 && euc && !(fro > 0.0)) s_bad |= (fro == fro) ? 2 : 8;
  if (tid == 0 && euc && fro > 1.7e308) s_bad |= 8;
  if (tid == 0 && lev && rank == 0) s_bad |= 2;
  __syncthreads();

  // per-row probabilities and quantisation; each thread owns a contiguous segment of rows
  const int64_t seg = (I + kTableThreads - 1) / kTableThreads;
  const int64_t i_beg = min((int64_t)tid * seg, I), i_end = min(i_beg + seg, I);
  unsigned long long local = 0;
  int bad = 0;
  for (int64_t i = i_beg; i < i_end; ++i) {
    double p;
    if (lev) {
      // forward substitution L y = a_{i,piv}
      double y[kMaxRank];
      double l = 0.0;
      for (int j = 0; j < rank; ++j) {
        double s = (double)A[i * R + piv[j]];
        for (int t = 0; t < j; ++t) s -= Gm[j * R + t] * y[t];
        y[j] = s / Gm[j * R + j];
        l += y[j] * y[j];
      }
      p = l / (double)rank;
    } else if (euc) {
      double rs = 0.0;
      for (int r = 0; r < R; ++r) rs += (double)A[i * R + r] * (double)A[i * R + r];
      p = fro > 0.0 ? rs / fro : 0.0;
    } else {
      p = 1.0 / (double)I;
    }
    uint64_t q;
    if (!lev && !euc) {
      q = 1;
    } else if (!(p == p) || p > 2.0) {
      bad = 1;
      q = 0;
    } else if (p > 0.0) {
      const double s = rint(p * 4294967296.0);
      q = (s < 1.0) ? 1ull : (uint64_t)s;
    } else {
      q = 0;
    }
    if (p_out) p_out[i] = p;
    cdf[i] = q;  // temporarily the count; scanned below
    local += q;
  }
  if (bad) atomicOr(&s_bad, 8);
  // block exclusive scan of the per-thread totals (integers: order-independent, exact)
  const int lane = tid & 31, wid = tid >> 5;
  unsigned long long incl = local;
  __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
  for (int o = 1; o < 32; o <<= 1) {
    unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    unsigned long long v = warp_tot[lane];
    __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    warp_tot[lane] = v;  // inclusive over warps
  }
  __syncthreads();
  unsigned long long run = (incl - local) + (wid > 0 ? warp_tot[wid - 1] : 0ull);
  for (int64_t i = i_beg; i < i_end; ++i) {
    run += cdf[i];
    cdf[i] = run;
  }
  if (tid == kTableThreads - 1) {
    const unsigned long long Ttot = run;
    *Tout = Ttot;
    int st = 0;
    if (s_bad & 8) st = -8;
    else if ((s_bad & 2) || Ttot == 0) st = -3;
    if (st != 0) atomicCAS(status, 0, st);
  }
}

// ==========================================================================================
// (a2, a3) sampler.  One thread per batch row.  Row-wise (eq:ik, Alg. 3): for position p of
// mode k: u = philox(b, purpose 0, slot p, r); r' = floor(u T_k / 2^64); i = #{cdf_k <= r'}.
// Block (eq:bik, Alg. 4, R2): per position one draw (x0 = 0, purpose 1) selects the row i*,
// window w = floor(i* / b_k) (identical to drawing from the window CDF); rows of the Cartesian
// product in index-map order.  Weights in the contract's exact fp64 order (no FMA possible:
// only products and quotients, written with explicit _rn intrinsics).
// ==========================================================================================
// stage the CDFs of the sampled modes (k != n) in shared memory; cdfp[k] -> smem or global
__device__ __forceinline__ void stage_cdfs(const SampleParams& p, uint64_t* s_cdf, const uint64_t** cdfp, int tid,
                                           int nthreads) {
  int64_t off = 0;
  for (int k = 0; k < p.N; ++k) {
    cdfp[k] = p.cdf[k];
    if (k == p.n || !p.stage_smem || p.strategy == 0) continue;
    cp_async_u64(s_cdf + off, p.cdf[k], p.dims[k], tid, nthreads);
    cdfp[k] = s_cdf + off;
    off += p.dims[k];
  }
  cp_async_wait<0>();
}

// rows [b0, b1) of the batch of mode p.n at iteration r: indices, exact weights, fiber offsets.
__device__ __forceinline__ void draw_rows(const SampleParams& p, const uint64_t* const* cdfp, uint64_t r_it,
                                          int64_t b0, int64_t b1, int tid, int nthreads,
                                          int32_t* sidx = nullptr /* shared [b1-b0][N-1] copy */,
                                          double* sw = nullptr /* shared [b1-b0] copy */) {
  const int N = p.N, n = p.n;
  const bool block = (p.strategy == 3 || p.strategy == 4);
  int32_t start[kMaxOrder], len[kMaxOrder];
  double wblk = 0.0;
  int64_t beff = p.B;
  if (block) {
    double prod = 1.0;
    beff = 1;
    int pos = 0;
    for (int k = 0; k < N; ++k) {
      if (k == n) continue;
      const int64_t bk = p.window[pos];
      const uint64_t Tk = p.Ttot[k];
      const uint64_t u = draw_word(p.seed, r_it, 0u, kPurposeWindow, (uint32_t)pos);
      const uint64_t rr = scale_draw(u, Tk);
      const uint64_t* c = cdfp[k];
      const int64_t istar = upper_bound_u64(c, p.dims[k], rr);   // == window draw (R6)
      const int64_t s0 = (istar / bk) * bk;
      const int64_t e0 = min(s0 + bk, p.dims[k]);
      const uint64_t cprev = c[s0 > 0 ? s0 - 1 : 0];  // unconditional load, then select
      const uint64_t Q = c[e0 - 1] - (s0 > 0 ? cprev : 0ull);
      start[pos] = (int32_t)s0;
      len[pos] = (int32_t)(e0 - s0);
      const double pt = __ddiv_rn((double)((uint64_t)p.dims[k] * Q), (double)Tk);
      prod = (pos == 0) ? pt : __dmul_rn(prod, pt);
      beff *= (e0 - s0);
      ++pos;
    }
    wblk = __ddiv_rn(1.0, prod);
  }
  if (b0 == 0 && tid == 0) *p.beff = beff;
  for (int64_t b = b0 + tid; b < b1; b += nthreads) {
    if (b >= beff) {
      if (p.fbase) p.fbase[b] = -1;
      if (sw) sw[b - b0] = 0.0;
      if (sidx)
        for (int q = 0; q < N - 1; ++q) sidx[(b - b0) * (N - 1) + q] = 0;
      continue;
    }
    int32_t* ib = p.idx + b * (N - 1);
    if (!block) {
      // stratified (R26): this row's stratum g and the slab's CDF base / mass (exact integers)
      const bool strat = p.strat_P > 1 && n != N - 1;
      int64_t Bw = p.B, slo = 0, shi = 0;
      uint64_t sbase = 0, smass = 0;
      if (strat) {
        const int64_t P = p.strat_P, q0 = p.B / P, rm = p.B % P;
        const int64_t g = b < rm * (q0 + 1) ? b / (q0 + 1) : rm + (b - rm * (q0 + 1)) / q0;
        Bw = q0 + (g < rm ? 1 : 0);
        slo = p.strat_lo[g];
        shi = p.strat_lo[g + 1];
        if (p.strategy == 0) {
          sbase = (uint64_t)slo;
          smass = (uint64_t)(shi - slo);
        } else {
          const uint64_t* c = cdfp[N - 1];
          const uint64_t cb = c[slo > 0 ? slo - 1 : 0];  // unconditional load, then select
          sbase = slo > 0 ? cb : 0ull;
          smass = c[shi - 1] - sbase;
        }
      }
      double prod = 1.0;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == n) continue;
        const bool sk = strat && k == N - 1;
        const uint64_t Tk = sk ? smass : (p.strategy == 0) ? (uint64_t)p.dims[k] : p.Ttot[k];
        const uint64_t u = draw_word(p.seed, r_it, (uint32_t)b, kPurposeRow, (uint32_t)pos);
        const uint64_t rr = (sk ? sbase : 0ull) + scale_draw(u, Tk);
        int64_t i;
        uint64_t qk;
        if (sk && smass == 0) {  // a zero-mass slab: no fiber of it can be drawn; the row carries w = 0
          i = slo;
          qk = 0;
        } else if (p.strategy == 0) {
          i = (int64_t)rr;
          qk = 1;
        } else {
          const uint64_t* c = cdfp[k];
          i = upper_bound_u64(c, p.dims[k], rr);
          const uint64_t cprev = c[i > 0 ? i - 1 : 0];  // unconditional load, then select
          qk = c[i] - (i > 0 ? cprev : 0ull);
        }
        ib[pos] = (int32_t)i;
        const double pt = qk == 0 ? 0.0 : __ddiv_rn((double)((uint64_t)p.dims[k] * qk), (double)Tk);
        prod = (pos == 0) ? pt : __dmul_rn(prod, pt);
        ++pos;
      }
      const double wv = prod == 0.0 ? 0.0 : __ddiv_rn(1.0, __dmul_rn((double)Bw, prod));
      p.w[b] = wv;
      if (sw) sw[b - b0] = wv;
    } else {
      int64_t rem = b;
      for (int q = 0; q < N - 1; ++q) {
        ib[q] = start[q] + (int32_t)(rem % len[q]);
        rem /= len[q];
      }
      p.w[b] = wblk;
      if (sw) sw[b - b0] = wblk;
    }
    if (sidx)
      for (int q = 0; q < N - 1; ++q) sidx[(b - b0) * (N - 1) + q] = ib[q];
    if (p.fbase) {  // fiber offset in the gather's layout (mode-major row, or native base)
      int64_t off = 0, jrow = 0, jmul = 1;
      bool own = true;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == n) continue;
        int64_t ik = ib[pos++];
        if (k == N - 1) {
          ik -= p.lo_last;
          if (ik < 0 || ik >= p.ldims[k]) own = false;
        }
        off += ik * p.lstride[k];
        jrow += ik * jmul;
        jmul *= p.ldims[k];
      }
      p.fbase[b] = own ? (p.mode_major ? jrow * p.pitch : off) : -1;
    }
  }
}

// SKR rows (Alg. 1) of rows [b0, b1): z_b[r] = prod_{k != n, ascending} A^(k)(i_k, r)
// Latency-friendly: each thread owns kSkrU elements and issues all their factor loads of one mode
// before multiplying (the product order over modes stays ascending).  Plain loads: A^(n) may have
// been written earlier in the same launch by another CTA.
constexpr int kSkrU = 8;
template <typename T>
__device__ __forceinline__ void skr_rows(const SampleParams& p, int64_t b0, int64_t b1, int tid, int nthreads) {
  const int N = p.N, n = p.n, R = p.R;
  T* Z = reinterpret_cast<T*>(p.zrow);
  const int cnt = (int)(b1 - b0) * R;
  for (int base = 0; base < cnt; base += nthreads * kSkrU) {
    int64_t row[kSkrU];
    int col[kSkrU];
    T z[kSkrU];
#pragma unroll
    for (int u = 0; u < kSkrU; ++u) {
      const int e = base + u * nthreads + tid;
      row[u] = e < cnt ? b0 + e / R : -1;
      col[u] = e < cnt ? e % R : 0;
      z[u] = T(1);
    }
    int32_t ix[kSkrU];
    int pos = 0;
    for (int k = 0; k < N; ++k) {
      if (k == n) continue;
      const T* F = reinterpret_cast<const T*>(p.factors[k]);
#pragma unroll
      for (int u = 0; u < kSkrU; ++u) ix[u] = row[u] >= 0 ? p.idx[row[u] * (N - 1) + pos] : 0;
      T f[kSkrU];
#pragma unroll
      for (int u = 0; u < kSkrU; ++u) f[u] = row[u] >= 0 ? F[(int64_t)ix[u] * R + col[u]] : T(0);
#pragma unroll
      for (int u = 0; u < kSkrU; ++u) z[u] = z[u] * f[u];
      ++pos;
    }
#pragma unroll
    for (int u = 0; u < kSkrU; ++u)
      if (row[u] >= 0) Z[row[u] * R + col[u]] = z[u];
  }
}

// weighted SKR rows zw_b = w_b z_b are stored padded to RP = ceil8(R) columns (zero past R and for
// padding rows); Gamma partials use 4x4 blocks (bi <= bj) with up to 4 fiber groups summed in order
__host__ __device__ inline int zg_rp(int R) { return (R + 7) / 8 * 8; }
__host__ __device__ inline int zg_groups(int R, int nthreads) {
  const int nb = (R + 3) / 4, nblk = nb * (nb + 1) / 2;
  const int g = nthreads / nblk;
  return g < 1 ? 1 : (g > 4 ? 4 : g);
}

// (a2, a3[, a4]) standalone sampler (API calls and the first step of a call).  grid-stride rows.
template <typename T>
__global__ void __launch_bounds__(256) k_sample(SampleParams p) {
  extern __shared__ uint64_t s_cdf[];
  __shared__ const uint64_t* cdfp[kMaxOrder];
  __shared__ uint64_t s_it;
  if (threadIdx.x == 0) s_it = *p.iter + p.iter_add;
  const uint64_t* cp[kMaxOrder];
  stage_cdfs(p, s_cdf, cp, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0)
    for (int k = 0; k < p.N; ++k) cdfp[k] = cp[k];
  __syncthreads();
  const int64_t per = (p.bmax + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * per, b1 = min(b0 + per, p.bmax);
  draw_rows(p, cdfp, s_it, b0, b1, threadIdx.x, blockDim.x);
  if (p.zrow) {
    __syncthreads();
    skr_rows<T>(p, b0, b1, threadIdx.x, blockDim.x);
  }
}

// ==========================================================================================
// (a4, a5, a6) fused SKR + fiber gather + partial contractions.
// grid = (I-tiles of 128 rows, batch chunks of TB fibers); 256 threads = 2 column halves x 128 rows.
// Per sub-batch of 32 fibers: z_b = (*)_{k != n, ascending} A^(k)(i_k, :) (Alg. 1),
// zw_b = omega_b z_b; x_b segment = X_(n)(i0:i0+128, j_b) (Alg. 5; contiguous rows of the
// mode-major copy, or stride S_n in the native layout); M_c += x zw^T; Gamma_c += zw z^T
// (I-tile 0 only).  Partials are reduced in a fixed order by k_update (deterministic).
// ==========================================================================================
constexpr int kGatherThreads = 256;
constexpr int kTI = 128;

template <typename T>
__host__ __device__ constexpr int gather_sb() { return sizeof(T) == 8 ? 16 : 32; }

// dynamic shared memory of k_gather<T, RPT>: max(main loop buffers, reduction buffers)
template <typename T, int RPT>
__host__ __device__ constexpr size_t gather_smem_bytes(int R) {
  // main: xs[SB][TI] + zw[SB][RP] + zu[SB][RP] + base[SB] (int64) + owned[SB] (int)
  // red : M tile [R][TI] + Gamma [R][R]
  return (size_t)(gather_sb<T>() * (kTI + 4 * RPT)) * sizeof(T) + gather_sb<T>() * 12 >
                 (size_t)(R * kTI + R * R) * sizeof(T)
             ? (size_t)(gather_sb<T>() * (kTI + 4 * RPT)) * sizeof(T) + gather_sb<T>() * 12
             : (size_t)(R * kTI + R * R) * sizeof(T);
}

// grid = (I-tiles, chunks) with cluster dims (1, CG): the CG chunk-CTAs of one I-tile reduce
// their partial tiles through distributed shared memory in rank order (deterministic), so
// k_update_table reads chunks/CG partials.
template <typename T, int RPT>
__global__ void __launch_bounds__(kGatherThreads) k_gather(GatherParams<T> p) {
  namespace cg = cooperative_groups;
  constexpr int RP = 2 * RPT;
  constexpr int kSB = gather_sb<T>();
  extern __shared__ __align__(16) unsigned char g_sm[];
  T* xs = reinterpret_cast<T*>(g_sm);            // [kSB][kTI]
  T* zw = xs + kSB * kTI;                         // [kSB][RP]
  T* zu = zw + kSB * RP;                          // [kSB][RP]
  int64_t* base = reinterpret_cast<int64_t*>(zu + kSB * RP);
  int* owned = reinterpret_cast<int*>(base + kSB);
  const int n = p.n, R = p.R;
  const int tid = threadIdx.x, il = tid % kTI, half = tid / kTI;
  const int64_t i0 = (int64_t)blockIdx.x * kTI;
  const int chunk = blockIdx.y;
  const int64_t beff = *p.beff;
  const int64_t b_begin = (int64_t)chunk * p.TB;
  const int64_t b_end = min(b_begin + p.TB, beff);
  const bool do_gamma = (blockIdx.x == 0);
  const int64_t estride = p.mode_major ? 1 : p.lstride[n];
  const bool row_ok = (i0 + il) < p.In_local;

  T acc[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) acc[j] = T(0);
  constexpr int GPT = (kMaxRank * kMaxRank + kGatherThreads - 1) / kGatherThreads;
  T gacc[GPT];
#pragma unroll
  for (int j = 0; j < GPT; ++j) gacc[j] = T(0);

  for (int64_t s = b_begin; s < b_end; s += kSB) {
    const int nb = (int)min((int64_t)kSB, b_end - s);
    // (a) per-fiber offsets (computed by the sampler)
    if (tid < kSB) {
      const int64_t fb = (tid < nb) ? p.fbase[s + tid] : -1;
      base[tid] = fb;
      owned[tid] = fb >= 0;
    }
    // (b) SKR rows (Alg. 1, prefetched by the sampler): weighted and unweighted, zero padded to RP
    for (int e = tid; e < kSB * RP; e += kGatherThreads) {
      const int bb = e / RP, r = e % RP;
      T z = T(0), zwv = T(0);
      if (bb < nb && r < R) {
        z = ldg(p.zrow + (s + bb) * R + r);
        zwv = (T)p.w[s + bb] * z;
      }
      zu[bb * RP + r] = z;
      zw[bb * RP + r] = zwv;
    }
    __syncthreads();
    // (c) fiber segments (Alg. 5): warp-coalesced along the row index, all loads in flight first
    {
      T v[kSB / 2];
#pragma unroll
      for (int q = 0; q < kSB / 2; ++q) {
        const int bb = half + 2 * q;
        v[q] = T(0);
        if (bb < nb && row_ok && owned[bb]) v[q] = ldg(p.X + base[bb] + (i0 + il) * estride);
      }
#pragma unroll
      for (int q = 0; q < kSB / 2; ++q) xs[(half + 2 * q) * kTI + il] = v[q];
    }
    __syncthreads();
    // (d) M tile += x zw^T
    for (int bb = 0; bb < nb; ++bb) {
      const T x = xs[bb * kTI + il];
#pragma unroll
      for (int j = 0; j < RPT; ++j) acc[j] += x * zw[bb * RP + half * RPT + j];
    }
    if (do_gamma) {
#pragma unroll
      for (int j = 0; j < GPT; ++j) {
        const int e = tid + j * kGatherThreads;
        if (e < R * R) {
          const int r1 = e / R, r2 = e % R;
          T g = gacc[j];
          for (int bb = 0; bb < nb; ++bb) g += zw[bb * RP + r1] * zu[bb * RP + r2];
          gacc[j] = g;
        }
      }
    }
    __syncthreads();
  }
  // ---- cluster reduction over the CG chunk-CTAs of this I-tile (rank order) ----
  cg::cluster_group cluster = cg::this_cluster();
  const int CG = (int)cluster.dim_blocks().y;
  const int q = (int)cluster.block_index().y;
  T* mred = reinterpret_cast<T*>(g_sm);   // [R][kTI] (aliases the main-loop buffers; synced above)
  T* gred = mred + R * kTI;               // [R][R]
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int r = half * RPT + j;
    if (r < R) mred[r * kTI + il] = acc[j];
  }
  if (do_gamma) {
#pragma unroll
    for (int j = 0; j < GPT; ++j) {
      const int e = tid + j * kGatherThreads;
      if (e < R * R) gred[e] = gacc[j];
    }
  }
  cluster.sync();
  const int part = chunk / CG;
  const int E = R * kTI;
  const int per = (E + CG - 1) / CG;
  for (int e = q * per + tid; e < min(E, (q + 1) * per); e += kGatherThreads) {
    T sum = T(0);
    for (int qq = 0; qq < CG; ++qq) sum += cluster.map_shared_rank(mred, qq)[e];
    const int r = e / kTI, ii = e % kTI;
    if (i0 + ii < p.In_local) p.Mp[((int64_t)part * R + r) * p.In_local + i0 + ii] = sum;
  }
  if (do_gamma) {
    const int EG = R * R, pg = (EG + CG - 1) / CG;
    for (int e = q * pg + tid; e < min(EG, (q + 1) * pg); e += kGatherThreads) {
      T sum = T(0);
      for (int qq = 0; qq < CG; ++qq) sum += cluster.map_shared_rank(gred, qq)[e];
      p.Gp[(int64_t)part * R * R + e] = sum;
    }
  }
  cluster.sync();  // keep every CTA's shared memory alive until the others finished reading it
}

// ==========================================================================================
// (a6, a7, a8) chunk reduction (fixed order), G = A Gamma - M, update.
//   fixed    : A <- A - alpha G                                  (eq:proposed)
//   adaptive : S <- S + G*G; A <- A - eta G / (b + S)^{1/2+eps}  (eq:etaada/eq:Aada, :531-537, R12)
// grid over blocks of kUR rows; 256 threads = kUR rows x (256/kUR) column groups.
// ==========================================================================================
constexpr int kUpdThreads = 256;
constexpr int kUR = 32;

template <typename T>
__global__ void __launch_bounds__(kUpdThreads) k_update(UpdateParams<T> p) {
  extern __shared__ __align__(16) unsigned char upd_sm[];
  const int R = p.R, tid = threadIdx.x;
  T* Gam = reinterpret_cast<T*>(upd_sm);   // R x R
  T* As = Gam + R * R;                      // kUR x (R+1)
  const int64_t r0 = (int64_t)blockIdx.x * kUR;
  // Gamma: fixed-order sum over chunks
  for (int e = tid; e < R * R; e += kUpdThreads) {
    T g;
    if (p.Gsum) {
      g = p.Gsum[e];
    } else {
      g = T(0);
      for (int c = 0; c < p.nchunks; ++c) g += p.Gp[(int64_t)c * R * R + e];
    }
    Gam[e] = g;
    if (blockIdx.x == 0 && p.Gam_out) p.Gam_out[e] = g;
  }
  for (int e = tid; e < kUR * R; e += kUpdThreads) {
    const int il = e / R, r = e % R;
    const int64_t i = r0 + il;
    As[il * (R + 1) + r] = (i < p.In_local) ? p.A[(p.row0 + i) * R + r] : T(0);
  }
  __syncthreads();
  const double alpha = p.alpha_dev ? *p.alpha_dev : p.alpha;
  if (p.iter && blockIdx.x == 0 && tid == 0) *p.iter += 1;  // r <- r + 1 (Alg. 6/7 line "r <- r+1")
  const int il = tid % kUR;
  const int64_t i = r0 + il;
  if (i >= p.In_local) return;
  for (int r = tid / kUR; r < R; r += kUpdThreads / kUR) {
    T m;
    if (p.Msum) {
      m = p.Msum[(int64_t)r * p.In_local + i];
    } else {
      m = T(0);
      for (int c = 0; c < p.nchunks; ++c) m += p.Mp[((int64_t)c * R + r) * p.In_local + i];
    }
    T ag = T(0);
    for (int c = 0; c < R; ++c) ag += As[il * (R + 1) + c] * Gam[c * R + r];
    const T g = ag - m;
    const int64_t gi = (p.row0 + i) * R + r;
    p.Gout[gi] = g;
    const T a = As[il * (R + 1) + r];
    if (p.rule == 0) {
      p.A[gi] = a - (T)alpha * g;
    } else {
      const T s = p.S[gi] + g * g;
      p.S[gi] = s;
      if (s > T(0)) {
        T step;
        if (p.eps == 0.0) step = (T)p.eta / sqrt((T)p.b + s);
        else step = (T)p.eta / (T)pow((double)((T)p.b + s), 0.5 + p.eps);
        p.A[gi] = a - step * g;
      }
    }
  }
}

// rank-ordered sum over the cluster of ptr[idx] in every CTA's shared memory: all remote loads are
// issued before the (fixed-order) additions; ranks >= CU contribute exact zeros.
template <typename T>
__device__ __forceinline__ T cluster_sum(const cooperative_groups::cluster_group& cl, T* ptr, int idx, int CU) {
  T v[16];
#pragma unroll
  for (int qq = 0; qq < 16; ++qq) v[qq] = (qq < CU) ? cl.map_shared_rank(ptr, qq)[idx] : T(0);
  T s = v[0];
#pragma unroll
  for (int qq = 1; qq < 16; ++qq) s += v[qq];
  return s;
}

// shared-memory mbarriers and 1-D bulk (TMA) copies
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// programmatic dependent launch (no-ops unless the launch carries the PDL attribute): the wide
// path's kernels let the next kernel of the chain be scheduled as soon as every CTA has started,
// and wait for the previous kernel's completion before touching its outputs
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// 1/x: MUFU approximation + two Newton steps (within ~1 ulp of 1/x).  The approximation flushes
// subnormals: valid for 2^-1021 < |x| < 2^1021, i.e. Gram entries (and pivots) in the normal range;
// a guard with a __drcp_rn fallback on the pivot chain measured ~15 % slower
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

// Inverse of the fp64 Gram on its numerically full-rank pivot set S by the symmetric sweep
// operator (Gauss-Jordan with diagonal pivoting in natural order, Goodnight 1979): sweeping pivot k
// maps M_ij -= M_ik M_kj / d (i, j != k), M_ik, M_kj /= d, M_kk = -1/d (d = M_kk).  The unswept
// diagonal is the Schur-complement diagonal, so a pivot whose value is <= tol is skipped (reading
// R4(b), the rank rule of a pivoted Cholesky); after sweeping S, M_SS = -(G_SS)^{-1}.
// Row groups x lanes: thread (g, c) of NT = 32 ceil(RMAX/32) G threads keeps rows
// [g RPG, (g + 1) RPG) of column c of the RMAX x RMAX matrix (identity past R; RMAX = ceil8(R),
// RPG = RMAX / G) in registers.  Pivots go in natural order in PAIRS P = {k, l = k + 1}; the pair
// loop is unrolled over the owner group's rows, so the pivot rows sit at STATIC register indices:
// the owner group publishes rows k and l interleaved (rb[2t] = M_kt, rb[2t+1] = M_lt; by symmetry
// also the pivot columns) with one 16-byte store per thread, one named barrier, then with
// B = M_PP = [[a, b], [b, c]] and det = a c - b^2:
//   a > tol and det > tol a  (both Schur diagonals a and det / a above tol: the single-pivot rule)
//     -> block sweep with ONE reciprocal 1/det (computed speculatively, before the test): per column
//        (f1, f2) = B^{-1} m with m = M_Pc (c not in P) or m = -e_k, -e_l (c in P: the negated
//        columns of B^{-1}); every held entry <- [c not in P] M_tc - rb[2t] f1 - rb[2t+1] f2 (two
//        DFMA, one 16-byte broadcast load, no selects); the owner group then sets rows k, l <- f1, f2
//        (the sweep operator on the block, M_PP -> -B^{-1});
//   otherwise single-pivot steps for k (if a > tol) and then l on the updated values (d > tol),
//   i.e. exactly the natural-order single-pivot sweep with the skip rule of R4(b).
// Cost history at R = 20 / 50 (cycles, tools/micro/sweep_grp.cu, sweep_st.cu): one pivot per
// barrier 9.6k / 37.7k -> 2x2 blocks 8.0k (8.7k) / 27.5k (29.2k) -> static pivot positions,
// interleaved 16-byte pivot rows, select-free update, Newton reciprocal 5.6k / 18.2k (results
// within 3e-16 relative of the previous form, same rank on rank-deficient inputs).
// Called by every thread of the CTA (>= NT threads); rowbuf: kSweepBuf doubles, 16-byte aligned;
// returns |S|.
template <int RMAX, int G>
__device__ int grp_sweep_inverse(double* Gm, int R, double tol, double* rowbuf, int* swept) {
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
  // |S| = popcount of the swept flags (two ballots per warp, R <= 64), not an R-long serial loop
  const int lane = tid & 31;
  const unsigned b0 = __ballot_sync(0xffffffffu, lane < R && swept[lane] != 0);
  const unsigned b1 = __ballot_sync(0xffffffffu, lane + 32 < R && swept[min(lane + 32, kMaxRank - 1)] != 0);
  return __popc(b0) + __popc(b1);
}

// MAXR: largest rank the calling kernel supports (instantiates only RMAX <= MAXR); needs 256 threads
// (128 for RMAX <= 32)
template <int MAXR = kMaxRank>
__device__ inline int grp_sweep_dispatch(double* Gm, int R, double tol, double* rowbuf, int* swept) {
  switch ((R + 7) / 8) {
    case 1: return grp_sweep_inverse<8, 4>(Gm, R, tol, rowbuf, swept);
    case 2: return grp_sweep_inverse<16, 4>(Gm, R, tol, rowbuf, swept);
    case 3: return grp_sweep_inverse<24, 4>(Gm, R, tol, rowbuf, swept);
    case 4: return grp_sweep_inverse<32, 4>(Gm, R, tol, rowbuf, swept);
    default: break;
  }
  if constexpr (MAXR > 32) {
    switch ((R + 7) / 8) {
      case 5: return grp_sweep_inverse<40, 4>(Gm, R, tol, rowbuf, swept);
      case 6: return grp_sweep_inverse<48, 4>(Gm, R, tol, rowbuf, swept);
      case 7: return grp_sweep_inverse<56, 4>(Gm, R, tol, rowbuf, swept);
      default: return grp_sweep_inverse<64, 4>(Gm, R, tol, rowbuf, swept);
    }
  }
  return 0;
}

// Pivoted variant (largest remaining Schur diagonal first, as a pivoted Cholesky would) for
// factors that can be rank deficient (I_n < 2R): dependent columns are left for last, where their
// residual Schur diagonals sit at rounding level and fall under tol.  Two barriers per pivot;
// the argmax is one warp reduction on a 32-bit key (26 high bits of the positive double + index).
template <int kSweepEPT>
__device__ int cta_sweep_inverse_pivoted(double* Gm, int R, double tol, double* rowbuf /* R */,
                                         int* swept /* R */, double* diag /* R */) {
  const int tid = threadIdx.x, nth = blockDim.x, RS = R + 1, lane = tid & 31;
  double v[kSweepEPT];
  int ei[kSweepEPT], ej[kSweepEPT];
#pragma unroll
  for (int t = 0; t < kSweepEPT; ++t) {
    const int e = tid + t * nth;
    ei[t] = (e < R * R) ? e / R : -1;
    ej[t] = (e < R * R) ? e % R : 0;
    v[t] = (e < R * R) ? Gm[ei[t] * RS + ej[t]] : 0.0;
  }
  for (int j = tid; j < R; j += nth) {
    diag[j] = Gm[j * RS + j];
    swept[j] = 0;
  }
  __syncthreads();
  int rank = 0;
  for (int step = 0; step < R; ++step) {
    unsigned key = 0u;
    for (int j = lane; j < R; j += 32) {
      const double d = diag[j];
      if (!swept[j] && d > 0.0) {
        const unsigned kj = ((unsigned)__double2hiint(d) & 0xFFFFFFC0u) | (unsigned)(63 - j);
        key = kj > key ? kj : key;
      }
    }
    key = __reduce_max_sync(0xffffffffu, key);
    if (key == 0u) break;
    const int k = 63 - (int)(key & 63u);
    const double d = diag[k];
    if (!(d > tol)) break;
#pragma unroll
    for (int t = 0; t < kSweepEPT; ++t)
      if (ei[t] == k) rowbuf[ej[t]] = v[t];
    __syncthreads();
    ++rank;
    const double dinv = __drcp_rn(d);
#pragma unroll
    for (int t = 0; t < kSweepEPT; ++t) {
      const int i = ei[t], j = ej[t];
      const double rki = rowbuf[i < 0 ? 0 : i], rkj = rowbuf[j];
      double nv = v[t] - rki * (rkj * dinv);
      nv = (j == k) ? rki * dinv : nv;
      nv = (i == k) ? rkj * dinv : nv;
      nv = (i == k && j == k) ? -dinv : nv;
      v[t] = (i >= 0) ? nv : v[t];
      if (i >= 0 && i == j && i != k) diag[i] = v[t];
    }
    if (tid == 0) swept[k] = 1;
    __syncthreads();
  }
#pragma unroll
  for (int t = 0; t < kSweepEPT; ++t) {
    const int i = ei[t], j = ej[t];
    if (i >= 0) Gm[i * RS + j] = (swept[i] && swept[j]) ? -v[t] : 0.0;
  }
  __syncthreads();
  return rank;
}

// ==========================================================================================
// (a6, a7, a8, a1, a9) fused update + table refresh: ONE thread-block cluster of CU <= 16 CTAs
// owns all rows of A^(n) (CTA q: rows [q*rows_per, ...)).
//   stage A (do_update): Gamma and M from the gather partials (fixed order), G = A Gamma - M,
//            fixed / adaptive update of the owned rows (eq:proposed / eq:Aada), r += 1
//   stage B (do_table) : importance table of the NEW A^(n) (R9):
//            leverage  -- partial fp64 Grams of the owned rows, summed over the cluster through
//                         DSMEM in rank order (identical in every CTA), pivoted Cholesky (every CTA
//                         redundantly, deterministic), l_i = ||L^{-1} a_{i,piv}||^2, p = l / rank
//            euclidean -- ||A||_F^2 = rank-ordered sum of per-CTA partials, p = ||a_i||^2 / ||A||^2
//            q = rint(p 2^32) (>= 1 if p > 0); CDF = integer scan: CTA-local scan + exclusive
//            prefix of the lower ranks' totals read through DSMEM.
// ==========================================================================================
template <typename T>
struct UTParams {
  int R, strategy, rule, do_update, do_table;
  int64_t In;            // rows of A^(n) (all rows)
  int64_t rows_per;      // rows per CTA
  int nparts;            // gather partials
  const T* Mp;           // [nparts][R][In]
  const T* Gp;           // [nparts][R][R]
  const T* Msum;         // sharded path: reduced M [R][In] (else NULL)
  const T* Gsum;         // sharded path: reduced Gamma (else NULL)
  T* A;
  T* S;
  T* Gout;
  T* Gam_out;
  double alpha;
  const double* alpha_dev;
  double eta, b, eps;
  uint64_t* iter;
  double* p_out;
  uint64_t* cdf;
  uint64_t* Tout;
  int* status;
  int sample_next;       // 1: draw the next step's batch (mode sp.n) after the table (a9 pipelining)
  SampleParams sp;
  long long* dbg;        // optional phase timestamps (CTA 0, thread 0), NULL in production
};

constexpr int kUTThreads = 256;

// fp64 blocking of the table stage: 4x4 register blocks, rows of stride RD = ceil4(R)
__host__ __device__ inline int ut_rd(int R) { return (R + 3) / 4 * 4; }
__host__ __device__ inline int ut_gram_groups(int R) {
  const int nb = (R + 3) / 4, nblk = nb * (nb + 1) / 2;
  const int g = kUTThreads / nblk;
  return g < 1 ? 1 : (g > 2 ? 2 : g);
}
__host__ __device__ inline size_t ut_work_bytes(int R, int64_t rows_per) {
  const size_t gram = sizeof(double) * (size_t)ut_gram_groups(R) * (R * (R + 1) / 2);
  const size_t scores = sizeof(double) * ((size_t)R * ut_rd(R) + (size_t)((R + 3) / 4) * rows_per);
  return gram > scores ? gram : scores;
}

// shared-memory carve-up of k_update_table (bytes), also used by the host to size the launch
__host__ __device__ inline size_t ut_smem_bytes(int R, int64_t rows_per, size_t esz) {
  size_t off = 0;
  auto take = [&](size_t bytes) { off = (off + 15) / 16 * 16; off += bytes; };
  take(esz * R * R);                     // Gam
  take(esz * rows_per * (R + 1));        // Aold
  take(esz * rows_per * (R + 1));        // Anew
  take(sizeof(double) * (R * (R + 1) / 2 + 1));  // partial Gram / partial ||A||^2 (read by peers)
  take(sizeof(double) * R * (R + 1));    // Gm (Gram -> inverse), row stride R+1
  take(sizeof(double) * kSweepBuf);   // sweep pivot-row buffers
  take(sizeof(int) * R);                 // swept flags
  take(sizeof(double) * rows_per);       // per-row p
  take(sizeof(unsigned long long) * rows_per);   // per-row q -> local inclusive scan
  take(sizeof(unsigned long long) * 2);  // CTA total (read by peers), pad
  take(sizeof(double) * rows_per * ut_rd(R));  // fp64 copy of the new rows (stride ceil4(R))
  take(ut_work_bytes(R, rows_per));      // Gram group partials | W (stride ceil4(R)) + score partials
  return off + 16;
}

#define UT_MARK(slot)                                                   \
  do {                                                                  \
    if (p.dbg && q == 0 && tid == 0) p.dbg[slot] = clock64();           \
  } while (0)

template <typename T>
__global__ void __launch_bounds__(kUTThreads) k_update_table(UTParams<T> p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int CU = (int)cluster.num_blocks();
  const int q = (int)cluster.block_rank();
  const int R = p.R, tid = threadIdx.x;
  const int64_t r_beg = min((int64_t)q * p.rows_per, p.In);
  const int64_t r_end = min(r_beg + p.rows_per, p.In);
  const int nr = (int)(r_end - r_beg);
  const int RS = R + 1;  // padded row stride
  extern __shared__ __align__(16) unsigned char ut_sm[];
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    off = (off + 15) / 16 * 16;
    unsigned char* ptr = ut_sm + off;
    off += bytes;
    return ptr;
  };
  T* Gam = reinterpret_cast<T*>(carve(sizeof(T) * R * R));
  T* Aold = reinterpret_cast<T*>(carve(sizeof(T) * p.rows_per * RS));
  T* Anew = reinterpret_cast<T*>(carve(sizeof(T) * p.rows_per * RS));
  double* gpart = reinterpret_cast<double*>(carve(sizeof(double) * (R * (R + 1) / 2 + 1)));
  double* Gm = reinterpret_cast<double*>(carve(sizeof(double) * R * (R + 1)));
  double* rowbuf = reinterpret_cast<double*>(carve(sizeof(double) * kSweepBuf));
  int* swept = reinterpret_cast<int*>(carve(sizeof(int) * R));
  double* prow = reinterpret_cast<double*>(carve(sizeof(double) * p.rows_per));
  unsigned long long* qrow = reinterpret_cast<unsigned long long*>(carve(sizeof(unsigned long long) * p.rows_per));
  unsigned long long* qtot = reinterpret_cast<unsigned long long*>(carve(sizeof(unsigned long long) * 2));
  const int RD = ut_rd(R);
  double* Ad = reinterpret_cast<double*>(carve(sizeof(double) * p.rows_per * RD));
  double* work = reinterpret_cast<double*>(carve(ut_work_bytes(R, p.rows_per)));
  __shared__ int piv[kMaxRank];
  __shared__ int s_rank, s_bad, s_stop, s_jm;
  __shared__ double s_red[kUTThreads / 32];
  __shared__ unsigned long long s_wtot[kUTThreads / 32];
  __shared__ double s_fro, s_tol;
  if (tid == 0) { s_bad = 0; s_rank = R; s_stop = 0; }
  const uint64_t r_now = *p.iter;  // every CTA reads r before CTA 0 may advance it (after a cluster barrier)
  UT_MARK(0);
  if (p.dbg && tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.dbg[16 + q] = smid;
  }

  // ---------------- stage A: update ----------------
#pragma unroll 8
  for (int e = tid; e < nr * R; e += kUTThreads) {
    const int il = e / R, c = e % R;
    Aold[il * RS + c] = p.A[(r_beg + il) * R + c];
  }
  if (p.do_update) {
    for (int e = tid; e < R * R; e += kUTThreads) {
      T g;
      if (p.Gsum) {
        g = p.Gsum[e];
      } else {
        g = T(0);
#pragma unroll 8
        for (int c = 0; c < p.nparts; ++c) g += p.Gp[(int64_t)c * R * R + e];
      }
      Gam[e] = g;
      if (q == 0 && p.Gam_out) p.Gam_out[e] = g;
    }
    __syncthreads();
    const double alpha = p.alpha_dev ? *p.alpha_dev : p.alpha;
    // element (il, r): consecutive threads -> consecutive rows (coalesced partial reads)
    for (int e = tid; e < nr * R; e += kUTThreads) {
      const int il = e % nr, r = e / nr;
      const int64_t i = r_beg + il;
      T m;
      if (p.Msum) {
        m = p.Msum[(int64_t)r * p.In + i];
      } else {
        m = T(0);
#pragma unroll 8
        for (int c = 0; c < p.nparts; ++c) m += p.Mp[((int64_t)c * R + r) * p.In + i];
      }
      T ag = T(0);
      for (int c = 0; c < R; ++c) ag += Aold[il * RS + c] * Gam[c * R + r];
      const T g = ag - m;
      const int64_t gi = i * R + r;
      p.Gout[gi] = g;
      const T a = Aold[il * RS + r];
      T an = a;
      if (p.rule == 0) {
        an = a - (T)alpha * g;
      } else {
        const T sv = p.S[gi] + g * g;
        p.S[gi] = sv;
        if (sv > T(0)) {
          T step;
          if (p.eps == 0.0) step = (T)p.eta / sqrt((T)p.b + sv);
          else step = (T)p.eta / (T)pow((double)((T)p.b + sv), 0.5 + p.eps);
          an = a - step * g;
        }
      }
      p.A[gi] = an;
      Anew[il * RS + r] = an;
    }
  } else {
    for (int e = tid; e < nr * R; e += kUTThreads) {
      const int il = e / R, c = e % R;
      Anew[il * RS + c] = Aold[il * RS + c];
    }
  }
  __syncthreads();
  bool synced = false;
  if (p.do_table && p.strategy != 0) {  // uniform tables are constant
  // ---------------- stage B: table of the new A^(n) ----------------
  UT_MARK(1);
  const bool lev = (p.strategy == 1 || p.strategy == 3);
  const int P = R * (R + 1) / 2;
  const int nb4 = (R + 3) >> 2;
  if (lev) {
    // fp64 copy of the owned rows, zero padded to RD
#pragma unroll 8
    for (int e = tid; e < nr * RD; e += kUTThreads) {
      const int il = e / RD, c = e % RD;
      Ad[e] = c < R ? (double)Anew[il * RS + c] : 0.0;
    }
    __syncthreads();
    // partial Gram sum_il a_il a_il^T: thread = (row group g, 4x4 block bi <= bj); groups summed in order
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
    for (int pair = tid; pair < P; pair += kUTThreads) {
      double s = work[pair];
      for (int gg = 1; gg < GG; ++gg) s += work[gg * P + pair];
      gpart[pair] = s;
    }
  } else {
    double acc = 0.0;
    for (int il = tid; il < nr; il += kUTThreads) {
      double rs = 0.0;
      for (int c = 0; c < R; ++c) rs += (double)Anew[il * RS + c] * (double)Anew[il * RS + c];
      prow[il] = rs;
      acc += rs;
    }
    // fixed-order block reduction
    __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) s_red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kUTThreads / 32; ++w) t += s_red[w];
      gpart[0] = t;
    }
  }
  cluster.sync();
  UT_MARK(2);
  if (lev) {
    for (int pair = tid; pair < P; pair += kUTThreads) {
      double v[16];
#pragma unroll
      for (int qq = 0; qq < 16; ++qq) v[qq] = (qq < CU) ? cluster.map_shared_rank(gpart, qq)[pair] : 0.0;
      double sum = 0.0;
#pragma unroll
      for (int qq = 0; qq < 16; ++qq) sum += v[qq];  // rank order (zeros past CU are exact)
      int r1 = 0, rem = pair;
      while (rem >= R - r1) { rem -= R - r1; ++r1; }
      const int r2 = r1 + rem;
      Gm[r1 * (R + 1) + r2] = sum;
      Gm[r2 * (R + 1) + r1] = sum;
    }
    __syncthreads();
    // Inverse of the Gram on its numerically full-rank pivot set S by the symmetric sweep
    // operator (Gauss-Jordan with diagonal pivoting, Goodnight 1979): sweeping pivot k maps
    //   M_ij -= M_ik M_kj / d (i,j != k),  M_ik, M_kj /= d,  M_kk = -1/d   (d = M_kk).
    // The unswept diagonal is the Schur-complement diagonal, so the pivot rule and the rank
    // tolerance R4(b) are those of a pivoted Cholesky; after sweeping S, M_SS = -(G_SS)^{-1}.
    // l_i = a_{i,S}^T (G_SS)^{-1} a_{i,S} = ||Q(i,:)||^2 (Def. 2.3) because range(A_S) = range(A).
    if (tid == 0) {
      double d0 = 0.0;
      bool fin = true;
      for (int j = 0; j < R; ++j) {
        const double dj = Gm[j * (R + 1) + j];
        d0 = fmax(d0, dj);
        fin = fin && (dj == dj) && dj < 1.7e308;
      }
      if (!fin) s_bad |= 8;
      s_tol = (double)(p.In > R ? p.In : R) * 2.220446049250313e-16 * d0;
    }
    __syncthreads();
    {
      constexpr int EPT = (kMaxRank * kMaxRank + kUTThreads - 1) / kUTThreads;
      const int rk = (p.In < 2 * R) ? cta_sweep_inverse_pivoted<EPT>(Gm, R, s_tol, rowbuf, swept, rowbuf + R)
                                    : grp_sweep_dispatch(Gm, R, s_tol, rowbuf, swept);
      if (tid == 0) {
        s_rank = rk;
        if (rk == 0) s_bad |= 2;
      }
    }
    __syncthreads();
    const int rank = s_rank;
    UT_MARK(4);
    // scores of the owned rows: l_i = sum_c (A W)_ic a_ic.  W -> stride RD (zero padded); thread
    // task = 4 rows x 4 columns of A W (k in pairs: 8 LDS.128 per 32 DFMA); per-column-group partials
    // summed in order.
    {
      double* Wd = work;
      double* sc = work + R * RD;  // [nb4][rows_per]
      for (int e = tid; e < R * RD; e += kUTThreads) {
        const int r1 = e / RD, c = e % RD;
        Wd[e] = c < R ? Gm[r1 * (R + 1) + c] : 0.0;
      }
      __syncthreads();
      const int nrg = (nr + 3) >> 2, ntask = nrg * nb4;
      for (int t = tid; t < ntask; t += kUTThreads) {
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
        for (int kk = 0; kk < R; kk += 2) {  // RD is a multiple of 4: the pair (kk, kk+1) is in range
          double2 av[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) av[a] = *reinterpret_cast<const double2*>(arow[a] + kk);
          const double2 w00 = *reinterpret_cast<const double2*>(Wd + kk * RD + 4 * cg);
          const double2 w01 = *reinterpret_cast<const double2*>(Wd + kk * RD + 4 * cg + 2);
          const double2 w10 = *reinterpret_cast<const double2*>(Wd + (kk + 1 < R ? kk + 1 : kk) * RD + 4 * cg);
          const double2 w11 = *reinterpret_cast<const double2*>(Wd + (kk + 1 < R ? kk + 1 : kk) * RD + 4 * cg + 2);
          const double wk0[4] = {w00.x, w00.y, w01.x, w01.y};
          const double wk1[4] = {kk + 1 < R ? w10.x : 0.0, kk + 1 < R ? w10.y : 0.0, kk + 1 < R ? w11.x : 0.0,
                                 kk + 1 < R ? w11.y : 0.0};
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
      for (int il = tid; il < nr; il += kUTThreads) {
        double l = 0.0;
        for (int cg = 0; cg < nb4; ++cg) l += sc[cg * p.rows_per + il];
        prow[il] = rank > 0 ? fmax(l, 0.0) / (double)rank : 0.0;
      }
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
    for (int il = tid; il < nr; il += kUTThreads) prow[il] = fro > 0.0 ? prow[il] / fro : 0.0;
  }
  __syncthreads();
  UT_MARK(5);
  // quantise + CTA-local inclusive scan (each thread a contiguous segment of rows)
  const int seg = (nr + kUTThreads - 1) / kUTThreads;
  const int a0 = min(tid * seg, nr), a1 = min(a0 + seg, nr);
  unsigned long long local = 0;
  int bad = 0;
  for (int il = a0; il < a1; ++il) {
    const double pv = prow[il];
    unsigned long long qv;
    if (!(pv == pv) || pv > 2.0) {
      bad = 1;
      qv = 0;
    } else if (pv > 0.0) {
      const double sc = rint(pv * 4294967296.0);
      qv = (sc < 1.0) ? 1ull : (unsigned long long)sc;
    } else {
      qv = 0;
    }
    if (p.p_out) p.p_out[r_beg + il] = pv;
    local += qv;
    qrow[il] = local;  // inclusive within the segment
  }
  if (bad) atomicOr(&s_bad, 8);
  const int lane = tid & 31, wid = tid >> 5;
  unsigned long long incl = local;
  __syncwarp();  // reconverge: a diverged warp takes the slow collective shuffle path
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_wtot[wid] = incl;
  __syncthreads();
  unsigned long long wpre = 0;
  for (int w = 0; w < wid; ++w) wpre += s_wtot[w];
  const unsigned long long seg_pre = wpre + incl - local;
  if (tid == kUTThreads - 1) qtot[0] = seg_pre + local;  // CTA total
  __syncthreads();
  cluster.sync();
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
  cluster.sync();  // peers may still read this CTA's shared memory; cdf visible cluster-wide
  synced = true;
  UT_MARK(6);
  }  // stage B

  // ---------------- stage C: the next step's batch (sampling contract; tables now current) ----
  if (p.sample_next) {
    if (!synced) {
      __threadfence();
      cluster.sync();  // updated A^(n) rows of every CTA visible (SKR reads them)
      synced = true;
    }
    uint64_t* s_cdf = reinterpret_cast<uint64_t*>(ut_sm + ((off + 15) / 16 * 16));
    const uint64_t* cp[kMaxOrder];
    stage_cdfs(p.sp, s_cdf, cp, tid, kUTThreads);
    __syncthreads();
    const int64_t per = (p.sp.bmax + CU - 1) / CU;
    const int64_t b0 = min((int64_t)q * per, p.sp.bmax), b1 = min(b0 + per, p.sp.bmax);
    draw_rows(p.sp, cp, r_now + (p.do_update ? 1 : 0), b0, b1, tid, kUTThreads);
    __syncthreads();
    skr_rows<T>(p.sp, b0, b1, tid, kUTThreads);
    UT_MARK(7);
  }
  if (p.do_update) {
    if (!synced) cluster.sync();   // all CTAs have read r_now
    if (q == 0 && tid == 0) *p.iter = r_now + 1;  // r <- r + 1 (Alg. 6/7)
  }
}

// squared Frobenius norms of the last-mode slices (cp_slice_sqnorms; SURVEY 8(e) mitigation 2, the
// data-side proxy of the slab masses): block (x, y) sums chunk x of slice y in fp64 -> part[y][x]
constexpr int kSliceChunks = 32;
template <typename T>
__global__ void __launch_bounds__(256) k_slice_sq(const T* __restrict__ X, int64_t slice_len, double* __restrict__ part) {
  const int64_t s = blockIdx.y, c = blockIdx.x;
  const int64_t per = (slice_len + kSliceChunks - 1) / kSliceChunks;
  const int64_t a = c * per, b = min(slice_len, a + per);
  const T* x = X + s * slice_len;
  double acc = 0.0;
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
    const double v = (double)x[i];
    acc = fma(v, v, acc);
  }
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[s * kSliceChunks + c] = t;
  }
}
template <int V = 0>  // headers hold only templates of __global__ functions (one emitting unit each)
__global__ void k_slice_sum(const double* __restrict__ part, int64_t nslices, double* __restrict__ out) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nslices) {
    double t = 0.0;
    for (int c = 0; c < kSliceChunks; ++c) t += part[s * kSliceChunks + c];  // chunk order
    out[s] = t;
  }
}

// reduce chunk partials into Msum [R][In_local] and Gsum [R][R] (sharded path, phase 0)
template <typename T>
__global__ void k_reduce_partials(const T* __restrict__ Mp, const T* __restrict__ Gp, int nchunks, int R,
                                  int64_t In_local, T* __restrict__ Msum, T* __restrict__ Gsum) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)R * In_local;
  if (e < tot) {
    T m = T(0);
    for (int c = 0; c < nchunks; ++c) m += Mp[(int64_t)c * tot + e];
    Msum[e] = m;
  }
  if (e < (int64_t)R * R) {
    T g = T(0);
    for (int c = 0; c < nchunks; ++c) g += Gp[(int64_t)c * R * R + e];
    Gsum[e] = g;
  }
}

// ==========================================================================================
// fit: per mode-0 fiber f (global tuple of modes 1..N-1), w_r = prod_{k>=1} A^(k)(i_k, r) in
// fp64, x_hat(i0) = sum_r A^(0)(i0, r) w_r; accumulate (x - x_hat)^2 and x^2 in fp64.
// One block handles fibers f = blockIdx.x, += gridDim.x; per-block partials (fixed order).
// ==========================================================================================
template <typename T>
__global__ void __launch_bounds__(256) k_fit(const T* __restrict__ X, int N, const int64_t* __restrict__ ldims_dev,
                                             int64_t lo_last, int R, const T* const* __restrict__ factors,
                                             int64_t nfib, double* __restrict__ partial) {
  __shared__ double wsh[kMaxRank];
  __shared__ double red[2][256];
  __shared__ int64_t ld[kMaxOrder];
  const int tid = threadIdx.x;
  if (tid < N) ld[tid] = ldims_dev[tid];
  __syncthreads();
  const int64_t I0 = ld[0];
  double res = 0.0, xx = 0.0;
  for (int64_t f = blockIdx.x; f < nfib; f += gridDim.x) {
    if (tid < R) {
      int64_t rem = f;
      double w = 1.0;
      for (int k = 1; k < N; ++k) {
        int64_t ik = rem % ld[k];
        rem /= ld[k];
        if (k == N - 1) ik += lo_last;
        w *= (double)factors[k][ik * R + tid];
      }
      wsh[tid] = w;
    }
    __syncthreads();
    const T* xf = X + f * I0;
    const T* A0 = factors[0];
    for (int64_t i = tid; i < I0; i += blockDim.x) {
      double xh = 0.0;
      for (int r = 0; r < R; ++r) xh += (double)A0[i * R + r] * wsh[r];
      const double x = (double)xf[i];
      res += (x - xh) * (x - xh);
      xx += x * x;
    }
    __syncthreads();
  }
  red[0][tid] = res;
  red[1][tid] = xx;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (tid < st) {
      red[0][tid] += red[0][tid + st];
      red[1][tid] += red[1][tid + st];
    }
    __syncthreads();
  }
  if (tid == 0) {
    partial[2 * blockIdx.x] = red[0][0];
    partial[2 * blockIdx.x + 1] = red[1][0];
  }
}

// ==========================================================================================
// mode-major copy: view X as [outer][I_n][inner] (inner = prod_{k<n} I_k) and write
// Y[(o*inner + in)*pitch + i] = X[(o*I_n + i)*inner + in]  (row j = in + inner*o = eq:map).
// 32x32 shared-memory tiles; grid (ceil(inner/32), ceil(I_n/32), outer).
// ==========================================================================================
template <typename T>
__global__ void k_transpose(const T* __restrict__ X, T* __restrict__ Y, int64_t In, int64_t inner, int64_t outer,
                            int64_t pitch) {
  __shared__ T tile[32][33];
  const int64_t in0 = (int64_t)blockIdx.x * 32, i0 = (int64_t)blockIdx.y * 32;
  for (int64_t o = blockIdx.z; o < outer; o += gridDim.z) {
    const T* Xo = X + o * In * inner;
    T* Yo = Y + o * inner * pitch;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const int64_t i = i0 + r, in = in0 + threadIdx.x;
      if (i < In && in < inner) tile[r][threadIdx.x] = Xo[i * inner + in];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
      const int64_t in = in0 + r, i = i0 + threadIdx.x;
      if (in < inner && i < In) Yo[in * pitch + i] = tile[threadIdx.x][r];
    }
    __syncthreads();
  }
}

}  // namespace cps
