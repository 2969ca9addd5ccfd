// gupdate.cuh -- k_gather_update: the wide single-GPU gather kernel for problems too large for one
// cluster (C4/C5 of BASELINE.json).  ONE launch does, for every row block of A^(n):
//
//   (a5) TensorSamp (Alg. 5): the I-tile segment of every sampled fiber,
//        staged HBM -> shared memory with cp.async (16-byte vectors of the mode-major copy, or
//        scalars of the native layout), NS-stage pipeline;
//   (a6) M_tile = X_F diag(w) Z_F restricted to the tile (eq:gradient1/2):
//        register-blocked FFMA (4 rows x CPT columns per thread) against the weighted SKR rows
//        zw_b = w_b z_b prepared by the sampler (Alg. 1);
//   (a6) deterministic split-K: the CK CTAs of an I-tile hold its CK batch chunks; their partial
//        tiles go to a global workspace, summed in chunk order by k_table_sample, which also forms
//        G = A Gamma - M and applies the update (a7, a8) before rebuilding the table.
//
// grid = (ceil(I_n / TI), CK); 256 threads: warp w = column group
// [w CPT, (w+1) CPT), lane l = rows [4l, 4l+4) of the tile.  RP = 8 CPT >= R (zero padded).
#pragma once
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cps {

constexpr int kGUThreads = 256;
constexpr int kGUTI = 128;     // rows per I-tile
constexpr int kGUKS = 32;      // fibers per pipeline stage
constexpr int kGUStages = 3;

template <typename T>
struct GUParams {
  int R;
  int64_t In;             // rows of A^(n)
  const T* X;             // gather base: mode-major copy of mode n (es = 1) or the native tensor
  int64_t es;             // element stride along a fiber
  int vec;                // 1: es == 1 and every fiber starts 16-byte aligned (16-byte cp.async)
  int64_t rowlen;         // tcgen05 path: readable elements per fiber row (pitch of the mode-major copy)
  const int64_t* fbase;   // [Bmax] element offset of fiber b (-1: padding row)
  const T* zwp;           // [Bmax][RP] weighted SKR rows, zero padded (sampler)
  const float* zimg;      // tcgen05 path: A-operand images {zh; zl} per stage of 32 fibers (zimg_off)
  int64_t bmax;           // rows of the batch buffers for this mode
  int64_t KB;             // fibers per chunk (= per CTA)
  const T* Gam;           // [R][R] Gamma of this batch (sampler)
  const T* gcl;           // [ncl][R][R] the sampler's cluster partials of Gamma
  int ncl;
  T* gam_sum;             // out: Gamma = sum of the partials in cluster order (read by k_update_wide)
  T* A;                   // A^(n), row-major I_n x R, updated in place
  T* S;                   // adaptive accumulator or NULL
  T* Gout;                // G (debug hook)
  T* Gam_out;             // Gamma (debug hook)
  int rule;
  double alpha;
  const double* alpha_dev;
  double eta, b, eps;
  uint64_t* iter;         // r <- r + 1 (Alg. 6/7)
  T* Mpart;               // [tiles][chunks][TI][R] partial tiles (split-K workspace)
  unsigned* cnt;          // [tiles] arrival counters (zero between launches)
  // replicas with a batch split (CP_FLAG_REPLICA): this launch's y-index q covers batch chunk c_first +
  // q c_step of the CK chunks (1 GPU: 0 + q 1, all of them)
  int CK, c_first, c_step;
  long long* dbg;         // optional phase timestamps (CTA (0,0), thread 0)
};

// shared memory: max(pipeline, epilogue) + Gamma + fiber offsets of the chunk
template <typename T, int CPT>
__host__ __device__ constexpr size_t gu_pipe_bytes() {
  return (size_t)kGUStages * kGUKS * (kGUTI + 8 * CPT) * sizeof(T);
}
// epilogue: partial tile [TI][RP+1]
template <typename T, int CPT>
__host__ __device__ constexpr size_t gu_epi_bytes() {
  return (size_t)kGUTI * (8 * CPT + 1) * sizeof(T);
}
template <typename T, int CPT>
__host__ __device__ inline size_t gu_smem_bytes(int64_t KB) {
  constexpr size_t a = gu_pipe_bytes<T, CPT>() > gu_epi_bytes<T, CPT>() ? gu_pipe_bytes<T, CPT>()
                                                                          : gu_epi_bytes<T, CPT>();
  return a + (size_t)kMaxRank * kMaxRank * sizeof(T) + (size_t)KB * sizeof(int64_t) + 64;
}

// Gamma = sum over the sampler's cluster partials in cluster order: entries [e0, E) with stride
// es, every load of an entry in flight at once.  Run by threads the gather kernels leave idle (the
// kernels themselves never read Gamma; k_update_wide does, after them).
template <typename T>
__device__ __forceinline__ void gu_gamma_sum(const GUParams<T>& p, int e0, int es) {
  const int E = p.R * p.R;
  for (int e = e0; e < E; e += es) {
    T v[16], s = T(0);
    for (int c0 = 0; c0 < p.ncl; c0 += 16) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {  // clamped unconditional loads, then masked (no branch per load)
        const T t = __ldcg(p.gcl + (int64_t)(c0 + k < p.ncl ? c0 + k : p.ncl - 1) * E + e);
        v[k] = c0 + k < p.ncl ? t : T(0);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) s += v[k];  // cluster order; zeros past ncl are exact
    }
    p.gam_sum[e] = s;
  }
}

template <typename T>
__device__ __forceinline__ int gu_chunk(const GUParams<T>& p) { return p.c_first + (int)blockIdx.y * p.c_step; }

// Epilogue shared by both mainloops: this CTA's partial tile M_c (shared, [TI][MS]) -> the split-K
// workspace p.Mpart[tile][chunk][R][TI] (row-contiguous, coalesced).  The chunk partials are summed
// in chunk order, and G = A Gamma - M and the update applied, by k_table_sample (the next launch).
template <typename T>
__device__ __forceinline__ void gu_finish(const GUParams<T>& p, const T* Mt, int MS, int64_t i0, int tid, int nth) {
  const int R = p.R, TI = kGUTI;
  const int nrow = (int)cmax64(0, cmin64(TI, p.In - i0));
  T* part = p.Mpart + ((int64_t)blockIdx.x * p.CK + gu_chunk(p)) * R * TI;
  for (int e = tid; e < R * TI; e += nth) {
    const int r = e / TI, rl = e % TI;
    if (rl < nrow) part[e] = Mt[rl * MS + r];
  }
  // r <- r + 1 (Alg. 6/7); nothing in this launch reads r (Gamma_out: k_update_wide)
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *p.iter += 1;
}

template <typename T, int CPT>
__global__ void __launch_bounds__(kGUThreads, 1) k_gather_update(GUParams<T> p) {
  constexpr int RP = 8 * CPT;
  constexpr int TI = kGUTI, KS = kGUKS, NS = kGUStages;
  constexpr int VE = 16 / (int)sizeof(T);      // elements per 16-byte vector
  constexpr int XV = TI / VE;                  // vectors per fiber segment
  constexpr int ZV = RP / VE;                  // vectors per zw row (RP*sizeof(T) is a multiple of 16)
  extern __shared__ __align__(16) unsigned char gu_sm[];
  T* pipe = reinterpret_cast<T*>(gu_sm);
  constexpr size_t kA = gu_pipe_bytes<T, CPT>() > gu_epi_bytes<T, CPT>() ? gu_pipe_bytes<T, CPT>()
                                                                           : gu_epi_bytes<T, CPT>();
  T* sGam = reinterpret_cast<T*>(gu_sm + kA);
  int64_t* sfb = reinterpret_cast<int64_t*>(gu_sm + kA + (size_t)kMaxRank * kMaxRank * sizeof(T));

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int R = p.R;
  const int64_t i0 = (int64_t)blockIdx.x * TI;
  const int64_t c0 = (int64_t)gu_chunk(p) * p.KB;
  const int64_t c1 = min(c0 + p.KB, p.bmax);
  const int nfib = (int)cmax64(0, c1 - c0);
  const int nst = (nfib + KS - 1) / KS;

  pdl_trigger();
  pdl_wait();  // the batch comes from the previous kernel
  {  // Gamma: one entry per thread over the whole grid
    const int lin = (blockIdx.y * gridDim.x + blockIdx.x) * kGUThreads + tid;
    gu_gamma_sum<T>(p, lin, gridDim.x * gridDim.y * kGUThreads);
  }
  cp_async_u64(reinterpret_cast<uint64_t*>(sfb), reinterpret_cast<const uint64_t*>(p.fbase + c0), nfib, tid,
               kGUThreads);
  cp_async_wait<0>();
  __syncthreads();

  auto xs_of = [&](int s) { return pipe + (size_t)s * KS * (TI + RP); };
  // issue the cp.async group of pipeline stage `st` (fibers [st*KS, st*KS + KS) of the chunk)
  auto load_stage = [&](int st) {
    T* xs = xs_of(st % NS);
    T* zs = xs + KS * TI;
    const int f0 = st * KS;
    if (p.vec) {
      for (int e = tid; e < KS * XV; e += kGUThreads) {
        const int kk = e / XV, v = e % XV;
        const int lb = f0 + kk;
        const int64_t fb = lb < nfib ? sfb[lb] : -1;
        const int64_t r0 = i0 + (int64_t)v * VE;
        int bytes = 0;
        const T* src = p.X;
        if (fb >= 0 && r0 < p.In) {
          bytes = (int)cmin64(p.In - r0, VE) * (int)sizeof(T);
          src = p.X + fb + r0;
        }
        cp_async16(xs + kk * TI + v * VE, src, bytes);
      }
    } else {
      for (int e = tid; e < KS * TI; e += kGUThreads) {
        const int kk = e / TI, il = e % TI;
        const int lb = f0 + kk;
        const int64_t fb = lb < nfib ? sfb[lb] : -1;
        const int64_t r = i0 + il;
        const bool ok = fb >= 0 && r < p.In;
        cp_async_small<sizeof(T)>(xs + kk * TI + il, ok ? p.X + fb + r * p.es : p.X, ok ? (int)sizeof(T) : 0);
      }
    }
    for (int e = tid; e < KS * ZV; e += kGUThreads) {
      const int kk = e / ZV, v = e % ZV;
      const int64_t b = c0 + f0 + kk;
      const bool ok = b < c1;
      cp_async16(zs + kk * RP + v * VE, ok ? p.zwp + b * RP + v * VE : p.zwp, ok ? 16 : 0);
    }
  };

  T acc[4][CPT];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[a][c] = T(0);

#pragma unroll
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nst) load_stage(s);
    cp_async_commit();
  }
  for (int st = 0; st < nst; ++st) {
    cp_async_wait<NS - 2>();
    __syncthreads();  // stage st landed for every thread; stage st-1's buffer is free
    if (st + NS - 1 < nst) load_stage(st + NS - 1);
    cp_async_commit();
    const T* xs = xs_of(st % NS);
    const T* zs = xs + KS * TI + wid * CPT;
    const int kmax = min(KS, nfib - st * KS);
#pragma unroll 4
    for (int kk = 0; kk < kmax; ++kk) {
      T xv[4];
      if constexpr (sizeof(T) == 4) {
        const float4 v = *reinterpret_cast<const float4*>(xs + kk * TI + 4 * lane);
        xv[0] = v.x; xv[1] = v.y; xv[2] = v.z; xv[3] = v.w;
      } else {
        const double2 v0 = *reinterpret_cast<const double2*>(xs + kk * TI + 4 * lane);
        const double2 v1 = *reinterpret_cast<const double2*>(xs + kk * TI + 4 * lane + 2);
        xv[0] = v0.x; xv[1] = v0.y; xv[2] = v1.x; xv[3] = v1.y;
      }
      T zv[CPT];
#pragma unroll
      for (int c = 0; c < CPT; ++c) zv[c] = zs[kk * RP + c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[a][c] = fma(xv[a], zv[c], acc[a][c]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- split-K: partial tile -> shared [TI][RP+1] -> gu_finish ----
  constexpr int MS = RP + 1;
  T* Mt = pipe;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < CPT; ++c) Mt[(4 * lane + a) * MS + wid * CPT + c] = acc[a][c];
  __syncthreads();
  gu_finish<T>(p, Mt, MS, i0, tid, kGUThreads);
}

}  // namespace cps
