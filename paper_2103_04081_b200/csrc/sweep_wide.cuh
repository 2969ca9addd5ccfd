// sweep_wide.cuh -- k_sweep_wide: the fp32 single-GPU wide path (C4-sized problems, every mode on the
// tcgen05 gather) as ONE cooperative persistent launch per cp_sgd_sweep / cp_sgd_step call.
//
// One CTA per SM (448 threads, the tcgen05 gather's shared-memory ring), all co-resident (cooperative
// launch).  Per SGD iteration r on mode n (Alg. 6 / Alg. 7):
//
//   S  (a2-a4)  the batch of mode n at r: 32-fiber units over the CTAs -- Philox draws from the
//               staged integer CDFs (eq:ik / eq:bik, contract DESIGN.md section 4), exact fp64
//               weights (eq:gradient1/2), fiber offsets, SKR rows (Alg. 1), the {zh; zl} 3xTF32
//               A-operand images, and per-CTA partials of Gamma = Z_F^T diag(w) Z_F (unit order)
//   -- grid barrier --
//   G  (a5, a6) TensorSamp (Alg. 5) + M = X_F diag(w) Z_F: (I-tile, batch chunk) items of the
//               warp-specialised tcgen05 mainloop (gupdate_tc.cuh), split-K partial tiles to the
//               workspace; idle lanes sum Gamma over the CTA partials (CTA order)
//   -- grid barrier --
//   U  (a6-a8)  16-row units: M = sum of the chunk partials (chunk order), G = A Gamma - M, fixed /
//               adaptive update (eq:proposed, eq:etaada/eq:Aada); fp64 Gram partials (leverage) or
//               row norms (Euclidean) of the new rows (a1)
//   -- grid barrier --
//   P  (a1)     leverage: the Gram's pairs summed over the unit partials (unit order), a slice per CTA;
//               an arrival counter (no grid barrier: only the inverse waits for it)
//   I  (a1)     every CTA with row units waits for the Gram and inverts it redundantly (natural-order
//               symmetric sweep on the numerically full-rank pivot set, R4(b)) -- the R-pivot chain
//               is serial; computing it everywhere saves the publish / poll round trip
//   Q  (a1)     scores of the unit's rows (a^T W a / |S| or ||a||^2 / ||A||_F^2), 2^-32 fixed-point
//               quantisation, unit aggregates published with a tag, decoupled look-back over the
//               preceding units' aggregates -> CDF rows; the last unit writes T and the status
//   -- grid barrier --  (the table of the new A^(n) is complete: R9)
//
// Deterministic: every sum has a fixed order (unit / chunk / CTA order), so results do not depend on
// scheduling.  Citations: PAPER.md:<lines> (<label>); R<k> = DESIGN.md readings.
#pragma once
#include <cooperative_groups.h>

#include "sweep_wide_params.cuh"

namespace cps {

// ------------------------------------------------------------------------------------------ sync
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// grid-wide barrier of the co-resident grid: a monotonic arrival counter (zeroed by the host before
// every launch), one fire-and-forget release reduction per CTA, one polling thread per CTA with a
// short back-off.  (Polling flags with every thread of every CTA made the flag lines an L2 hot spot
// that slowed every other load of the launch; so did polling without back-off.)
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
  while ((int)(ld_acquire_u32(p) - target) < 0) {
  }
}
__device__ __forceinline__ void grid_barrier(unsigned* cnt, unsigned& nbar) {
  __syncthreads();
  ++nbar;
  if (threadIdx.x == 0) {
    red_release_add(cnt, 1u);
    wait_count(cnt, nbar * gridDim.x);
  }
  __syncthreads();
  __syncwarp();  // warp 0 reconverged after its single-thread branch
}

// global -> shared copy of `bytes` contiguous bytes (src and dst 16-byte aligned) in 16-byte L2-only
// cp.async chunks, all in flight (one commit group; the caller waits): data written by other CTAs of
// this launch must not be read through L1
__device__ __forceinline__ void cpcg_bytes(void* dst, const void* src, int64_t bytes, int tid, int nth) {
  unsigned char* d = reinterpret_cast<unsigned char*>(dst);
  const unsigned char* s8 = reinterpret_cast<const unsigned char*>(src);
  for (int64_t o = (int64_t)tid * 16; o < bytes; o += (int64_t)nth * 16)
    cp_async16(d + o, s8 + o, (int)cmin64(16, bytes - o));
  cp_async_commit();
}

// global -> shared copy through L2 (data written by other CTAs of this launch): 8 loads in flight
// per thread
__device__ __forceinline__ void ldcg_copy_u64(uint64_t* dst, const uint64_t* src, int64_t n, int tid, int nth) {
  for (int64_t i0 = tid; i0 < n; i0 += 8 * (int64_t)nth) {
    uint64_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + (int64_t)u * nth;
      v[u] = __ldcg(src + (i < n ? i : n - 1));  // unconditional (clamped) load: no branch per load
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + (int64_t)u * nth;
      if (i < n) dst[i] = v[u];
    }
  }
}

// Broadcast reads (data every CTA fetches at the same moment: the CDFs, Gamma, the Gram): ONE thread
// issues TMA bulk copies completing on the CTA's mbarrier, every thread waits on its phase.  Per-thread
// 16-byte requests from every CTA queue on the few L2 lines holding such data; a bulk copy is one request
// stream per CTA.  The generic-proxy writes of other CTAs were acquired at the preceding barrier; the
// proxy fence orders them before the async-proxy reads.  bytes: multiples of 16, 16-byte aligned.
struct PWBulk {
  uint64_t* bar;
  uint32_t ph;  // parity of the next phase (identical in every thread of the CTA)
};
__device__ __forceinline__ void pw_bulk_begin(const PWBulk& b, uint32_t total_bytes) {  // one thread
  // all state spaces: the global data (see above) and the shared destination's earlier generic accesses
  // (the caller passed a CTA barrier after them)
  asm volatile("fence.proxy.async;" ::: "memory");
  mbar_expect_tx(b.bar, total_bytes);
}
__device__ __forceinline__ void pw_bulk_wait(PWBulk& b) {  // every thread
  mbar_wait(b.bar, b.ph);
  b.ph ^= 1u;
}
__host__ __device__ inline uint32_t pw_b16(int64_t bytes) { return (uint32_t)((bytes + 15) / 16 * 16); }

// ------------------------------------------------------------------------------------------ phase S
struct PWShared {  // static shared state of the phases
  const uint64_t* cp[kMaxOrder];
  // per-mode parameters the sampling phase indexes with run-time modes, staged once per phase (register-indexed
  // constant-bank loads on the draw chain miss in the constant cache)
  int64_t dims[kMaxOrder], lstride[kMaxOrder];
  const float* fac[kMaxOrder];
  int64_t coff[kMaxOrder];         // offset of mode k's staged CDF in the shared CDF area
  uint64_t T[kMaxOrder];
  int32_t start[kMaxOrder], len[kMaxOrder];
  double wblk;
  int64_t beff;
  int bad;
  double tol;
  unsigned long long carry;
  unsigned long long wtot[kPWThreads / 32];
  double red[kPWThreads / 32];
};

#define PW_MK(slot)                                 \
  do {                                              \
    if (mk && threadIdx.x == 0) mk[slot] = clock64(); \
    __syncwarp();                                     \
  } while (0)
// finer marks of thread 0 of CTA 0 (no warp sync; a second block of 32 slots per iteration: dbg[3072 + 32 s + slot])
#define PW_MK2(slot)                                               \
  do {                                                             \
    if (mk && threadIdx.x == 0) mk[2560 + (slot)] = clock64();     \
  } while (0)

// Two-level CDF search (no staging of whole CDFs): coarse[j] = the inclusive CDF at the end of 16-row block j
// (staged in shared memory), then the block's 16 entries straight from L2 -- the CDF rows of a mode, or, for the
// mode rebuilt in the previous iteration (pend), its raw q rows with the block's base coarse[j - 1].  Returns
// exactly the full search's i = #{i : CDF[i] <= r} and q_i (eq:ik under the contract of DESIGN.md section 4).
// Rows past I are padding of the 16-row allocations and are masked.
__device__ __forceinline__ void pw_cdf_search(const uint64_t* src, bool pend, const uint64_t* coarse, int ncb,
                                              int64_t I, uint64_t r, int64_t& i, uint64_t& qk) {
  // j = #{blocks whose inclusive end <= r}: a branch-free binary search with a fixed step count (every lane of a warp
  // walks the same instruction stream: no divergence per step)
  int j = 0;
  for (int step = 1 << (31 - __clz(ncb)); step > 0; step >>= 1) {
    const int c = j + step;
    const uint64_t v = coarse[min(c, ncb) - 1];
    j = (c <= ncb && v <= r) ? c : j;
  }
  if (j >= ncb) j = ncb - 1;  // T = 0 (degenerate table, the status is set): keep the addresses valid
  const uint64_t cb = coarse[j > 0 ? j - 1 : 0];  // unconditional load, then select
  const uint64_t base = j > 0 ? cb : 0ull;
  const int64_t lo = (int64_t)j * kPWRows;
  const int cnt = (int)cmin64(kPWRows, I - lo);
  uint64_t v[kPWRows];
#pragma unroll
  for (int t = 0; t < kPWRows; t += 2) {
    const ulonglong2 x = __ldcg(reinterpret_cast<const ulonglong2*>(src + lo + t));
    v[t] = x.x;
    v[t + 1] = x.y;
  }
  // idx = #{t < cnt : CDF[lo + t] <= r} and q of row lo + idx, by selects only (the CDF is monotone)
  int idx = 0;
  uint64_t c = base, qsel = 0, prev = base;
#pragma unroll
  for (int t = 0; t < kPWRows; ++t) {
    const uint64_t e = pend ? c + v[t] : v[t];  // the inclusive CDF at row lo + t
    const bool in = t < cnt, le = in && e <= r;
    qsel = (in && !le && idx == t) ? e - prev : qsel;
    prev = le ? e : prev;
    idx = le ? t + 1 : idx;
    c = e;
  }
  if (idx >= cnt) {  // r beyond the table (T = 0): the last row, q of it
    idx = cnt - 1;
    qsel = 0;
  }
  i = lo + idx;
  qk = qsel;
}

// the inclusive CDF at row x (block windows, eq:bik): coarse base + the block's entries up to x
__device__ __forceinline__ uint64_t pw_cdf_at(const uint64_t* src, bool pend, const uint64_t* coarse, int64_t x) {
  if (x < 0) return 0ull;
  const int j = (int)(x / kPWRows);
  if (!pend) return __ldcg(src + x);
  uint64_t c = j > 0 ? coarse[j - 1] : 0ull;
  for (int64_t t = (int64_t)j * kPWRows; t <= x; ++t) c += __ldcg(src + t);
  return c;
}

// NT: the tensor order as a compile-time constant (3: the benchmark shapes -- position loops unrolled, no run-time
// division by N - 1 on the draw chain) or 0 (any order up to kMaxOrder)
template <int NT>
static __device__ void pw_sample(const PWParams& p, int n, uint64_t r, unsigned char* sm, PWShared& ss, PWBulk& bk,
                                 long long* mk, int pend) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int N = NT > 0 ? NT : p.N, NP = N - 1, R = p.R, RP = zg_rp(R), nb4 = (R + 3) >> 2;
  const bool block = (p.strategy == 3 || p.strategy == 4);
  const int64_t bmax = p.bmax[n];
  const int nunits = pw_units_fib(bmax);
  const int nsamp = nunits < (int)gridDim.x ? nunits : (int)gridDim.x;  // CTAs with units (Gamma partials)
  if ((int)blockIdx.x >= nsamp) return;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    off = (off + 15) / 16 * 16;
    unsigned char* ptr = sm + off;
    off += bytes;
    return ptr;
  };
  int64_t cdf_elems = 0;
  if (p.strategy != 0)
    for (int k = 0; k < N; ++k)
      if (k != n) cdf_elems += p.dims[k];
  uint64_t* cdfs = reinterpret_cast<uint64_t*>(carve(sizeof(uint64_t) * (cdf_elems + kMaxOrder)));
  int32_t* sidx = reinterpret_cast<int32_t*>(carve(sizeof(int32_t) * kPWFib * NP));
  double* spt = reinterpret_cast<double*>(carve(sizeof(double) * kPWFib * NP));
  double* sw = reinterpret_cast<double*>(carve(sizeof(double) * kPWFib));
  float* zs = reinterpret_cast<float*>(carve(sizeof(float) * kPWFib * RP));
  const int GG = zg_groups(R, nth);
  float* red = reinterpret_cast<float*>(carve(sizeof(float) * (size_t)GG * R * R));
  float* gacc = reinterpret_cast<float*>(carve(sizeof(float) * R * R));
  {
    // coarse CDFs of the sampled modes (the inclusive CDF at the end of every 16-row block): for the mode rebuilt in
    // the previous iteration, the inclusive scan of its unit aggregates (its CDF rows are written concurrently, from
    // its raw q rows); for the others, every 16th row of their CDF.  All loads of a thread in flight at once.
    int64_t o = 0;
    for (int k = 0; k < N; ++k) {
      if (k == n || p.strategy == 0) {
        if (tid == 0) ss.T[k] = p.strategy == 0 ? (uint64_t)p.dims[k] : 0ull;
        continue;
      }
      const int ncb = (int)((p.dims[k] + kPWRows - 1) / kPWRows);
      uint64_t* co = cdfs + o;
      if (tid == 0) ss.coff[k] = o;
      if (k == pend) {  // warp 0: inclusive scan of the aggregates (unit order; exact integers): every load of a
                        // chunk of 256 units in flight at once (lane-owned runs of 8), then one warp scan
        if (tid < 32) {
          uint64_t carry = 0;
          for (int u0 = 0; u0 < ncb; u0 += 256) {
            uint64_t a[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {  // clamped unconditional loads, then masked
              const int u = u0 + 8 * tid + j;
              const uint64_t t = __ldcg(p.agg + (u < ncb ? u : ncb - 1));
              a[j] = u < ncb ? t : 0ull;
            }
#pragma unroll
            for (int j = 1; j < 8; ++j) a[j] += a[j - 1];
            uint64_t sc = a[7];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const uint64_t t = __shfl_up_sync(0xffffffffu, sc, d);
              if (tid >= d) sc += t;
            }
            const uint64_t ex = carry + sc - a[7];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const int u = u0 + 8 * tid + j;
              if (u < ncb) co[u] = ex + a[j];
            }
            carry += __shfl_sync(0xffffffffu, sc, 31);
          }
          if (tid == 0) ss.T[k] = carry;
        }
      } else {
        for (int j = tid; j < ncb; j += nth) co[j] = __ldcg(p.coarse[k] + j);  // contiguous: coalesced
        if (tid == 0) ss.T[k] = __ldcg(p.Ttot + k);
      }
      o += (ncb + 1) & ~1;
    }
    // the CTA's Gamma accumulator starts at zero (R > 32: the first unit's tensor-core partial is stored, not added)
    if (!(R > 32 && !(p.ablate & 0x200u)))
      for (int e = tid; e < R * R; e += nth) gacc[e] = 0.f;
  }
  __syncthreads();
  PW_MK(11);
  if (block && tid == 0) {  // window draws (eq:bik, Alg. 4, R2/R6): common to the whole batch
    double prod = 1.0;
    int64_t beff = 1;
    int pos = 0;
    for (int k = 0; k < N; ++k) {
      if (k == n) continue;
      const int64_t bk = p.window[n][pos];
      const uint64_t Tk = ss.T[k];
      const uint64_t rr = scale_draw(draw_word(p.seed, r, 0u, kPurposeWindow, (uint32_t)pos), Tk);
      const uint64_t* co = cdfs + ss.coff[k];
      const bool pk = (k == pend);
      const uint64_t* src = pk ? p.qraw : p.cdf[k];
      int64_t istar;
      uint64_t qdummy;
      pw_cdf_search(src, pk, co, (int)((p.dims[k] + kPWRows - 1) / kPWRows), p.dims[k], rr, istar, qdummy);
      const int64_t s0 = (istar / bk) * bk, e0 = min(s0 + bk, p.dims[k]);
      const uint64_t Q = pw_cdf_at(src, pk, co, e0 - 1) - pw_cdf_at(src, pk, co, s0 - 1);
      ss.start[pos] = (int32_t)s0;
      ss.len[pos] = (int32_t)(e0 - s0);
      const double pt = __ddiv_rn((double)((uint64_t)p.dims[k] * Q), (double)Tk);
      prod = (pos == 0) ? pt : __dmul_rn(prod, pt);
      beff *= (e0 - s0);
      ++pos;
    }
    ss.wblk = __ddiv_rn(1.0, prod);
    ss.beff = beff;
    if (blockIdx.x == 0) *p.beff = beff;
  } else if (!block && tid == 0 && blockIdx.x == 0) {
    *p.beff = p.B;
  }
  if (block) {  // (uniform) the windows of thread 0 for every thread
    __syncthreads();
    __syncwarp();
  }
  const int64_t beff = block ? ss.beff : p.B;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const int64_t b0 = (int64_t)u * kPWFib;
    const int nf = (int)cmin64(kPWFib, bmax - b0);
    if (!block) {
      // row-wise draws (eq:ik, R8): one thread per (fiber, position)
      const bool m2 = u == (int)blockIdx.x;
      if (m2) PW_MK2(0);
      for (int e = tid; e < nf * NP; e += nth) {
        const int lb = e / NP, pos = e % NP;
        const int k = pos < n ? pos : pos + 1;
        const uint64_t Tk = ss.T[k];
        const uint64_t rr = scale_draw(draw_word(p.seed, r, (uint32_t)(b0 + lb), kPurposeRow, (uint32_t)pos), Tk);
        if (m2 && mk && e == 0) {  // timing marks of element 0 (stores wait for their operands: issue order)
          ss.carry = rr;
          PW_MK2(1);
        }
        int64_t i;
        uint64_t qk;
        if (p.strategy == 0) {
          i = (int64_t)rr;
          qk = 1;
        } else {
          const bool pk = (k == pend);
          const int64_t Ik = ss.dims[k];
          pw_cdf_search(pk ? p.qraw : ss.cp[k], pk, cdfs + ss.coff[k], (int)((Ik + kPWRows - 1) / kPWRows), Ik, rr, i, qk);
        }
        sidx[e] = (int32_t)i;
        if (m2 && e == 0) PW_MK2(2);
        spt[e] = __ddiv_rn((double)((uint64_t)ss.dims[k] * qk), (double)Tk);
        if (m2 && e == 0) PW_MK2(3);
      }
      __syncthreads();
      if (m2) PW_MK2(4);
    }
    // per fiber: the exact weight (DESIGN.md section 4 order), indices, offset
    for (int lb = tid; lb < kPWFib; lb += nth) {
      const int64_t b = b0 + lb;
      if (lb >= nf || b >= beff) {
        sw[lb] = 0.0;
        for (int q = 0; q < NP; ++q) sidx[lb * NP + q] = 0;
        if (lb < nf) {
          p.fbase[b] = -1;
          p.w[b] = 0.0;
          for (int q = 0; q < NP; ++q) p.idx[b * NP + q] = 0;
        }
        continue;
      }
      double wv;
      if (!block) {
        double prod = spt[lb * NP];
        for (int pos = 1; pos < NP; ++pos) prod = __dmul_rn(prod, spt[lb * NP + pos]);
        wv = __ddiv_rn(1.0, __dmul_rn((double)p.B, prod));
      } else {
        uint32_t rem = (uint32_t)b;
        for (int q = 0; q < NP; ++q) {
          const uint32_t L = (uint32_t)ss.len[q];
          sidx[lb * NP + q] = ss.start[q] + (int32_t)(rem % L);
          rem /= L;
        }
        wv = ss.wblk;
      }
      sw[lb] = wv;
      p.w[b] = wv;
      int64_t offn = 0, jrow = 0, jmul = 1;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == n) continue;
        const int64_t ik = sidx[lb * NP + pos];
        p.idx[b * NP + pos] = (int32_t)ik;
        ++pos;
        offn += ik * ss.lstride[k];
        jrow += ik * jmul;
        jmul *= ss.dims[k];
      }
      p.fbase[b] = p.pitch[n] ? jrow * p.pitch[n] : offn;
    }
    __syncthreads();
    if (u == (int)blockIdx.x) PW_MK(12);
    // SKR rows (Alg. 1): z[lb][r] = prod_{k != n, ascending} A^(k)(i_k, r); all
    // factor loads of a thread's elements of one mode are issued before the products
    {
      constexpr int U = (kPWFib * kMaxRank + kPWThreads - 1) / kPWThreads;
      int lbu[U], ru[U];
      float z[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int e = tid + q * nth;
        lbu[q] = e / RP;
        ru[q] = e % RP;
        z[q] = (e < kPWFib * RP && lbu[q] < nf && ru[q] < R) ? 1.f : 0.f;
      }
      // two modes per round (one L2 round trip for N = 3), products in ascending mode order
      for (int pos = 0; pos < NP; pos += 2) {
        const int pos2 = pos + 1 < NP ? pos + 1 : pos;
        const int k = pos < n ? pos : pos + 1, k2 = pos2 < n ? pos2 : pos2 + 1;
        const float* F = ss.fac[k];
        const float* F2 = ss.fac[k2];
        float f[U], f2[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {  // every load issued (clamped address), then selected: no branch per load
          const int lb = lbu[q] < kPWFib ? lbu[q] : kPWFib - 1, rr = ru[q] < R ? ru[q] : R - 1;
          const float v = __ldcg(F + (int64_t)sidx[lb * NP + pos] * R + rr);
          const float v2 = __ldcg(F2 + (int64_t)sidx[lb * NP + pos2] * R + rr);
          f[q] = z[q] != 0.f ? v : 0.f;
          f2[q] = (z[q] != 0.f && pos2 != pos) ? v2 : 1.f;
        }
#pragma unroll
        for (int q = 0; q < U; ++q) z[q] = (z[q] * f[q]) * f2[q];
      }
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (tid + q * nth < kPWFib * RP) zs[tid + q * nth] = z[q];
    }
    __syncthreads();
    if (u == (int)blockIdx.x) PW_MK(13);
    // the tcgen05 A-operand images of the unit: zh / zl rows (zero past nf), one 16-byte chunk (4
    // consecutive fibers of one row) per task
    for (int e = tid; e < R * (kPWFib / 4); e += nth) {
      const int rr = e / (kPWFib / 4), l0 = 4 * (e % (kPWFib / 4));
      float h[4], l[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int lb = l0 + j;
        const float zw = lb < nf ? (float)((float)sw[lb] * zs[lb * RP + rr]) : 0.f;
        h[j] = __uint_as_float(__float_as_uint(zw) & 0xFFFFE000u);
        l[j] = zw - h[j];
      }
      *reinterpret_cast<float4*>(p.zimg + (zimg_off(b0 + l0, rr) >> 2)) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(p.zimg + (zimg_off(b0 + l0, 64 + rr) >> 2)) = make_float4(l[0], l[1], l[2], l[3]);
    }
    if (u == (int)blockIdx.x) PW_MK(23);
    // Gamma partial of the unit: sum_b (w_b z_b) z_b^T.  R > 32: on fp64 tensor cores (mma.sync m8n8k4 f64), 8x8
    // tiles I <= J one per warp, the unit's fibers in k-steps of 4 (products and sums in fp64: the fp32 operands
    // and w_b are exact there), each tile rounded once into the CTA's fp32 accumulator (both triangles).
    if (R > 32 && !(p.ablate & 0x200u)) {
      const int ncb = (R + 7) >> 3, ntile = ncb * (ncb + 1) / 2, lane = tid & 31, gr = lane >> 2, gc = lane & 3;
      for (int t = tid >> 5; t < ntile; t += nth >> 5) {
        int I = 0, rem = t;
        while (rem >= ncb - I) { rem -= ncb - I; ++I; }
        const int J = I + rem;
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < kPWFib; k0 += 4) {  // zs rows past nf and columns past R are zero, sw past nf too
          const int kk = k0 + gc;
          const double av = sw[kk] * (double)zs[kk * RP + 8 * I + gr], bv = (double)zs[kk * RP + 8 * J + gr];
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(d0), "+d"(d1)
                       : "d"(av), "d"(bv));
        }
        const int r1 = 8 * I + gr;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r2 = 8 * J + 2 * gc + i;
          if (r1 < R && r2 < R) {
            const float v = (float)(i ? d1 : d0);
            const bool fu = u == (int)blockIdx.x;  // the CTA's first unit: store (no zeroing pass)
            gacc[r1 * R + r2] = fu ? v : gacc[r1 * R + r2] + v;
            if (I != J) gacc[r2 * R + r1] = fu ? v : gacc[r2 * R + r1] + v;
          }
        }
      }
      __syncthreads();
      if (u == (int)blockIdx.x) PW_MK(24);
    } else {
      const int nblk = nb4 * (nb4 + 1) / 2;
      const int GE = nblk >= 64 ? 1 : GG;
      const int g = tid / nblk, blk = tid % nblk;
      if (g < GE) {
        int bi = 0, rem = blk;
        while (rem >= nb4 - bi) { rem -= nb4 - bi; ++bi; }
        const int bj = bi + rem;
        float acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = 0.f;
        // four fibers per round: every shared-memory load of the round issued before its FMAs (16-byte vectors:
        // 4 ceil(R/4) <= RP, always inside the padded row); fibers past nf have zero rows and weight
#pragma unroll 1
        for (int k0 = g; k0 < nf; k0 += 4 * GE) {
          float4 xv[4], yv[4];
          float wk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int kk = min(k0 + j * GE, kPWFib - 1);
            wk[j] = k0 + j * GE < nf ? (float)sw[kk] : 0.f;
            xv[j] = *reinterpret_cast<const float4*>(zs + kk * RP + 4 * bi);
            yv[j] = *reinterpret_cast<const float4*>(zs + kk * RP + 4 * bj);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float x[4] = {wk[j] * xv[j].x, wk[j] * xv[j].y, wk[j] * xv[j].z, wk[j] * xv[j].w};
            const float y[4] = {yv[j].x, yv[j].y, yv[j].z, yv[j].w};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int c = 0; c < 4; ++c) acc[a][c] = fmaf(x[a], y[c], acc[a][c]);
          }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int r1 = 4 * bi + a, r2 = 4 * bj + c;
            if (r1 < R && r2 < R) {
              if (GE == 1) {
                gacc[r1 * R + r2] += acc[a][c];
                if (bi != bj) gacc[r2 * R + r1] += acc[a][c];
              } else {
                red[(g * R + r1) * R + r2] = acc[a][c];
                if (bi != bj) red[(g * R + r2) * R + r1] = acc[a][c];
              }
            }
          }
      }
      __syncthreads();
      if (u == (int)blockIdx.x) PW_MK(24);
      if (GE > 1) {
        for (int e = tid; e < R * R; e += nth) {
          float s = red[e];
          for (int gg = 1; gg < GE; ++gg) s += red[gg * R * R + e];
          gacc[e] += s;
        }
        __syncthreads();
      }
    }
  }
  PW_MK(14);
  float* gcl = p.gcl + (int64_t)blockIdx.x * R * R;
  for (int e = tid; e < R * R; e += nth) gcl[e] = gacc[e];
}

// ------------------------------------------------------------------------------------------ phase G
struct PWBars {
  uint64_t xfull[16], xempty[16], sdone[4], mdone[4], afull[4], afree[4], accf, bc;
};

// Gamma = sum of the sampling CTAs' partials in CTA order; entries [e0, E) with stride es
__device__ __forceinline__ void pw_gamma_sum(const PWParams& p, int nsamp, int e0, int es) {
  const int E = p.R * p.R;
  for (int e = e0; e < E; e += es) {
    float v[16], s = 0.f;
    for (int c0 = 0; c0 < nsamp; c0 += 16) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {  // clamped unconditional loads (no branch per load), then masked
        const float t = __ldcg(p.gcl + (int64_t)(c0 + k < nsamp ? c0 + k : nsamp - 1) * E + e);
        v[k] = c0 + k < nsamp ? t : 0.f;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) s += v[k];  // CTA order; zeros past nsamp are exact
    }
    p.gam[e] = s;
  }
}

// the tcgen05 mainloop of gupdate_tc.cuh over this CTA's (I-tile, chunk) items; gs / gi: this CTA's
// running stage / item counters (the mbarrier phases continue across items and iterations)
static __device__ void pw_gather(const PWParams& p, int n, unsigned char* sm, PWBars& B, uint32_t tmem, uint32_t& gs,
                          uint32_t& gi, long long* mk) {
  constexpr int KS = kTCKS, NX = kTCNX, NP = kTCPairs, NZ = kTCNZ, TI = kGUTI;
  constexpr uint32_t A_BYTES = kTCABytes;
  constexpr uint32_t IDESC = umma_idesc_tf32_mn(128, 256) & ~((1u << 15) | (1u << 16));
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int R = p.R;
  const int64_t In = p.dims[n];
  const int tiles = (int)((In + TI - 1) / TI), CK = p.CK[n];
  const int64_t KB = p.KB[n], bmax = p.bmax[n];
  const int nitems = tiles * CK;
  const int nsamp = min(pw_units_fib(bmax), (int)gridDim.x);
  const float* X = p.Xg[n];
  const int64_t rowlen = p.rowlen[n];
  unsigned char* xsp = sm;
  unsigned char* xring = sm + NP * 2 * A_BYTES;
  unsigned char* zring = xring + NX * A_BYTES;
  const size_t body = (size_t)NP * 2 * A_BYTES + (size_t)NX * A_BYTES + (size_t)NZ * kTCZBytes;
  const size_t epi = (size_t)128 * kTCEpiStride * 4;
  int64_t* sfb = reinterpret_cast<int64_t*>(sm + (body > epi ? body : epi));
  // the Gamma sum's index space: lanes 1-31 of warp 12 of the CTAs with items, then every thread
  // of the CTAs without one
  const int with_items = min(nitems, (int)gridDim.x);
  const int gamma_stride = with_items * 31 + ((int)gridDim.x - with_items) * kPWThreads;
  if ((int)blockIdx.x >= nitems) {
    pw_gamma_sum(p, nsamp, with_items * 31 + ((int)blockIdx.x - nitems) * kPWThreads + tid, gamma_stride);
    return;
  }
  bool first = true;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int tile = item / CK, chunk = item % CK;
    const int64_t i0 = (int64_t)tile * TI, c0 = (int64_t)chunk * KB;
    const int nfib = (int)cmax64(0, cmin64(KB, bmax - c0));
    const int nst = (nfib + KS - 1) / KS;
    for (int64_t i = tid; i < nfib; i += kPWThreads) sfb[i] = __ldcg(p.fbase + c0 + i);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (mk && first && tid == 0) mk[25] = clock64();
    if (wid < 4) {
      // X loaders: 16-byte cp.async chunks of the sampled fiber segments (Alg. 5 TensorSamp)
      for (int st = 0; st < nst; ++st) {
        const uint32_t g = gs + st;
        const int slot = g % NX;
        if (g >= (uint32_t)NX) mbar_wait(&B.xempty[slot], ((g / NX) - 1) & 1);
        unsigned char* A = xring + slot * A_BYTES;
        const int f0 = st * KS;
#pragma unroll
        for (int rep = 0; rep < KS * 32 / 128; ++rep) {
          const int e = tid + 128 * rep;
          const int kk = e >> 5, j = e & 31;
          const int lb = f0 + kk;
          const int64_t fbv = sfb[lb < nfib ? lb : 0];  // unconditional load, then select
          const int64_t fb = lb < nfib ? fbv : -1;
          const int64_t r0 = i0 + 4 * j;
          if (fb >= 0 && r0 < rowlen && !(p.ablate & 2u)) cp_async16(A + kk * 512 + 16 * j, X + fb + r0, 16);
        }
        cp_async_mbar_arrive_noinc(&B.xfull[slot]);
      }
    } else if (wid <= 11) {
      // 3xTF32 split / transpose into the K-major swizzled {xh; xl} pair
      const int t = tid - 128;
      const int iq = t & 31, kq = t >> 5;
      for (int st = 0; st < nst; ++st) {
        const uint32_t g = gs + st;
        const int slot = g % NX, hb = g % NP;
        mbar_wait(&B.xfull[slot], (g / NX) & 1);
        if (mk && first && t == 0 && st == 0) mk[26] = clock64();
        if (g >= (uint32_t)NP) mbar_wait(&B.mdone[hb], ((g / NP) - 1) & 1);
        const float* A = reinterpret_cast<const float*>(xring + slot * A_BYTES);
        unsigned char* H = xsp + hb * 2 * A_BYTES;
        unsigned char* L = H + A_BYTES;
        const int f0 = st * KS;
        float x[4][4];
        for (int rep = (p.ablate & 64u) ? 0 : 1; rep < 2; ++rep) {  // timing experiment (64): the split twice
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int kk = 4 * kq + u, lb = f0 + kk;
          const bool ok = lb < nfib && sfb[lb] >= 0;
#pragma unroll
          for (int a = 0; a < 4; ++a) {  // load unconditionally (inside the ring), then select
            const float t = A[kk * 128 + iq + 32 * a];
            x[u][a] = ok ? t : 0.f;
          }
        }
        if (rep == 1) mbar_arrive(&B.xempty[slot]);
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const float4 h = make_float4(tf32_trunc(x[0][a]), tf32_trunc(x[1][a]), tf32_trunc(x[2][a]), tf32_trunc(x[3][a]));
          const float4 l = make_float4(x[0][a] - h.x, x[1][a] - h.y, x[2][a] - h.z, x[3][a] - h.w);
          const uint32_t o = kmaj_off(iq + 32 * a, 4 * kq);
          *reinterpret_cast<float4*>(H + o) = h;
          *reinterpret_cast<float4*>(L + o) = l;
        }
        }
        fence_proxy_async_smem();
        mbar_arrive(&B.sdone[hb]);
        if (mk && first && t == 0 && st == nst - 1) mk[27] = clock64();
      }
    } else if (wid == 12) {
      if (lane != 0) {
        if (first) pw_gamma_sum(p, nsamp, (int)blockIdx.x * 31 + lane - 1, gamma_stride);
      } else {
        for (int st = 0; st < nst; ++st) {
          const uint32_t g = gs + st;
          const int zs = g % NZ;
          if (g >= (uint32_t)NZ) mbar_wait(&B.afree[zs], ((g / NZ) - 1) & 1);
          const int64_t sb = (c0 + (int64_t)st * KS) / KS;
          if (p.ablate & 128u) {  // timing experiment: no A-image copy (stale images)
            mbar_arrive(&B.afull[zs]);
          } else {
            mbar_expect_tx(&B.afull[zs], kTCZBytes);
            bulk_g2s(zring + zs * kTCZBytes, p.zimg + sb * (kTCZBytes / 4), kTCZBytes, &B.afull[zs]);
          }
        }
      }
    } else if (wid == 13 && lane == 0) {
      const uint64_t dx = umma_desc_sw128(smem_u32(xsp), 16, 1024);
      const uint64_t dz = umma_desc_sw128(smem_u32(zring), 16, 1024);
      for (int st = 0; st < nst; ++st) {
        const uint32_t g = gs + st;
        const int hb = g % NP, as = g % NZ;
        mbar_wait(&B.sdone[hb], (g / NP) & 1);
        mbar_wait(&B.afull[as], (g / NZ) & 1);
        tc_fence_after();
        const uint64_t b = dx + ((uint64_t)(hb * 2 * A_BYTES) >> 4);
        const uint64_t a = dz + ((uint64_t)(as * kTCZBytes) >> 4);
#pragma unroll
        for (int k = 0; k < KS / 8; ++k) umma_tf32(tmem, a + 2 * k, b + 2 * k, IDESC, (st > 0 || k > 0) ? 1u : 0u);
        if (p.ablate & 32u)  // timing experiment: every MMA twice
          for (int k = 0; k < KS / 8; ++k) umma_tf32(tmem, a + 2 * k, b + 2 * k, IDESC, 1u);
        umma_commit(&B.mdone[hb]);
        umma_commit(&B.afree[as]);
      }
      if (nst > 0) umma_commit(&B.accf);
    }
    __syncthreads();
    // epilogue: E[L][i] = D[L][i] + D[L][128 + i] (x = xh + xl) staged in shared memory, then
    // M^T[r][i] = E[r][i] + E[64 + r][i] (zw = zh + zl) -> the split-K workspace
    if (nst > 0) mbar_wait(&B.accf, gi & 1);
    tc_fence_after();
    if (mk && first && tid == 0) mk[28] = clock64();
    float* E = reinterpret_cast<float*>(sm);
    if (wid >= 4 && wid <= 11) {
      const int L = 32 * (wid & 3) + lane, hh = (wid - 4) >> 2;
      const uint32_t trow = tmem + ((uint32_t)(32 * (wid & 3)) << 16);
#pragma unroll 1
      for (int c = 64 * hh; c < 64 * hh + 64; c += 16) {
        float v1[16], v2[16];
        if (nst > 0) {
          tmem_ld16(trow + (uint32_t)c, v1);
          tmem_ld16(trow + 128u + (uint32_t)c, v2);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) v1[j] = v2[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < 16; j += 4)
          *reinterpret_cast<float4*>(E + L * kTCEpiStride + c + j) =
              make_float4(v1[j] + v2[j], v1[j + 1] + v2[j + 1], v1[j + 2] + v2[j + 2], v1[j + 3] + v2[j + 3]);
      }
    }
    tc_fence_before();
    __syncthreads();
    {
      const int nrow = (int)cmax64(0, cmin64(TI, In - i0));
      float* part = p.Mpart + ((int64_t)tile * CK + chunk) * R * TI;
      for (int e = tid; e < R * (TI / 4); e += kPWThreads) {
        const int r = e / (TI / 4), i = 4 * (e % (TI / 4));
        const float4 a = *reinterpret_cast<const float4*>(E + r * kTCEpiStride + i);
        const float4 b = *reinterpret_cast<const float4*>(E + (64 + r) * kTCEpiStride + i);
        const float4 s = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
        if (i + 4 <= nrow) {
          *reinterpret_cast<float4*>(part + r * TI + i) = s;
        } else {
          if (i < nrow) part[r * TI + i] = s.x;
          if (i + 1 < nrow) part[r * TI + i + 1] = s.y;
          if (i + 2 < nrow) part[r * TI + i + 2] = s.z;
        }
      }
    }
    gs += nst;
    if (nst > 0) ++gi;
    if (mk && first && tid == 0) mk[29] = clock64();
    first = false;
    __syncthreads();  // the ring / staging area is rewritten by the next item
  }
}

// ------------------------------------------------------------------------------------------ phase U
// rows [r0, r0 + nr) of A^(n): M (chunk order), G = A Gamma - M, update; leaves the new rows in sA
// (stride R+1) and writes the unit's table partial
static __device__ void pw_update_unit(const PWParams& p, int n, int unit, double alpha, float* sA, float* sS, float* sM,
                               const float* sG, double* sgp_d, PWShared& ss, PWBulk* bkw, long long* mk) {
  float* sgp_f = reinterpret_cast<float*>(sgp_d);  // scratch (16-byte aligned): the G partials, then the Gram's
  constexpr int TI = kGUTI;
  const int R = p.R, RS = R + 1, AS = R, tid = threadIdx.x, nth = blockDim.x, nb4 = (R + 3) >> 2;
  const int64_t In = p.dims[n];
  const int64_t r0 = (int64_t)unit * kPWRows;
  const int nr = (int)cmin64(kPWRows, In - r0);
  const int CK = p.CK[n];
  float* A = p.factors[n];
  float* S = p.S[n];
  // the unit's rows of A and S: contiguous, 16-byte L2 copies all in flight (rows written earlier in
  // this launch); stride R in shared memory
  cpcg_bytes(sA, A + r0 * R, (int64_t)nr * R * 4, tid, nth);
  if (p.rule == 1) cpcg_bytes(sS, S + r0 * R, (int64_t)nr * R * 4, tid, nth);
  {  // M = sum of the chunk partials, in chunk order (16-byte vectors of 4 consecutive rows)
    const int64_t tile = r0 / TI, lr0 = r0 % TI;
    const int ng = (nr + 3) / 4;
    for (int t = tid; t < R * ng; t += nth) {
      const int r = t / ng, gq = t % ng;
      const float* base = p.Mpart + ((tile * CK) * R + r) * TI + lr0 + gq * 4;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      for (int c0 = 0; c0 < CK; c0 += 16) {  // CK <= 16 at one wave: every chunk's load in flight at once
        float4 ld[16];
#pragma unroll
        for (int k = 0; k < 16; ++k)  // clamped unconditional loads, then masked adds (chunk order)
          ld[k] = __ldcg(reinterpret_cast<const float4*>(base + (int64_t)min(c0 + k, CK - 1) * R * TI));
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (c0 + k < CK) {
            acc[0] += ld[k].x;
            acc[1] += ld[k].y;
            acc[2] += ld[k].z;
            acc[3] += ld[k].w;
          }
      }
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (gq * 4 + w < nr) sM[(gq * 4 + w) * RS + r] = acc[w];
    }
  }
  PW_MK2(7);
  cp_async_wait<0>();
  PW_MK2(8);
  if (bkw) pw_bulk_wait(*bkw);  // Gamma (first unit of the CTA)
  PW_MK2(9);
  __syncthreads();
  PW_MK(15);
  // G = A Gamma - M.  R > 32: on fp64 tensor cores (mma.sync m8n8k4 f64; 8x8 tiles of the 16 x R block, one per warp,
  // the R-long contraction in k-steps of 4, the fp32 operands exact in fp64), G = (float)(A Gamma - M) rounded once,
  // left in sM.  Else: task = (4 x 4 block of G, k group); KG groups split the R-long contraction (short dependent
  // chains), their partials summed in group order
  if (R > 32 && !(p.ablate & 0x200u)) {
    const int ncb = (R + 7) >> 3, lane = tid & 31, gr = lane >> 2, gc = lane & 3;
    const int kr4 = (R + 3) & ~3;
    for (int t = tid >> 5; t < 2 * ncb; t += nth >> 5) {
      const int rb = t / ncb, cb = t % ncb;
      const int row = 8 * rb + gr, col = 8 * cb + gr, rowc = min(row, nr - 1), colc = min(col, R - 1);
      double d0 = 0.0, d1 = 0.0;
#pragma unroll 4
      for (int k0 = 0; k0 < kr4; k0 += 4) {  // A[r][k] = sA[row][k], B[k][n] = Gamma[k][col]; clamped loads, then select
        const int k = k0 + gc, kc = min(k, R - 1);
        const float av = sA[rowc * AS + kc], bv = sG[kc * R + colc];
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(d0), "+d"(d1)
                     : "d"((row < nr && k < R) ? (double)av : 0.0), "d"((k < R && col < R) ? (double)bv : 0.0));
      }
      const int c0 = 8 * cb + 2 * gc;
      __syncwarp();
      if (row < nr) {
        if (c0 < R) sM[row * RS + c0] = (float)(d0 - (double)sM[row * RS + c0]);
        if (c0 + 1 < R) sM[row * RS + c0 + 1] = (float)(d1 - (double)sM[row * RS + c0 + 1]);
      }
    }
  } else {
    const int nbt = ((nr + 3) >> 2) * nb4;
    const int KG = max(1, min(kPWUpdKG, nth / max(1, nbt)));
    const int kper = (R + KG - 1) / KG;
    float* redG = sgp_f;  // [KG][16][R]
    for (int t = tid; t < nbt * KG; t += nth) {
      const int g = t / nbt, bt = t % nbt;
      const int a0 = 4 * (bt / nb4), q0 = 4 * (bt % nb4);
      const int k0 = g * kper, k1 = min(R, k0 + kper);
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.f;
      for (int k = k0; k < k1; ++k) {
        float x[4], y[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) x[a] = sA[(a0 + a) * AS + k];  // rows < 16: inside the buffer
#pragma unroll
        for (int c = 0; c < 4; ++c) y[c] = sG[k * R + min(q0 + c, R - 1)];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fmaf(x[a], y[c], acc[a][c]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (q0 + c < R) redG[(g * kPWRows + a0 + a) * R + q0 + c] = acc[a][c];
    }
    __syncthreads();
    for (int e = tid; e < nr * R; e += nth) {
      const int il = e / R, r = e % R;
      float sum = 0.f;
      for (int g = 0; g < KG; ++g) sum += redG[(g * kPWRows + il) * R + r];
      sM[il * RS + r] = sum - sM[il * RS + r];
    }
  }
  __syncthreads();
  // fixed (eq:proposed) / adaptive (eq:etaada/eq:Aada, :531-537, R12) update; thread -> (row
  // tid / 28, columns tid % 28 + 28 j): 448 = 16 rows x 28, no run-time division per element
  static_assert(kPWThreads == kPWRows * 28, "16 rows x 28 columns per pass");
  const int ilt = tid / 28, rt0 = tid % 28;
  for (int r = rt0, il = ilt; il < nr && r < R; r += 28) {
    const int64_t gi = (r0 + il) * R + r;
    const float g = sM[il * RS + r];
    p.Gout[gi] = g;
    const float a = sA[il * AS + r];
    float an = a;
    if (p.rule == 0) {
      an = a - (float)alpha * g;
    } else {
      const float sv = sS[il * AS + r] + g * g;
      S[gi] = sv;
      if (sv > 0.f) {
        float step;
        if (p.eps == 0.0) step = (float)p.eta / sqrtf((float)p.b + sv);
        else step = (float)p.eta / (float)pow((double)((float)p.b + sv), 0.5 + p.eps);
        an = a - step * g;
      }
    }
    A[gi] = an;
    sA[il * AS + r] = an;
  }
  __syncthreads();
  PW_MK(16);
  // table partials of the new rows (R9)
  if ((p.strategy == 1 || p.strategy == 3) && !(p.ablate & 8u)) {  // leverage: partial fp64 Gram, packed upper triangle
    // task = (4 x 4 block bi <= bj, row group): the rows split into RG groups (short chains), an fp64
    // copy of the rows (converted once), the group partials summed in group order
    const int P = R * (R + 1) / 2;
    const int RD = ut_rd(R);
    const int nblk = nb4 * (nb4 + 1) / 2;
    const int RG = max(1, min(4, nth / nblk));
    double* sAd = sgp_d;                              // [16][RD], zero past R
    double* redP = sgp_d + kPWRows * RD;              // [RG][P]
    if (R > 32 && !(p.ablate & 0x200u)) {
      // R > 32 on fp64 tensor cores (mma.sync m8n8k4 f64): the unit's Gram = A_u^T A_u as 8x8 tiles I <= J (one
      // per warp, round robin), the 16 rows in four k-steps, the fp32 rows read as operands directly (exact in fp64);
      // stored straight into the packed pair partials
      const int ncb = (R + 7) >> 3, ntile = ncb * (ncb + 1) / 2, lane = tid & 31, gr = lane >> 2, gc = lane & 3;
      double* gp = p.gpart + unit;  // [P][gstride]: the pair sums read each pair's unit partials contiguously
      for (int t = tid >> 5; t < ntile; t += nth >> 5) {
        int I = 0, rem = t;
        while (rem >= ncb - I) { rem -= ncb - I; ++I; }
        const int J = I + rem;
        const int ca = 8 * I + gr, cb = 8 * J + gr, cac = min(ca, R - 1), cbc = min(cb, R - 1);
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < kPWRows; k0 += 4) {  // A[r][k] = A_u[k][8I + r], B[k][n] = A_u[k][8J + n]
          const int kr = k0 + gc;
          const float av = sA[kr * AS + cac], bv = sA[kr * AS + cbc];  // rows < 16: inside the buffer; clamped
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(d0), "+d"(d1)
                       : "d"((ca < R && kr < nr) ? (double)av : 0.0), "d"((cb < R && kr < nr) ? (double)bv : 0.0));
        }
        const int r1 = 8 * I + gr;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int r2 = 8 * J + 2 * gc + i;
          if (r1 < R && r2 < R && r1 <= r2) gp[(int64_t)(r1 * R - r1 * (r1 - 1) / 2 + (r2 - r1)) * p.gstride] = i ? d1 : d0;
        }
      }
    } else {
    for (int c = tid % 28, il = tid / 28; c < RD; c += 28) {  // 16 rows x 28 threads (no division per element)
      const float v = sA[il * AS + min(c, R - 1)];  // rows < 16: inside the buffer
      sAd[il * RD + c] = (il < nr && c < R) ? (double)v : 0.0;
    }
    __syncthreads();
    for (int t = tid; t < nblk * RG; t += nth) {
      const int g = t / nblk, blk = t % nblk;
      int bi = 0, rem = blk;
      while (rem >= nb4 - bi) { rem -= nb4 - bi; ++bi; }
      const int bj = bi + rem;
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
      for (int il = g; il < nr; il += RG) {
        const double2 x01 = *reinterpret_cast<const double2*>(sAd + il * RD + 4 * bi);
        const double2 x23 = *reinterpret_cast<const double2*>(sAd + il * RD + 4 * bi + 2);
        const double2 y01 = *reinterpret_cast<const double2*>(sAd + il * RD + 4 * bj);
        const double2 y23 = *reinterpret_cast<const double2*>(sAd + il * RD + 4 * bj + 2);
        const double x[4] = {x01.x, x01.y, x23.x, x23.y}, y[4] = {y01.x, y01.y, y23.x, y23.y};
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
          if (r1 < R && r2 < R && r1 <= r2) redP[g * P + r1 * R - r1 * (r1 - 1) / 2 + (r2 - r1)] = acc[a][c];
        }
    }
    __syncthreads();
    double* gp = p.gpart + unit;  // [P][gstride]: the pair sums read each pair's unit partials contiguously
    for (int e = tid; e < P; e += nth) {
      double sum = 0.0;
      for (int g = 0; g < RG; ++g) sum += redP[g * P + e];
      gp[(int64_t)e * p.gstride] = sum;
    }
    }
  } else if (p.strategy == 2 || p.strategy == 4) {  // Euclidean: row norms + the unit's partial ||A||^2
    double acc = 0.0;
    for (int il = tid; il < nr; il += nth) {
      double rs = 0.0;
      for (int c = 0; c < R; ++c) rs += (double)sA[il * AS + c] * (double)sA[il * AS + c];
      p.rownorm[r0 + il] = rs;
      acc += rs;
    }
    __syncwarp();  // reconverged: a diverged warp runs every shuffle on the slow collective path
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) ss.red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < nth / 32; ++w) t += ss.red[w];
      p.gpart[unit] = t;
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------ phase Q
// scores + quantisation of the unit's rows, look-back prefix, CDF rows
static __device__ void pw_table_unit(const PWParams& p, int n, int unit, int nunits, uint32_t tag, const double* Wm,
                                     int rank, double fro, int bad0, double* Ad, const float* sAu, PWShared& ss,
                                     long long* mk) {
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int R = p.R, RS = R + 1, RD = ut_rd(R);
  const bool lev = (p.strategy == 1 || p.strategy == 3);
  const int64_t In = p.dims[n];
  const int64_t r0 = (int64_t)unit * kPWRows;
  const int nr = (int)cmin64(kPWRows, In - r0);
  __shared__ double s_p[kPWRows];
  __shared__ unsigned long long s_q[kPWRows];
  __shared__ int s_badu;
  if (tid == 0) s_badu = bad0;
  if (lev) {
    // the unit's new rows in fp64 (stride RD, zero padded): from this CTA's own update phase (sAu, stride
    // R, still in shared memory when this is the CTA's last unit) or re-read through L2
    for (int c = tid % 28, il = tid / 28; c < RD; c += 28) {  // 16 rows x 28 threads (no division per element)
      const int ilc = min(il, nr - 1), cc = min(c, R - 1);  // clamped, then select
      const float v = sAu ? sAu[ilc * R + cc] : __ldcg(p.factors[n] + (r0 + ilc) * R + cc);
      Ad[il * RD + c] = (il < nr && c < R) ? (double)v : 0.0;
    }
    __syncthreads();
    // l_i = a_i^T W a_i: warp w takes rows 2w, 2w + 1; lane c holds columns c and c + 32 of y = W a
    // (W symmetric: W_kc read along a row of the inverse, consecutive lanes -> consecutive words), k split
    // into even / odd chains, then l = sum_c a_c y_c by a fixed xor-shuffle tree (deterministic)
    if (R > 32 && !(p.ablate & 0x210u)) {
      // R > 32 on fp64 tensor cores (mma.sync m8n8k4 f64): Y = A_u W as 8x8 tiles (rows 8 rb.., columns 8 cb..),
      // one tile per warp, the k-steps chained in order; l_i = sum_c a_ic y_ic: per tile a quad xor-tree over
      // its 8 columns, then the column blocks summed in order (deterministic)
      __shared__ double s_part[kMaxRank / 8][kPWRows];
      const int ncb = (R + 7) >> 3, gr = lane >> 2, gc = lane & 3;
      for (int t = wid; t < 2 * ncb; t += nth >> 5) {
        const int rb = t / ncb, cb = t % ncb;
        const int col = 8 * cb + gr, colc = min(col, R - 1);
        double y0 = 0.0, y1 = 0.0;
        const double* arow = Ad + (8 * rb + gr) * RD;
#pragma unroll 4
        for (int k0 = 0; k0 < RD; k0 += 4) {
          const int kr = k0 + gc, krc = min(kr, R - 1);
          const double wv = Wm[krc * RS + colc];  // clamped unconditional load, then select
          const double bv = (kr < R && col < R) ? wv : 0.0;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                       : "+d"(y0), "+d"(y1)
                       : "d"(arow[k0 + gc]), "d"(bv));
        }
        // lane (gr, gc) holds y[8 rb + gr][8 cb + 2 gc + {0, 1}] (Ad is zero past R and past nr)
        double part = arow[8 * cb + 2 * gc] * y0 + arow[8 * cb + 2 * gc + 1] * y1;
        if (8 * cb + 2 * gc >= RD) part = 0.0;  // columns past the padded row (R > RD - 8)
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        if (gc == 0) s_part[cb][8 * rb + gr] = part;
      }
      __syncthreads();
      if (tid < nr) {
        double l = 0.0;
        for (int cb = 0; cb < ncb; ++cb) l += s_part[cb][tid];
        s_p[tid] = rank > 0 ? fmax(l, 0.0) / (double)rank : 0.0;
      }
    } else if (wid < ((nr + 1) >> 1) && !(p.ablate & 16u)) {
      const int il = 2 * wid;
      const double* a0 = Ad + il * RD;
      const double* a1 = a0 + RD;  // row il + 1 < 16: inside the buffer (zeros past nr)
      const int c0 = lane, c1 = lane + 32;
      const int c0c = min(c0, R - 1), c1c = min(c1, R - 1);
      double y[2][2][2] = {};  // [row][column][k parity]
      if (R > 32) {
#pragma unroll 2
        for (int k = 0; k < R; ++k) {
          const int pk = k & 1;
          const double x0 = a0[k], x1 = a1[k];
          const double w0 = Wm[k * RS + c0c], w1 = Wm[k * RS + c1c];
          y[0][0][pk] = fma(w0, x0, y[0][0][pk]);
          y[0][1][pk] = fma(w1, x0, y[0][1][pk]);
          y[1][0][pk] = fma(w0, x1, y[1][0][pk]);
          y[1][1][pk] = fma(w1, x1, y[1][1][pk]);
        }
      } else {
#pragma unroll 2
        for (int k = 0; k < R; ++k) {
          const int pk = k & 1;
          const double x0 = a0[k], x1 = a1[k];
          const double w0 = Wm[k * RS + c0c];
          y[0][0][pk] = fma(w0, x0, y[0][0][pk]);
          y[1][0][pk] = fma(w0, x1, y[1][0][pk]);
        }
      }
      double l0 = 0.0, l1 = 0.0;
      if (c0 < R) {
        l0 = a0[c0] * (y[0][0][0] + y[0][0][1]);
        l1 = a1[c0] * (y[1][0][0] + y[1][0][1]);
      }
      if (c1 < R) {
        l0 += a0[c1] * (y[0][1][0] + y[0][1][1]);
        l1 += a1[c1] * (y[1][1][0] + y[1][1][1]);
      }
      __syncwarp();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      }
      if (lane == 0) {
        s_p[il] = rank > 0 ? fmax(l0, 0.0) / (double)rank : 0.0;
        if (il + 1 < nr) s_p[il + 1] = rank > 0 ? fmax(l1, 0.0) / (double)rank : 0.0;
      }
    }
  } else if (tid < nr) {
    s_p[tid] = fro > 0.0 ? __ldcg(p.rownorm + r0 + tid) / fro : 0.0;
  }
  __syncthreads();
  if (tid < nr) {
    const double pv = s_p[tid];
    unsigned long long qv = 0;
    if (!(pv == pv) || pv > 2.0) {
      atomicOr(&s_badu, 8);
    } else if (pv > 0.0) {
      const double s = rint(pv * 4294967296.0);
      qv = (s < 1.0) ? 1ull : (unsigned long long)s;
    }
    p.pprob[n][r0 + tid] = pv;
    s_q[tid] = qv;
  }
  __syncthreads();
  PW_MK(21);
  // the unit's raw q rows (into its CDF rows, converted by pw_table_prefix), aggregate and bad bits:
  // plain stores, published for the whole CTA by one release on the arrival counter (kernel)
  if (tid < 32) {  // warp 0: raw q rows, the unit aggregate by a xor tree (exact integers: any order)
    unsigned long long a = tid < nr ? s_q[tid] : 0ull;
    if (tid < nr) p.qraw[r0 + tid] = a;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (tid == 0) p.agg[unit] = a;
  }
  if (tid == 0) {
    p.aggf[2 * unit] = (unsigned)s_badu;
    // a bad table is visible to every CTA as soon as the arrivals are (the launch stops before drawing from it)
    if (s_badu) atomicCAS(p.status, 0, (s_badu & 8) ? -8 : -3);
  }
  __syncthreads();
}

// after every unit of an iteration has published (arrival counter; run during the next sampling phase): the exclusive prefix of
// the unit over the preceding units' aggregates (plain L2 loads, all in flight; exact integer sums in any
// order) + the unit's inclusive scan -> CDF rows; the last unit writes T and the table status
static __device__ void pw_table_prefix(const PWParams& p, int n, int unit, int nunits, PWShared& ss) {
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int64_t In = p.dims[n];
  const int64_t r0 = (int64_t)unit * kPWRows;
  const int nr = (int)cmin64(kPWRows, In - r0);
  unsigned long long pre = 0;
  unsigned badv = 0;
  for (int u = tid; u < unit; u += nth) {
    pre += __ldcg(p.agg + u);
    badv |= __ldcg(p.aggf + 2 * u);
  }
  if (unit == nunits - 1)  // the last unit also collects its own bad bits
    for (int u = tid; u == unit; u += nth) badv |= __ldcg(p.aggf + 2 * u);
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    pre += __shfl_xor_sync(0xffffffffu, pre, o);
    badv |= __shfl_xor_sync(0xffffffffu, badv, o);
  }
  if (lane == 0) {
    ss.wtot[wid] = pre;
    ss.red[wid] = __longlong_as_double((long long)badv);
  }
  __syncthreads();
  if (wid == 0) {  // predecessors' total + the unit's inclusive scan -> CDF rows (warp 0)
    __syncwarp();
    unsigned long long t = lane < nth / 32 ? ss.wtot[lane] : 0ull;
    unsigned bb = lane < nth / 32 ? (unsigned)__double_as_longlong(ss.red[lane]) : 0u;
    unsigned long long c = lane < nr ? __ldcg(p.qraw + r0 + min(lane, nr - 1)) : 0ull;  // the unit's raw q
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t += __shfl_xor_sync(0xffffffffu, t, o);
      bb |= __shfl_xor_sync(0xffffffffu, bb, o);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, c, o);
      if (lane >= o) c += v;
    }
    c += t;
    if (lane < nr) p.cdf[n][r0 + lane] = c;
    if (lane == nr - 1) p.coarse[n][unit] = c;  // the inclusive CDF at the unit's last row
    if (unit == nunits - 1 && lane == nr - 1) {  // the last unit: T and the table status
      p.Ttot[n] = c;
      int st = 0;
      if (bb & 8) st = -8;
      else if ((bb & 2) || c == 0) st = -3;
      if (st != 0) atomicCAS(p.status, 0, st);
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------------------ trace
static __device__ void pw_trace(const PWParams& p, int s, int n, uint64_t r) {
  const int64_t slot = p.tr.first + s;
  if (slot >= p.tr.cap) return;
  unsigned char* base = p.tr.base + slot * p.tr.stride;
  const int NP = p.N - 1, R = p.R;
  const int64_t bm = p.bmax[n], In = p.dims[n];
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, ts = (int64_t)gridDim.x * blockDim.x;
  int32_t* ti = reinterpret_cast<int32_t*>(base + p.tr.o_idx);
  double* tw = reinterpret_cast<double*>(base + p.tr.o_w);
  float* tA = reinterpret_cast<float*>(base + p.tr.o_A);
  float* tS = reinterpret_cast<float*>(base + p.tr.o_S);
  uint64_t* tc = reinterpret_cast<uint64_t*>(base + p.tr.o_cdf);
  int64_t* tm = reinterpret_cast<int64_t*>(base + p.tr.o_meta);
  for (int64_t e = t0; e < bm * NP; e += ts) ti[e] = __ldcg(p.idx + e);
  for (int64_t e = t0; e < bm; e += ts) tw[e] = __ldcg(p.w + e);
  for (int64_t e = t0; e < In * R; e += ts) {
    tA[e] = __ldcg(p.factors[n] + e);
    if (p.rule == 1) tS[e] = __ldcg(p.S[n] + e);
  }
  for (int64_t e = t0; e < In; e += ts) tc[e] = __ldcg(p.cdf[n] + e);
  if (t0 == 0) {
    tm[0] = n;
    tm[1] = (int64_t)r;
    tm[2] = __ldcg(p.beff);
    tm[3] = 0;
  }
}

// ------------------------------------------------------------------------------------------ kernel
#define PW_MARK(slot)                                                                              \
  do {                                                                                             \
    if (p.dbg && tid == 0 && s < 8) {                                                              \
      const long long t_ = clock64();                                                              \
      if (blockIdx.x == 0) p.dbg[512 + 32 * s + (slot)] = t_;                                      \
      if (blockIdx.x < 160) p.dbg[4096 + ((int64_t)s * 160 + blockIdx.x) * 32 + (slot)] = t_;      \
    }                                                                                              \
    __syncwarp();                                                                                  \
  } while (0)

// ------------------------------------------------------------------------------------------ inverse (R > 32)
// The same symmetric sweep (natural pivot order, reading R4(b)) in 8-pivot blocks on fp64 tensor cores (mma.sync
// m8n8k4 f64) with a look-ahead pivot warp.  The RMAX x RMAX matrix lives in DMMA accumulator fragments: the
// upper-triangle 8x8 tiles round robin over warps 1..13 (the owners).  Warp 0 (the pivot warp) runs the serial
// chain: it sweeps the 8x8 pivot block B_kb in registers (one pivot per step, shuffles), publishes -B_kb^-1, and
// forms the NEXT pivot block itself, B_kb+1 = D - Q^T B_kb^-1 Q (Q: the published block row's next column block,
// D: the next diagonal tile as published) with the same DMMA sequence the owners apply to that tile (bitwise the
// same values), so it sweeps B_kb+1 while the owners form F = B^-1 M_P,: (one column block per warp, 2 DMMA) and
// update their tiles (C -= M_:,P F, 2 DMMA; the pivot row / column blocks <- F / F^T, the pivot block <- -B^-1)
// and publish the next block row.  Block operations = the sweep operator on the pivot block (Goodnight 1979), so
// the result is the natural-order sweep's to rounding.  Returns |S| = R, or -1 when a pivot fails the single-pivot
// rule (d > tol, checked per pivot inside the blocks): the caller then runs grp_sweep_inverse from the Gram.
// Measured (tools/micro/dmma_la.cu, R = 50): 14.8k vs 18.2k cycles for the 2x2-pivot register sweep.
struct PWInvBars {
  uint64_t rows[kMaxRank / 8], binv[kMaxRank / 8];
};
__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__host__ __device__ constexpr size_t pw_dinv_bytes(int rmax) {  // Prow, Dd, Sw, Fb, scratch (doubles)
  return sizeof(double) * ((size_t)(rmax / 8) * 8 * (rmax + 2) + 2 * (size_t)(rmax / 8) * 64 + 8 * (size_t)(rmax + 2) + 64);
}
template <int RMAX>
__device__ int dmma_sweep_inverse(double* Gm, const double* gpk, int R, double tol, double* buf, PWInvBars& bars,
                                  int* s_fail) {
  constexpr int NB = RMAX / 8, NT = NB * (NB + 1) / 2, NO = kPWThreads / 32 - 1, TPW = (NT + NO - 1) / NO,
                LD = RMAX + 2;
  static_assert(RMAX % 8 == 0 && NB <= NO, "8x8 tiles");
  double* Prow = buf;                   // [NB][8][LD] block row kb as published
  double* Dd = Prow + NB * 8 * LD;      // [NB][64] diagonal tile kb + 1 as published with block row kb
  double* Sw = Dd + NB * 64;            // [NB][64] -B_kb^-1
  double* Fb = Sw + NB * 64;            // [8][LD] F of the current step
  double* scr = Fb + 8 * LD;            // [64] the pivot warp's scratch
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, gr = lane >> 2, gc = lane & 3, RS = R + 1;
  if (tid == 0) {
    *s_fail = 0;
    for (int k = 0; k < NB; ++k) {
      mbar_init(&bars.rows[k], 32 * NO);
      mbar_init(&bars.binv[k], 32);
    }
  }
  int tI[TPW], tJ[TPW];
  double c0[TPW], c1[TPW];
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int t = (w - 1) + NO * j;
    int I = 0, rem = t;
    while (I < NB && rem >= NB - I) { rem -= NB - I; ++I; }
    tI[j] = (w >= 1 && t < NT) ? I : -1;
    tJ[j] = I + rem;
    const int r = 8 * I + gr, c = 8 * tJ[j] + 2 * gc;
    const int rc = min(r, R - 1), cc0 = min(c, R - 1), cc1 = min(c + 1, R - 1);
    // the packed upper triangle (row a <= column b at a R - a (a - 1) / 2 + b - a); clamped, then select (identity
    // past R)
    auto pk = [&](int a, int b) { return gpk[(a <= b) ? a * R - a * (a - 1) / 2 + (b - a) : b * R - b * (b - 1) / 2 + (a - b)]; };
    const double g0 = pk(rc, cc0), g1 = pk(rc, cc1);
    c0[j] = tI[j] < 0 ? 0.0 : (r < R && c < R) ? g0 : (r == c ? 1.0 : 0.0);
    c1[j] = tI[j] < 0 ? 0.0 : (r < R && c + 1 < R) ? g1 : (r == c + 1 ? 1.0 : 0.0);
  }
  __syncthreads();
  // the Gram's entry (r, c) as the tiles start (identity past R)
  auto gval = [&](int r, int c) {
    const int rc = min(r, R - 1), cc = min(c, R - 1);
    const int a = rc <= cc ? rc : cc, b = rc <= cc ? cc : rc;
    const double v = gpk[a * R - a * (a - 1) / 2 + (b - a)];  // clamped, then select
    return (r < R && c < R) ? v : (r == c ? 1.0 : 0.0);
  };
  if (w == 0) {  // ---------------- the pivot warp
    // block 0 and its Schur step read the Gram itself (the same values the owners publish): no wait to start
    double b0 = gval(gr, 2 * gc), b1 = gval(gr, 2 * gc + 1);
#pragma unroll 1
    for (int kb = 0; kb < NB; ++kb) {
      bool ok = true;
#pragma unroll
      for (int k = 0; k < 8; ++k) {  // the pivot block's sweep, one pivot per step
        const double d = __shfl_sync(0xffffffffu, (k & 1) ? b1 : b0, 4 * k + (k >> 1));
        const double rk0 = __shfl_sync(0xffffffffu, b0, 4 * k + gc), rk1 = __shfl_sync(0xffffffffu, b1, 4 * k + gc);
        const double ck = __shfl_sync(0xffffffffu, (k & 1) ? b1 : b0, 4 * gr + (k >> 1));
        if (8 * kb + k < R && !(d > tol)) ok = false;
        const double dinv = rcp_nr(d);
        const double f = ck * dinv;
        const bool pr = (gr == k);
        const double n0 = pr ? rk0 * dinv : fma(-f, rk0, b0), n1 = pr ? rk1 * dinv : fma(-f, rk1, b1);
        b0 = (2 * gc == k) ? (pr ? -dinv : f) : n0;
        b1 = (2 * gc + 1 == k) ? (pr ? -dinv : f) : n1;
      }
      if (!ok && lane == 0) *s_fail = 1;
      Sw[kb * 64 + gr * 8 + 2 * gc] = b0;
      Sw[kb * 64 + gr * 8 + 2 * gc + 1] = b1;
      mbar_arrive(&bars.binv[kb]);
      if (!ok || kb + 1 == NB) break;
      const double* P = Prow + kb * 8 * LD;
      const int J = kb + 1;
      double q0, q1, d0, d1;  // Q = block row kb's column block J (rows gc, gc + 4; column gr), D = tile (J, J)
      if (kb == 0) {
        q0 = gval(gc, 8 * J + gr);
        q1 = gval(gc + 4, 8 * J + gr);
        d0 = gval(8 * J + gr, 8 * J + 2 * gc);
        d1 = gval(8 * J + gr, 8 * J + 2 * gc + 1);
      } else {
        mbar_wait(&bars.rows[kb], 0);
        q0 = P[gc * LD + 8 * J + gr];
        q1 = P[(gc + 4) * LD + 8 * J + gr];
        d0 = Dd[J * 64 + gr * 8 + 2 * gc];
        d1 = Dd[J * 64 + gr * 8 + 2 * gc + 1];
      }
      double f0 = 0.0, f1 = 0.0;
      dmma_f64(f0, f1, -Sw[kb * 64 + gr * 8 + gc], q0);
      dmma_f64(f0, f1, -Sw[kb * 64 + gr * 8 + gc + 4], q1);
      scr[gr * 8 + 2 * gc] = f0;
      scr[gr * 8 + 2 * gc + 1] = f1;
      __syncwarp();
      dmma_f64(d0, d1, -q0, scr[gc * 8 + gr]);
      dmma_f64(d0, d1, -q1, scr[(gc + 4) * 8 + gr]);
      __syncwarp();
      b0 = d0;
      b1 = d1;
    }
  } else {  // ---------------- the owners
#pragma unroll 1
    for (int kb = 0; kb < NB; ++kb) {
      double* P = Prow + kb * 8 * LD;
#pragma unroll
      for (int j = 0; j < TPW; ++j) {  // publish block row kb and the next diagonal tile
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
          Dd[(kb + 1) * 64 + gr * 8 + 2 * gc] = c0[j];
          Dd[(kb + 1) * 64 + gr * 8 + 2 * gc + 1] = c1[j];
        }
      }
      mbar_arrive(&bars.rows[kb]);
      mbar_wait(&bars.rows[kb], 0);
      mbar_wait(&bars.binv[kb], 0);
      if (*s_fail) break;
      if (w <= NB) {  // F_J = B^-1 P[:, block J], J = w - 1
        const int J = w - 1;
        double f0 = 0.0, f1 = 0.0;
        dmma_f64(f0, f1, -Sw[kb * 64 + gr * 8 + gc], P[gc * LD + 8 * J + gr]);
        dmma_f64(f0, f1, -Sw[kb * 64 + gr * 8 + gc + 4], P[(gc + 4) * LD + 8 * J + gr]);
        Fb[gr * LD + 8 * J + 2 * gc] = f0;
        Fb[gr * LD + 8 * J + 2 * gc + 1] = f1;
      }
      named_bar_sync(2, 32 * NO);
#pragma unroll
      for (int j = 0; j < TPW; ++j) {
        const int I = tI[j], J = tJ[j];
        if (I < 0) continue;
        if (I == kb && J == kb) {
          c0[j] = Sw[kb * 64 + gr * 8 + 2 * gc];
          c1[j] = Sw[kb * 64 + gr * 8 + 2 * gc + 1];
        } else if (I == kb) {
          c0[j] = Fb[gr * LD + 8 * J + 2 * gc];
          c1[j] = Fb[gr * LD + 8 * J + 2 * gc + 1];
        } else if (J == kb) {  // (F_I)^T
          c0[j] = Fb[(2 * gc) * LD + 8 * I + gr];
          c1[j] = Fb[(2 * gc + 1) * LD + 8 * I + gr];
        } else {
          dmma_f64(c0[j], c1[j], -P[gc * LD + 8 * I + gr], Fb[gc * LD + 8 * J + gr]);
          dmma_f64(c0[j], c1[j], -P[(gc + 4) * LD + 8 * I + gr], Fb[(gc + 4) * LD + 8 * J + gr]);
        }
      }
    }
  }
  __syncthreads();
  const bool failed = *s_fail != 0;
  if (tid == 0)
    for (int k = 0; k < NB; ++k) {  // the barriers are initialised again by the next call
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars.rows[k])) : "memory");
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(&bars.binv[k])) : "memory");
    }
  if (failed) return -1;
  // W = -M on the first R rows / columns (both triangles from the upper tiles)
#pragma unroll
  for (int j = 0; j < TPW; ++j) {
    const int I = tI[j], J = tJ[j];
    if (I < 0) continue;
    const int r = 8 * I + gr, c = 8 * J + 2 * gc;
    if (r < R && c < R) {
      Gm[r * RS + c] = -c0[j];
      Gm[c * RS + r] = -c0[j];
    }
    if (r < R && c + 1 < R) {
      Gm[r * RS + c + 1] = -c1[j];
      Gm[(c + 1) * RS + r] = -c1[j];
    }
  }
  __syncthreads();
  return R;
}

// row groups of the sweep inverse per RMAX: as many as 448 threads hold (32 ceil(RMAX/32) lanes per
// group, RMAX a multiple of 2 groups): fewer rows per thread shorten every pivot step
template <int RMAX>
constexpr int kPWSweepGroups = RMAX == 16 ? 8 : RMAX == 32 ? 8 : RMAX == 56 ? 7 : 4;

// RMAX: R rounded up to 16 (one instance of the sweep inverse per kernel: the whole kernel's code must
// stay instruction-cache resident across iterations -- a kernel carrying every sweep variant measured
// ~25k instructions and stalled on instruction fetch in its short phases)
template <int RMAX>
__global__ void __launch_bounds__(kPWThreads, 1) k_sweep_wide(PWParams p) {
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int N = p.N, R = p.R, RS = R + 1, G = (int)gridDim.x;
  extern __shared__ __align__(16) unsigned char pw_raw[];
  unsigned char* sm = pw_raw + ((1024u - (smem_u32(pw_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) PWBars B;
  __shared__ PWShared ss;
  __shared__ uint32_t s_tmem;
  __shared__ uint64_t s_r0;
  __shared__ int s_stop;
  __shared__ __align__(8) PWInvBars s_invb;  // dmma_sweep_inverse's barriers (initialised per call)
  __shared__ int s_invfail;
  if (wid == 13) {  // TMEM accumulator for the whole launch
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < kTCNX; ++s) {
      mbar_init(&B.xfull[s], 128);
      mbar_init(&B.xempty[s], 256);
    }
    for (int s = 0; s < kTCPairs; ++s) {
      mbar_init(&B.sdone[s], 256);
      mbar_init(&B.mdone[s], 1);
    }
    for (int s = 0; s < kTCNZ; ++s) {
      mbar_init(&B.afull[s], 1);
      mbar_init(&B.afree[s], 1);
    }
    mbar_init(&B.accf, 1);
    mbar_init(&B.bc, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_r0 = *reinterpret_cast<volatile uint64_t*>(p.iter);
    for (int k = 0; k < p.N; ++k) {  // per-mode parameters of the sampling phase, staged once per launch
      ss.dims[k] = p.dims[k];
      ss.lstride[k] = p.lstride[k];
      ss.fac[k] = p.factors[k];
      ss.cp[k] = p.cdf[k];
    }
    s_stop = 0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (p.chg) {  // cp_sgd_steps_host, optimistic: changed host factors -> nothing done, the host takes over and re-runs
    if (tid == 0) {
      int any = 0;
      for (int k = 0; k < p.N; ++k) any |= __ldcg(p.chg + k);
      s_stop = any;
      if (any && blockIdx.x == 0) atomicCAS(p.status, 0, kPWTakeOver);
    }
    __syncthreads();
    if (s_stop) {
      if (wid == 13) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
      return;
    }
  }
  unsigned gen = 0;  // barriers passed in this launch
  uint64_t r = s_r0;
  uint32_t gs = 0, gi = 0;
  PWBulk bk{&B.bc, 0u};
  unsigned qtarget = 0;  // table-unit arrivals expected before this iteration (all iterations so far)
  int pend = -1;         // mode whose table was rebuilt by the previous iteration, CDF rows not yet written
  int n_done = -1;
  const bool lev = (p.strategy == 1 || p.strategy == 3);
  const int P = R * (R + 1) / 2;

  // the coarse CDFs of every mode (the inclusive CDF at the end of each 16-row block) from the tables as the
  // launch found them (built by init or by other kernels); kept current by the table phase from here on
  if (p.strategy != 0) {
    for (int k = 0; k < N; ++k) {
      const int nb = pw_units_rows(p.dims[k]);
      for (int j = (int)blockIdx.x * kPWThreads + tid; j < nb; j += G * kPWThreads)
        p.coarse[k][j] = __ldcg(p.cdf[k] + min((int64_t)j * kPWRows + kPWRows - 1, p.dims[k] - 1));
    }
    grid_barrier(p.bar, gen);
  }
#pragma unroll 1
  for (int s = 0; s < p.nsteps; ++s) {
    const int n = p.order == 1 ? random_mode(p.seed, r, N) : (p.first_mode + s) % N;
    const int64_t In = p.dims[n];
    const int nu = pw_units_rows(In);
    const double alpha = p.alphas ? p.alphas[s] : (p.alpha_dev ? *p.alpha_dev : p.alpha);
    PW_MARK(0);
    if (p.dbg && tid == 0 && s < 8 && blockIdx.x == 0) p.dbg[512 + 32 * s + 30] = gtimer();
    long long* mk = (p.dbg && s < 8 && blockIdx.x == 0) ? p.dbg + 512 + 32 * s : nullptr;
    // ---- the table rebuilt in the previous iteration (mode pend): every unit has published its raw q rows and
    // aggregate (arrival counter, no grid barrier); a bad table stops the launch before anything is drawn ----
    if (pend >= 0) {
      if (tid == 0) {
        wait_count(p.qcnt, qtarget);
        s_stop = __ldcg(p.status) != 0 && !(p.ablate & 0x100u);
      }
      __syncthreads();
      PW_MK2(6);
      if (s_stop) break;
    }
    // ---- S: the batch of mode n at r (from the coarse CDFs; pend: from its aggregates / raw q rows) ----
    if (N == 3) pw_sample<3>(p, n, r, sm, ss, bk, mk, pend);
    else pw_sample<0>(p, n, r, sm, ss, bk, mk, pend);
    // ---- the pending table's CDF rows, T and status (read from the next sampling phase on): by the CTAs without
    // sampling units when there are any (off the sampling phase's critical path), else by every CTA ----
    if (pend >= 0) {
      const int nsamp = min(pw_units_fib(p.bmax[n]), G);
      const int c0 = nsamp < G ? nsamp : 0, nc = G - c0;
      const int nup = pw_units_rows(p.dims[pend]);
      if ((int)blockIdx.x >= c0)
        for (int u = (int)blockIdx.x - c0; u < nup; u += nc) pw_table_prefix(p, pend, u, nup, ss);
      pend = -1;
    }
    PW_MARK(1);
    grid_barrier(p.bar, gen);
    PW_MARK(2);
    // ---- G: TensorSamp + tcgen05 contraction -> split-K partial tiles; Gamma sum ----
    pw_gather(p, n, sm, B, tmem, gs, gi, mk);
    PW_MARK(3);
    grid_barrier(p.bar, gen);
    PW_MARK(4);
    // ---- U: update of the row units, table partials ----
    {
      // 16-byte aligned: Gamma [R][R], A / S rows [16][R] (cp.async targets), M rows [16][R+1]
      float* sG = reinterpret_cast<float*>(sm);
      float* sA = sG + ((R * R + 3) & ~3);
      float* sS = sA + ((kPWRows * R + 3) & ~3);
      float* sM = sS + ((kPWRows * R + 3) & ~3);
      double* sgp = reinterpret_cast<double*>(sm + ((sizeof(float) * (3 * kPWRows * RS + R * R + 12) + 15) / 16) * 16);
      // the Gamma debug hook: the last CTA (idle here whenever nu < G), off the update's critical path
      if ((int)blockIdx.x == G - 1)
        for (int e = tid; e < R * R; e += kPWThreads) p.Gam_out[e] = __ldcg(p.gam + e);
      if ((int)blockIdx.x < nu) {
        if (tid == kPWThreads - 32) {  // Gamma (every CTA reads it now): a bulk copy, waited for with the unit's rows
                                       // (issued by a thread without M-sum work: the proxy fence stalls its issuer)
          pw_bulk_begin(bk, pw_b16((int64_t)R * R * 4));
          bulk_g2s(sG, p.gam, pw_b16((int64_t)R * R * 4), bk.bar);
        }

        for (int u = blockIdx.x; u < nu; u += G) pw_update_unit(p, n, u, alpha, sA, sS, sM, sG, sgp, ss, u == (int)blockIdx.x ? &bk : nullptr,
                                                                 u == (int)blockIdx.x ? mk : nullptr);
      }
    }
    PW_MARK(5);
    grid_barrier(p.bar, gen);
    PW_MARK(6);
    if (p.strategy != 0) {
      // ---- P: the Gram's pairs (leverage) over the unit partials, a slice per CTA ----
      // one warp per pair: lane l sums the partials of units l, l + 32, ... (all loads in flight),
      // then a fixed xor-shuffle tree (deterministic); done flag per CTA, tagged by the iteration
      const uint32_t tag = p.tag0 + (uint32_t)s;
      if (lev && !(p.ablate & 4u)) {
        const int per = (P + G - 1) / G;
        const int a0 = (int)blockIdx.x * per, a1 = min(P, a0 + per);
        for (int pair = a0 + wid; pair < a1; pair += kPWThreads / 32) {
          double v[8], sacc = 0.0;
          for (int c0 = 0; c0 < nu; c0 += 8 * 32) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int u = c0 + 32 * k + lane;
              const double t = __ldcg(p.gpart + (int64_t)pair * p.gstride + (u < nu ? u : nu - 1));
              v[k] = u < nu ? t : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) sacc += v[k];
          }
          __syncwarp();
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
          if (lane == 0) p.gram[pair] = sacc;
        }
        __syncthreads();
        if (tid == 0) red_release_add(p.pcnt, 1u);
      }
      PW_MARK(7);
      // ---- I: the inverse (leverage) / ||A||_F^2 (Euclidean), every CTA with row units ----
      if ((int)blockIdx.x < nu) {
        unsigned char* ext = sm + uw_step_bytes(R, 4) + 256;
        double* Gm = reinterpret_cast<double*>(ext);
        double* rowbuf = Gm + R * RS;
        double* diag = rowbuf + kSweepBuf;
        int* swept = reinterpret_cast<int*>(diag + kMaxRank);
        // W at a 16-byte aligned OFFSET from the shared base (an integer-cast pointer would turn every
        // access into a generic load)
        const size_t offW = ((uw_step_bytes(R, 4) + 256 + sizeof(double) * ((size_t)R * RS + kSweepBuf + kMaxRank) +
                              sizeof(int) * kMaxRank + 16) + 15) / 16 * 16;
        double* Wd = reinterpret_cast<double*>(sm + offW);
        const int RD = ut_rd(R);
        double* Ad = Wd + R * RD;
        int rank = 0, bad0 = 0;
        double fro = 0.0;
        // the tensor-core block inverse (R > 32, I_n >= 2R): its tiles straight from the packed Gram
        const bool dpath = R > 32 && In >= 2 * R && !(p.ablate & 0x201u);
        if (lev) {
          if (tid == 0 && !(p.ablate & 4u)) wait_count(p.pcnt, (unsigned)G * (unsigned)(s + 1));
          __syncthreads();
          PW_MARK(18);
          {  // the packed Gram (a bulk copy: every CTA reads it now) -> the full symmetric matrix
            double* gst = Wd;  // staging
            if (tid == 0 && !(p.ablate & 4u)) {
              pw_bulk_begin(bk, pw_b16((int64_t)P * 8));
              bulk_g2s(gst, p.gram, pw_b16((int64_t)P * 8), bk.bar);
            }
            if (!(p.ablate & 4u)) pw_bulk_wait(bk);
            if (!dpath)  // the tensor-core inverse reads its tiles from the packed Gram itself
              for (int e = tid; e < R * R; e += kPWThreads) {
                const int r1 = e / R, r2 = e % R;
                const int a = r1 <= r2 ? r1 : r2, b = r1 <= r2 ? r2 : r1;
                Gm[r1 * RS + r2] = gst[a * R - a * (a - 1) / 2 + (b - a)];
              }
          }
          __syncthreads();
          if (tid < 32) {
            __syncwarp();
            double d0 = 0.0;
            bool fin = true;
            for (int j = lane; j < R; j += 32) {
              const double d = Wd[j * R - j * (j - 1) / 2];  // the packed diagonal
              d0 = fmax(d0, d);
              fin = fin && (d == d) && d < 1.7e308;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d0 = fmax(d0, __shfl_xor_sync(0xffffffffu, d0, o));
            const bool allfin = __all_sync(0xffffffffu, fin);
            if (lane == 0) {
              ss.bad = allfin ? 0 : 8;
              ss.tol = (double)(In > R ? In : R) * 2.220446049250313e-16 * d0;
            }
          }
          __syncthreads();
          constexpr int EPT = (kMaxRank * kMaxRank + kPWThreads - 1) / kPWThreads;
          PW_MARK(19);
          constexpr int SG = kPWSweepGroups<RMAX>;
          if (p.ablate & 1u) {  // timing experiment: no sweep; W = diag(1 / G_jj) (a valid table, no degenerate draws)
            for (int e = tid; e < R * R; e += kPWThreads) {
              const int r1 = e / R, r2 = e % R;
              if (r1 != r2) Gm[r1 * RS + r2] = 0.0;
            }
            for (int j = tid; j < R; j += kPWThreads) Gm[j * RS + j] = 1.0 / Gm[j * RS + j];
            __syncthreads();
            rank = R;
          } else if (In < 2 * R) {
            rank = cta_sweep_inverse_pivoted<EPT>(Gm, R, ss.tol, rowbuf, swept, diag);
          } else {
            rank = -1;
            if (dpath) {
              double* dbuf = reinterpret_cast<double*>(
                  sm + (offW + sizeof(double) * ((size_t)(R + kPWRows) * RD + 4 * (size_t)kPWRows * ((R + 3) / 4)) + 15) / 16 * 16);
              rank = dmma_sweep_inverse<RMAX>(Gm, Wd, R, ss.tol, dbuf, s_invb, &s_invfail);
              if (rank < 0) {  // a pivot failed the rule inside a block: the pivot-by-pivot sweep from the Gram again
                for (int e = tid; e < R * R; e += kPWThreads) {
                  const int r1 = e / R, r2 = e % R;
                  const int a = r1 <= r2 ? r1 : r2, b = r1 <= r2 ? r2 : r1;
                  Gm[r1 * RS + r2] = Wd[a * R - a * (a - 1) / 2 + (b - a)];
                }
                __syncthreads();
              } else {
                for (int j = tid; j < R; j += kPWThreads) swept[j] = 1;
              }
            }
            if (rank < 0) rank = grp_sweep_inverse<RMAX, SG>(Gm, R, ss.tol, rowbuf, swept);
          }
          PW_MARK(20);
          bad0 = ss.bad | (rank == 0 ? 2 : 0);
        } else {
          if (wid == 0) {  // ||A||_F^2: lane-strided unit partials, then a fixed xor tree (deterministic)
            __syncwarp();
            double t = 0.0;
            for (int u = lane; u < nu; u += 32) t += __ldcg(p.gpart + u);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            if (lane == 0) ss.tol = t;
          }
          __syncthreads();
          fro = ss.tol;
          if (!(fro == fro) || fro > 1.7e308) bad0 = 8;
          else if (!(fro > 0.0)) bad0 = 2;
        }
        PW_MARK(8);
        // ---- Q: scores, quantisation, look-back prefix -> CDF rows, T, status ----
        // the update phase left the new rows of this CTA's last unit in shared memory (sA, stride R; the
        // pair sums and the inverse use the area past uw_step_bytes only)
        const float* sAlast = reinterpret_cast<const float*>(sm) + ((R * R + 3) & ~3);
        for (int u = blockIdx.x; u < nu; u += G)
          pw_table_unit(p, n, u, nu, tag, Gm, rank, fro, bad0, Ad, u + G >= nu ? sAlast : nullptr, ss,
                        u == (int)blockIdx.x ? mk : nullptr);
        // this CTA's units published: one release (no wait: the next sampling phase waits for all of them)
        if (tid == 0) red_release_add(p.qcnt, (unsigned)((nu - 1 - (int)blockIdx.x) / G + 1));
      }
      PW_MARK(9);
      qtarget += (unsigned)nu;
      pend = n;  // the table of the new A^(n) is complete once every unit has arrived (R9)
    }
    PW_MARK(10);
    if (p.dbg && tid == 0 && s < 8 && blockIdx.x == 0) p.dbg[512 + 32 * s + 31] = gtimer();
    ++r;
    n_done = n;
    if (p.tr.base) {  // debug trace: complete the table first, then record the iteration
      if (pend >= 0) {
        if (tid == 0) wait_count(p.qcnt, qtarget);
        __syncthreads();
        for (int u = blockIdx.x; u < pw_units_rows(p.dims[pend]); u += G) pw_table_prefix(p, pend, u, pw_units_rows(p.dims[pend]), ss);
        pend = -1;
      }
      grid_barrier(p.bar, gen);
      pw_trace(p, s, n, r - 1);
      if (s + 1 < p.nsteps) grid_barrier(p.bar, gen);  // before the next batch overwrites idx / w
    }
    if (p.strategy == 0) {  // uniform (no table): the barrier after the update orders it before the next batch
      if (tid == 0) s_stop = __ldcg(p.status) != 0 && !(p.ablate & 0x100u);
      __syncthreads();
      if (s_stop) break;
    }
  }
  // the last iteration's table (or the one the stop found bad): its CDF rows, T and status
  if (pend >= 0) {
    if (tid == 0) wait_count(p.qcnt, qtarget);
    __syncthreads();
    for (int u = blockIdx.x; u < pw_units_rows(p.dims[pend]); u += G) pw_table_prefix(p, pend, u, pw_units_rows(p.dims[pend]), ss);
  }
  __syncthreads();
  if (wid == 13) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  if (blockIdx.x == 0 && tid == 0) {
    *p.iter = r;
    if (n_done >= 0) *p.last_mode = n_done;
  }
}

}  // namespace cps
