// gupdate_tc.cuh -- k_gather_update_tc: the fp32 wide-path step kernel with the sampled MTTKRP
// M_tile = X_F diag(w) Z_F (eq:gradient1/2) on the 5th-generation tensor cores.
//
//   3xTF32 (SURVEY section 7 hard part 3): x = xh + xl, zw = zh + zl with h = trunc_tf32(.) and
//   l = . - h (exact in fp32).  ONE tcgen05.mma (kind::tf32, M = 128, N = 256, K = 8) per 8 fibers
//   computes all four products at once:
//
//      A (SMEM, 128 rows x K)   = [ zh_0..zh_63 ; zl_0..zl_63 ]          (rows r >= R are zero)
//      B (SMEM, 256 rows x K)   = [ xh_i (i = 0..127) ; xl_i (i = 0..127) ]
//      D (TMEM, 128 x 256 fp32) = A B^T,  M^T[r][i] = D[r][i] + D[r][128+i] + D[64+r][i] + D[64+r][128+i]
//
//   (zl xl is kept: the result is the full fp32 product up to accumulation rounding.)  A tcgen05.mma
//   costs ~100 cycles whatever its N below ~128 on this part (N = 256: ~170, tools/micro/umma_ts.cu),
//   so four products in one N = 256 instruction replace the twelve N = 56 ones of a 3-MMA split.
//
// Both operands in shared memory, canonical UMMA layout "K-major, 128-byte swizzle": an atom is 8 rows
// x 128 B (the 32 fibers of a stage), 16-byte chunk c of row rr stored at chunk (c ^ rr); 8-row
// groups at SBO = 1024 B (xl's 128 rows follow xh's directly); UMMA K-step k starts 32k bytes into
// the atom.  The X tile arrives by cp.async in plain [fiber][row] order (a fiber segment is 512
// contiguous bytes of the mode-major copy: the HBM stream of Alg. 5 TensorSamp); one pass transposes
// 4x4 blocks in registers and writes xh and xl.  (MN-major tf32 operands read as zeros on this
// toolchain/driver -- tools/micro/umma.cu -- so B is K-major.)  A is produced by the sampler directly
// in this layout (one 16 KB image per stage, zimg_off in kernels.cuh) and copied linearly.
//
// Warp-specialised pipeline (stages of KS = 32 fibers; 448 threads):
//   warps 0-3   X loaders: 16-byte cp.async chunks of the sampled fiber segments into an NX-deep raw
//               ring; completion on xfull[s] via cp.async.mbarrier.arrive.noinc; recycled via xempty[s];
//   warps 4-11  split: 4x4 register transposes -> {xh, xl} pair s % NP (free once stage s-NP's MMAs
//               retired: mdone), fence.proxy.async, arrive sdone;
//   warp 12     A producer (one thread): the stage's image, one 16 KB cp.async.bulk into slot s % NZ
//               (completion: afull[s] transaction bytes; slot freed by tcgen05.commit -> afree);
//   warp 13     MMA issuer (one thread): 4 tcgen05.mma per stage, commits -> mdone, afree; last -> accf.
//   epilogue    warps 4-11 fold the xh / xl halves (tcgen05.ld.32x32b) into shared memory, then all
//               threads fold the zh / zl halves and write the partial tile to the split-K workspace.
#pragma once
#include <cooperative_groups.h>

#include "gupdate.cuh"

namespace cps {

constexpr int kTCThreads = 448;
constexpr int kTCKS = 32;      // fibers per stage (4 UMMA K-steps)


__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 64-bit UMMA shared-memory descriptor: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48) (sm_100), base offset 0, layout 2 = 128-byte swizzle [61,64)
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor, kind::tf32: D f32 [4,6)=1, A tf32 [7,10)=2, B tf32 [10,13)=2, A and B
// MN-major [15], [16], N >> 3 [17,23), M >> 4 [24,29)
__host__ __device__ constexpr uint32_t umma_idesc_tf32_mn(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// byte offset of (MN row m, fiber kk of a 32-fiber stage) in a K-major 128-byte-swizzle operand
__host__ __device__ __forceinline__ uint32_t kmaj_off(int m, int kk) {
  const int rr = m & 7, c = (kk >> 2) & 7;
  return (uint32_t)((m >> 3) * 1024 + rr * 128 + ((c ^ rr) << 4) + ((kk & 3) << 2));
}

// shared-memory rings (bytes): NX stages of raw X, NPAIR pairs {xh, xl} of the K-major UMMA B operand
constexpr uint32_t kTCABytes = kTCKS * 128 * 4;  // one stage of raw X / one K-major half (16 KB)
constexpr int kTCPairs = 2;
constexpr int kTCNZ = 3;                          // A-operand (zw hi / lo image) stages
constexpr uint32_t kTCZBytes = 128 * kTCKS * 4;   // one image stage: 128 rows x 128 B (16 KB)
constexpr int kTCNX = (int)((200u * 1024u - kTCPairs * 2u * kTCABytes - kTCNZ * kTCZBytes) / kTCABytes);
constexpr int kTCEpiStride = kGUTI + 4;  // epilogue staging row pitch (floats): conflict-free float4 rows
__host__ __device__ inline size_t tc_smem_bytes(int64_t KB) {
  const size_t ring = (size_t)kTCNX * kTCABytes + (size_t)kTCPairs * 2 * kTCABytes + (size_t)kTCNZ * kTCZBytes;
  const size_t epi = (size_t)128 * kTCEpiStride * 4;
  return 1024 + (ring > epi ? ring : epi) + (size_t)KB * 8 + 256;
}

__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// a template (one instance, V = 0) so that only the translation unit that launches it emits it
template <int V = 0>
__global__ void __launch_bounds__(kTCThreads, 1) k_gather_update_tc(GUParams<float> p) {
  constexpr int KS = kTCKS, NX = kTCNX, NP = kTCPairs, NZ = kTCNZ, TI = kGUTI;
  constexpr uint32_t A_BYTES = kTCABytes;
  constexpr uint32_t TMEM_COLS = 256;    // D: 128 lanes x 256 fp32 columns
  // M = 128 (A rows: zh 0-63, zl 64-127), N = 256 (B rows: xh 0-127, xl 128-255), both K-major
  constexpr uint32_t IDESC = umma_idesc_tf32_mn(128, 256) & ~((1u << 15) | (1u << 16));
  extern __shared__ __align__(16) unsigned char tc_raw[];
  // 1024-byte aligned base, derived from the shared array itself so every access stays LDS / STS
  // (integer round-tripping the pointer turns them into generic LD / ST)
  unsigned char* sm = tc_raw + ((1024u - (smem_u32(tc_raw) & 1023u)) & 1023u);
  unsigned char* xsp = sm;                          // NP x {xh, xl} (K-major, 128-byte swizzle, contiguous)
  unsigned char* xring = sm + NP * 2 * A_BYTES;     // NX x raw X [32 fibers][512 B]
  unsigned char* zring = xring + NX * A_BYTES;      // NZ x A image [128 rows][128 B] (K-major, swizzled)
  const size_t body = (size_t)NP * 2 * A_BYTES + (size_t)NX * A_BYTES + (size_t)NZ * kTCZBytes;
  const size_t epi = (size_t)128 * kTCEpiStride * 4;
  int64_t* sfb = reinterpret_cast<int64_t*>(sm + (body > epi ? body : epi));
  __shared__ __align__(8) uint64_t xfull[16], xempty[16], sdone[4], mdone[4], afull[4], afree[4], accf;
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int R = p.R;
  const int64_t i0 = (int64_t)blockIdx.x * TI;
  const int64_t c0 = (int64_t)gu_chunk(p) * p.KB;
  const int nfib = (int)cmax64(0, cmin64(p.KB, p.bmax - c0));
  const int nst = (nfib + KS - 1) / KS;
  const bool mark = p.dbg && blockIdx.x == 0 && blockIdx.y == 0 && tid == 128;
  if (mark) p.dbg[32] = clock64();
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  long long gt0 = 0;
  if (p.dbg && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));

  if (wid == 13) {  // TMEM accumulator
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < NX; ++s) {
      mbar_init(&xfull[s], 128);   // the 128 loader threads' cp.async.mbarrier.arrive.noinc
      mbar_init(&xempty[s], 256);  // the 256 split threads are done reading the raw stage
    }
    for (int s = 0; s < NP; ++s) {
      mbar_init(&sdone[s], 256);
      mbar_init(&mdone[s], 1);  // tcgen05.commit: MMAs of the stage retired (xh/xl pair free)
    }
    for (int s = 0; s < NZ; ++s) {
      mbar_init(&afull[s], 1);  // expect_tx arrival + the bulk copy's bytes
      mbar_init(&afree[s], 1);  // tcgen05.commit: the A slot may be overwritten
    }
    mbar_init(&accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();  // the batch (fiber offsets, A images) comes from the previous kernel
  cp_async_u64(reinterpret_cast<uint64_t*>(sfb), reinterpret_cast<const uint64_t*>(p.fbase + c0), nfib, tid,
               kTCThreads);
  cp_async_commit();
  cp_async_wait<0>();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (mark) p.dbg[33] = clock64();

  if (wid < 4) {
    // ======================= X loaders (128 threads): 16-byte cp.async chunks =======================
    // (one TMA bulk copy per 512-byte segment sustains only ~0.3 TB/s on this part; per-thread
    // cp.async ~2 TB/s -- tools/micro/gather2.cu)
    const int lt = tid;  // 0..127
    for (int st = 0; st < nst; ++st) {
      const int slot = st % NX;
      if (st >= NX) mbar_wait(&xempty[slot], (uint32_t)(((st / NX) - 1) & 1));
      if (p.dbg && blockIdx.x == 0 && blockIdx.y == 0 && st == 8 && lt == 0) p.dbg[23] = clock64();
      unsigned char* A = xring + slot * A_BYTES;
      const int f0 = st * KS;
#pragma unroll
      for (int rep = 0; rep < KS * 32 / 128; ++rep) {
        const int e = lt + 128 * rep;
        const int kk = e >> 5, j = e & 31;
        const int lb = f0 + kk;
        const int64_t fb = lb < nfib ? sfb[lb] : -1;
        const int64_t r0 = i0 + 4 * j;
        if (fb >= 0 && r0 < p.rowlen) cp_async16(A + kk * 512 + 16 * j, p.X + fb + r0, 16);
      }
      cp_async_mbar_arrive_noinc(&xfull[slot]);
    }
  } else if (wid <= 11) {
    // ======================= 3xTF32 split / transpose (256 threads) =======================
    // block = 4 fibers (4kq..) x 4 rows {iq, iq+32, iq+64, iq+96}: lanes run over iq, so the raw
    // loads (4 B, consecutive rows) and the K-major stores (row & 7 = iq & 7) are conflict-free
    const int t = tid - 128;
    const int iq = t & 31, kq = t >> 5;  // warp -> fiber quad kq (0..7)
    for (int st = 0; st < nst; ++st) {
      const int slot = st % NX, hb = st % NP;
      if (mark && st == 8) p.dbg[26] = clock64();
      if (mark && st == 9) p.dbg[27] = clock64();
      if (mark && st == 12) p.dbg[28] = clock64();
      mbar_wait(&xfull[slot], (uint32_t)((st / NX) & 1));
      if (mark && st == 8) p.dbg[18] = clock64();
      if (st >= NP) mbar_wait(&mdone[hb], (uint32_t)(((st / NP) - 1) & 1));  // xh/xl pair hb free
      if (mark && st == 8) p.dbg[19] = clock64();
      const float* A = reinterpret_cast<const float*>(xring + slot * A_BYTES);
      unsigned char* H = xsp + hb * 2 * A_BYTES;
      unsigned char* L = H + A_BYTES;
      const int f0 = st * KS;
      float x[4][4];  // x[fiber u][row a]
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = 4 * kq + u, lb = f0 + kk;
        const bool ok = lb < nfib && sfb[lb] >= 0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {  // load unconditionally (inside the ring), then select: a
          const float t = A[kk * 128 + iq + 32 * a];  // conditional load compiles to a branch per load
          x[u][a] = ok ? t : 0.f;
        }
      }
      mbar_arrive(&xempty[slot]);  // raw stage consumed (values are in registers)
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const float4 h = make_float4(tf32_trunc(x[0][a]), tf32_trunc(x[1][a]), tf32_trunc(x[2][a]), tf32_trunc(x[3][a]));
        const float4 l = make_float4(x[0][a] - h.x, x[1][a] - h.y, x[2][a] - h.z, x[3][a] - h.w);
        const uint32_t o = kmaj_off(iq + 32 * a, 4 * kq);
        *reinterpret_cast<float4*>(H + o) = h;
        *reinterpret_cast<float4*>(L + o) = l;
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
      mbar_arrive(&sdone[hb]);
      if (mark && st == 8) p.dbg[20] = clock64();
    }
  } else if (wid == 12) {
    // ======================= A producer (one thread): the sampler's zh / zl image of the stage =======================
    // (lanes 1-31: Gamma as the cluster-ordered sum of the sampler's partials, spread over the grid)
    if (lane != 0) {
      const int cta_lin = blockIdx.y * gridDim.x + blockIdx.x;
      gu_gamma_sum<float>(p, cta_lin * 31 + lane - 1, gridDim.x * gridDim.y * 31);
    } else {
      for (int st = 0; st < nst; ++st) {
        const int zs = st % NZ;
        if (st >= NZ) mbar_wait(&afree[zs], (uint32_t)(((st / NZ) - 1) & 1));
        const int64_t sb = (c0 + (int64_t)st * KS) / KS;  // stage index in the images
        mbar_expect_tx(&afull[zs], kTCZBytes);
        bulk_g2s(zring + zs * kTCZBytes, p.zimg + sb * (kTCZBytes / 4), kTCZBytes, &afull[zs]);
      }
    }
  } else if (wid == 13 && lane == 0) {
    // ======================= MMA issuer =======================
    const bool mk = p.dbg && blockIdx.x == 0 && blockIdx.y == 0;
    const uint64_t dx = umma_desc_sw128(smem_u32(xsp), 16, 1024);   // B = {xh; xl} of pair 0
    const uint64_t dz = umma_desc_sw128(smem_u32(zring), 16, 1024);  // A = {zh; zl} of slot 0
    for (int st = 0; st < nst; ++st) {
      const int hb = st % NP, as = st % NZ;
      if (mk && st == 8) p.dbg[24] = clock64();
      mbar_wait(&sdone[hb], (uint32_t)((st / NP) & 1));
      if (mk && st == 8) p.dbg[25] = clock64();
      mbar_wait(&afull[as], (uint32_t)((st / NZ) & 1));
      tc_fence_after();
      if (mk && st == 8) p.dbg[21] = clock64();
      const uint64_t b = dx + ((uint64_t)(hb * 2 * A_BYTES) >> 4);
      const uint64_t a = dz + ((uint64_t)(as * kTCZBytes) >> 4);
#pragma unroll
      for (int k = 0; k < KS / 8; ++k)  // K-step k: fibers 8k..8k+7 = bytes 32k.. of every atom row
        umma_tf32(tmem, a + 2 * k, b + 2 * k, IDESC, (st > 0 || k > 0) ? 1u : 0u);
      umma_commit(&mdone[hb]);
      umma_commit(&afree[as]);
      if (mk && st == 8) p.dbg[22] = clock64();
    }
    umma_commit(&accf);
  }
  __syncthreads();
  pdl_trigger();  // mainloop done: the next kernel may start its launch
  if (mark) p.dbg[34] = clock64();
  // ---- epilogue: E[L][i] = D[L][i] + D[L][128 + i] (x = xh + xl) staged in shared memory, then
  //      M^T[r][i] = E[r][i] + E[64 + r][i] (zw = zh + zl) -> the split-K workspace ----
  if (nst > 0) mbar_wait(&accf, 0u);
  tc_fence_after();
  float* E = reinterpret_cast<float*>(sm);  // every ring is dead
  if (wid >= 4 && wid <= 11) {  // warp w: TMEM lanes 32 (w & 3).., tile rows [64 hh, 64 hh + 64)
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
  if (wid == 13) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  if (mark) p.dbg[35] = clock64();
  {
    const int nrow = (int)cmax64(0, cmin64(TI, p.In - i0));
    float* part = p.Mpart + ((int64_t)blockIdx.x * p.CK + gu_chunk(p)) * R * TI;
    for (int e = tid; e < R * (TI / 4); e += kTCThreads) {
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
    // r <- r + 1 (Alg. 6/7); nothing in this launch reads r (Gamma_out: k_update_wide)
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *p.iter += 1;
  }
  if (p.dbg && tid == 0 && cta < 1000) {
    long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    p.dbg[1024 + 2 * cta] = gt0;
    p.dbg[1025 + 2 * cta] = gt1;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.dbg[3072 + cta] = smid;
  }
  if (mark) p.dbg[36] = clock64();
}

}  // namespace cps
