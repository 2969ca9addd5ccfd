// gupdate_tc.cuh -- k_gather_update_tc: the fp32 wide-path step kernel with the sampled MTTKRP
// M_tile = X_F diag(w) Z_F (eq:gradient1/2) on the 5th-generation tensor cores.
//
//   D[i][r] (TMEM, fp32) = sum_b X[i][b] ZW[b][r]     i: 128 rows of the I-tile (UMMA M = 128)
//                                                      r: NB = 32*ceil(R/32) columns (UMMA N)
//                                                      b: fibers, K = 8 per tcgen05.mma (kind::tf32)
//   3xTF32 (SURVEY section 7 hard part 3): x = xh + xl, zw = zh + zl with xh = trunc_tf32(x) and
//   xl = x - xh (exact in fp32), D += xh zh + xh zl + xl zh  -> ~fp32 accuracy (dropped xl zl ~ 2^-22).
//
// Operands in shared memory, canonical UMMA layout "K-major, 128-byte swizzle": an atom is 8 MN-rows
// x 128 B (the 32 fibers of a stage), 16-byte chunk c of row rr stored at chunk (c ^ rr); 8-row
// groups at SBO = 1024 B; UMMA K-step k (8 fibers = 32 B) starts 32k bytes into the atom.  The X
// tile arrives by cp.async in plain [fiber][row] order (a fiber segment is 512 contiguous bytes of
// the mode-major copy: the HBM stream of Alg. 5 TensorSamp); one pass transposes 4x4 blocks in
// registers and writes xh and xl in the K-major layout.  B (zh, zl) is produced by the sampler
// directly as layout images and copied linearly.  (MN-major tf32 operands read as zeros on this
// toolchain/driver -- tools/micro/umma.cu -- so both operands are K-major.)
//
// Warp-specialised pipeline (stages of KS = 32 fibers; 448 threads):
//   warps 0-3   X loaders: 16-byte cp.async chunks of the sampled fiber segments (512 contiguous bytes
//               of the mode-major copy each) into an NX-deep raw ring; completion on xfull[s] via
//               cp.async.mbarrier.arrive.noinc; slots recycled through xempty[s];
//   warp 13     B producer (one thread): the hi / lo B images of the stage (2 bulk copies, 2-deep ring);
//   warps 4-11  split: 4x4 register transposes -> xh / xl (K-major) in pair s & 1 (free once stage
//               s-2's MMAs retired: mdone), fence.proxy.async, arrive sdone;
//   warp 12     MMA issuer (one thread): 12 tcgen05.mma per stage, tcgen05.commit -> mdone[s & 1];
//               last commit -> accf.
//   epilogue    warps 4-7 read the accumulator (tcgen05.ld.32x32b: warp w <-> TMEM lanes 32(w%4)..),
//               then all threads write the partial tile (gu_finish).
#pragma once
#include <cooperative_groups.h>

#include "gupdate.cuh"

namespace cps {

constexpr int kTCThreads = 448;
constexpr int kTCKS = 32;      // fibers per stage (4 UMMA K-steps)

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

// ring sizes (bytes): NX stages of raw X, 2 stages of B (hi, lo), 2 pairs of K-major (xh, xl)
template <int NB8>
__host__ __device__ constexpr uint32_t tc_b_bytes() { return (uint32_t)kTCKS * 8 * NB8 * 4; }
constexpr uint32_t kTCABytes = kTCKS * 128 * 4;
template <int NB8>
__host__ __device__ constexpr int tc_nx() {  // deepest X ring that fits next to the other buffers
  return (int)((200u * 1024u - 4u * kTCABytes - 4u * tc_b_bytes<NB8>()) / kTCABytes);
}
template <int NB8>
__host__ __device__ inline size_t tc_smem_bytes(int R, int64_t KB) {
  const size_t ring = (size_t)tc_nx<NB8>() * kTCABytes + 4 * (size_t)tc_b_bytes<NB8>() + 4 * (size_t)kTCABytes;
  const size_t epi = (size_t)kGUTI * (8 * NB8 + 1) * 4;
  return 1024 + (ring > epi ? ring : epi) + (size_t)R * R * 4 + (size_t)KB * 8 + 256;
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int NB8>
__global__ void __launch_bounds__(448, 1) k_gather_update_tc(GUParams<float> p) {
  constexpr int NB = 8 * NB8;                                   // UMMA N (columns r >= R are zero)
  constexpr int TMEM_COLS = NB <= 32 ? 32 : 64;
  constexpr int KS = kTCKS, NX = tc_nx<NB8>(), TI = kGUTI;
  constexpr uint32_t A_BYTES = kTCABytes, B_BYTES = tc_b_bytes<NB8>();
  constexpr uint32_t IDESC = umma_idesc_tf32_mn(128, NB) & ~((1u << 15) | (1u << 16));  // K-major A and B
  extern __shared__ __align__(16) unsigned char tc_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(tc_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* xsp = sm;                          // 2 x {xh, xl} (K-major, 128-byte swizzle)
  unsigned char* bring = sm + 4 * A_BYTES;          // 2 x {B hi, B lo}
  unsigned char* xring = bring + 4 * B_BYTES;       // NX x raw X [32 fibers][512 B]
  const size_t body = (size_t)4 * A_BYTES + 4 * B_BYTES + (size_t)NX * A_BYTES;
  const size_t epi = (size_t)TI * (NB + 1) * 4;
  float* sGam = reinterpret_cast<float*>(sm + (body > epi ? body : epi));
  int64_t* sfb = reinterpret_cast<int64_t*>(sGam + p.R * p.R + (p.R * p.R & 1));
  __shared__ __align__(8) uint64_t xfull[16], xempty[16], bfull[2], sdone[2], mdone[2], accf;
  __shared__ uint32_t s_tmem;

  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int R = p.R;
  const int64_t i0 = (int64_t)blockIdx.x * TI;
  const int64_t c0 = (int64_t)blockIdx.y * p.KB;
  const int nfib = (int)cmax64(0, cmin64(p.KB, p.bmax - c0));
  const int nst = (nfib + KS - 1) / KS;
  const bool mark = p.dbg && blockIdx.x == 0 && blockIdx.y == 0 && tid == 128;
  if (mark) p.dbg[32] = clock64();
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  long long gt0 = 0;
  if (p.dbg && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));

  if (wid == 12) {  // TMEM accumulator: 128 lanes x TMEM_COLS columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"((uint32_t)TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int s = 0; s < NX; ++s) {
      mbar_init(&xfull[s], 128);   // the 128 loader threads' cp.async.mbarrier.arrive.noinc
      mbar_init(&xempty[s], 256);  // the 256 split threads are done reading the raw stage
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&sdone[s], 256);
      mbar_init(&mdone[s], 1);  // tcgen05.commit: MMAs of the stage retired (xh/xl pair + B slot free)
    }
    mbar_init(&accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cp_async_u64(reinterpret_cast<uint64_t*>(sfb), reinterpret_cast<const uint64_t*>(p.fbase + c0), nfib, tid, 448);
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
  } else if (wid == 13) {
    // ======================= B producer (one thread): hi / lo images, 2-deep ring =======================
    if (lane == 0) {
      for (int st = 0; st < nst; ++st) {
        const int slot = st & 1;
        if (st >= 2) mbar_wait(&mdone[slot], (uint32_t)(((st >> 1) - 1) & 1));
        unsigned char* Bh = bring + slot * 2 * B_BYTES;
        const int64_t sb = (c0 + (int64_t)st * KS) / KS;  // stage index in the images ([stage][NB rows][128 B])
        mbar_expect_tx(&bfull[slot], 2 * B_BYTES);
        bulk_g2s(Bh, p.zhi + sb * (B_BYTES / 4), B_BYTES, &bfull[slot]);
        bulk_g2s(Bh + B_BYTES, p.zlo + sb * (B_BYTES / 4), B_BYTES, &bfull[slot]);
      }
    }
  } else if (wid >= 4 && wid <= 11) {
    // ======================= 3xTF32 split / transpose (256 threads) =======================
    // block = 4 fibers (4kq..) x 4 rows {iq, iq+32, iq+64, iq+96}: lanes run over iq, so the raw
    // loads (4 B, consecutive rows) and the K-major stores (row & 7 = iq & 7) are conflict-free
    const int t = tid - 128;
    const int iq = t & 31, kq = t >> 5;  // warp -> fiber quad kq (0..7)
    for (int st = 0; st < nst; ++st) {
      const int slot = st % NX, hb = st & 1;
      mbar_wait(&xfull[slot], (uint32_t)((st / NX) & 1));
      if (mark && st == 8) p.dbg[18] = clock64();
      if (st >= 2) mbar_wait(&mdone[hb], (uint32_t)(((st >> 1) - 1) & 1));  // xh/xl pair hb free
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
        for (int a = 0; a < 4; ++a) x[u][a] = ok ? A[kk * 128 + iq + 32 * a] : 0.f;
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
  } else if (wid == 12 && lane == 0) {
    // ======================= MMA issuer =======================
    const bool mk = p.dbg && blockIdx.x == 0 && blockIdx.y == 0;
    const uint64_t dx = umma_desc_sw128(smem_u32(xsp), 16, 1024);    // xh of pair 0
    const uint64_t dbz = umma_desc_sw128(smem_u32(bring), 16, 1024);  // B hi of slot 0
    for (int st = 0; st < nst; ++st) {
      const int hb = st & 1;
      mbar_wait(&sdone[hb], (uint32_t)((st >> 1) & 1));
      mbar_wait(&bfull[hb], (uint32_t)((st >> 1) & 1));
      tc_fence_after();
      if (mk && st == 8) p.dbg[21] = clock64();
      const uint64_t h = dx + ((uint64_t)(hb * 2 * A_BYTES) >> 4);
      const uint64_t l = h + (A_BYTES >> 4);
      const uint64_t bh = dbz + ((uint64_t)(hb * 2 * B_BYTES) >> 4), bl = bh + (B_BYTES >> 4);
#pragma unroll
      for (int k = 0; k < KS / 8; ++k) {  // K-step k: fibers 8k..8k+7 = bytes 32k.. of every atom row
        umma_tf32(tmem, h + 2 * k, bh + 2 * k, IDESC, (st > 0 || k > 0) ? 1u : 0u);
        umma_tf32(tmem, h + 2 * k, bl + 2 * k, IDESC, 1u);
        umma_tf32(tmem, l + 2 * k, bh + 2 * k, IDESC, 1u);
      }
      umma_commit(&mdone[hb]);
      if (mk && st == 8) p.dbg[22] = clock64();
    }
    umma_commit(&accf);
  }
  __syncthreads();
  if (mark) p.dbg[34] = clock64();
  // ---- accumulator -> shared partial tile [TI][NB+1] (zero if this CTA had no fibers) ----
  if (nst > 0) mbar_wait(&accf, 0u);
  tc_fence_after();
  constexpr int MS = NB + 1;
  float* Mt = reinterpret_cast<float*>(sm);  // every ring is dead
  if (wid >= 4 && wid <= 7) {
    const int lg = wid & 3;          // TMEM lane group of this warp
    const int row = 32 * lg + lane;  // TMEM lane = tile row
#pragma unroll
    for (int cb = 0; cb < NB; cb += 8) {
      uint32_t r[8];
      if (nst > 0) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(tmem + ((uint32_t)(32 * lg) << 16) + (uint32_t)cb));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = 0u;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) Mt[row * MS + cb + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 12) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)TMEM_COLS));
  if (mark) p.dbg[35] = clock64();
  if (p.dbg && tid == 0 && cta < 1000) {
    long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    p.dbg[1024 + 2 * cta] = gt0;
    p.dbg[1025 + 2 * cta] = gt1;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.dbg[3072 + cta] = smid;
  }
  gu_finish<float>(p, Mt, MS, i0, tid, 448);
  if (mark) p.dbg[36] = clock64();
}

}  // namespace cps
