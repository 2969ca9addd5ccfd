// micro-test of the tcgen05 kind::tf32 MN-major SW128 path used by k_gather_update_tc:
// D[128 x NB] = X[128 x K] * Z[K x NB] with operands staged in the canonical layout; compares to CPU.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/gupdate_tc.cuh"
using namespace cps;
template <int ATOMS_MN>
__device__ __forceinline__ uint32_t sw128_off(int kk, int m) {
  const int rr = kk & 7, c = (m >> 2) & 7;
  return (uint32_t)((kk >> 3) * ATOMS_MN * 1024 + (m >> 5) * 1024 + rr * 128 + ((c ^ rr) << 4) + ((m & 3) << 2));
}
template <int NMB>
__global__ void k(const float* X /* [K][128] */, const float* Z /* [K][NB] */, int K, float* D, int mode,
                  unsigned long long* dbg) {
  constexpr int NB = 32 * NMB;
  extern __shared__ __align__(16) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  unsigned char* A = sm;                       // K/8 groups x 4 atoms x 1KB
  unsigned char* B = sm + K * 128 * 4;         // K/8 groups x NMB atoms x 1KB
  __shared__ uint32_t s_tmem;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  auto mnone = [](int m, int kk, int sbo, int lbo) {  // MN-major no-swizzle: core = 8 K-rows x 16 B (4 MN)
    return (uint32_t)((m >> 2) * sbo + (kk >> 3) * lbo + (kk & 7) * 16 + (m & 3) * 4);
  };
  auto kmaj = [](int m, int kk) {  // K-major SW128, K = 32 (one atom along K): (m/8)*1024 + (m%8)*128 + chunk^row
    const int rr = m & 7, c = (kk >> 2) & 7;
    return (uint32_t)((m >> 3) * 1024 + rr * 128 + ((c ^ rr) << 4) + ((kk & 3) << 2));
  };
  for (int e = tid; e < K * 128; e += blockDim.x) {
    const int kk = e / 128, m = e % 128;
    *reinterpret_cast<float*>(A + ((mode & 32) ? mnone(m, kk, 128, 4096) : (mode & 8) ? kmaj(m, kk) : sw128_off<4>(kk, m))) = X[kk * 128 + m];
  }
  for (int e = tid; e < K * NB; e += blockDim.x) {
    const int kk = e / NB, m = e % NB;
    *reinterpret_cast<float*>(B + ((mode & 32) ? mnone(m, kk, 128, NB * 32) : (mode & 8) ? kmaj(m, kk) : sw128_off<NMB>(kk, m))) = Z[kk * NB + m];
  }
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"((uint32_t)NB));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (mode & 2) {  // pre-fill the accumulator with 1.0 through tcgen05.st (32x32b.x16)
    uint32_t one = __float_as_uint(1.0f);
    for (int cb = 0; cb < NB; cb += 16)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" :: "r"(tmem + ((uint32_t)(32 * wid) << 16) + (uint32_t)cb), "r"(one));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  if (tid == 0) {
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    const uint32_t IDESC = (mode & 8) ? (umma_idesc_tf32_mn(128, NB) & ~((1u << 15) | (1u << 16))) : umma_idesc_tf32_mn(128, NB);
    dbg[0] = umma_desc_sw128(a, 1024, 1024);
    dbg[1] = IDESC;
    dbg[2] = tmem;
    for (int k = 0; k < K / 8; ++k) {
      uint64_t da = umma_desc_sw128(a + k * 4096, mode & 1 ? 4096 : 1024, mode & 1 ? 1024 : 4096);
      uint64_t db = umma_desc_sw128(b + k * NMB * 1024, mode & 1 ? NMB * 1024 : 1024, mode & 1 ? 1024 : NMB * 1024);
      if (mode & 8) {  // K-major: advance 32 bytes per K-step inside the atom; SBO = 1024 (8-row groups)
        da = umma_desc_sw128(a + k * 32, 16, 1024);
        db = umma_desc_sw128(b + k * 32, 16, 1024);
      }
      if (mode & 32) {  // MN-major, no swizzle: core matrices along MN at 128 B, K-groups at (MN/4)*128 B
        const uint32_t sA = 128, lA = 4096, sB = 128, lB = NB * 32;
        auto nd = [](uint32_t addr, uint32_t lbo, uint32_t sbo) {
          return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
                 ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
        };
        da = (mode & 1) ? nd(a + k * lA, sA, lA) : nd(a + k * lA, lA, sA);
        db = (mode & 1) ? nd(b + k * lB, sB, lB) : nd(b + k * lB, lB, sB);
      }
      if (mode & 16) {  // MN-major with layout type 1 (128B swizzle, 32B atomicity)
        da = (da & ~((uint64_t)7 << 61)) | ((uint64_t)1 << 61);
        db = (db & ~((uint64_t)7 << 61)) | ((uint64_t)1 << 61);
      }
      umma_tf32(tmem, da, db, IDESC, (k > 0 || (mode & 2)) ? 1u : 0u);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  if (mode & 4) { for (int i = 0; i < 100; ++i) __nanosleep(1000); }
  tc_fence_after();
  const int row = 32 * wid + lane;
  for (int cb = 0; cb < NB; cb += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * wid) << 16) + (uint32_t)cb, v);
    for (int j = 0; j < 16; ++j) D[row * NB + cb + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)NB));
}
template <int NMB>
void run(int mode) {
  constexpr int NB = 32 * NMB;
  const int K = 32;
  std::vector<float> X(K * 128), Z(K * NB), D(128 * NB);
  unsigned s = 7;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int)((s >> 16) % 7) - 3; };  // small ints: exact in tf32
  for (auto& x : X) x = (float)rnd();
  for (auto& z : Z) z = (float)rnd();
  float *dX, *dZ, *dD; unsigned long long* dd; unsigned long long hd[3];
  cudaMalloc(&dX, 4 * X.size()); cudaMalloc(&dZ, 4 * Z.size()); cudaMalloc(&dD, 4 * D.size()); cudaMalloc(&dd, 64);
  cudaMemcpy(dX, X.data(), 4 * X.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dZ, Z.data(), 4 * Z.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, 4 * D.size());
  const size_t smem = 1024 + K * 128 * 4 + K * NB * 4;
  cudaFuncSetAttribute(k<NMB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<NMB><<<1, 128, smem>>>(dX, dZ, K, dD, mode, dd);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(hd, dd, 24, cudaMemcpyDeviceToHost);
  int bad = 0; double maxerr = 0;
  for (int i = 0; i < 128; ++i)
    for (int r = 0; r < NB; ++r) {
      double ref = 0;
      for (int kk = 0; kk < K; ++kk) ref += (double)X[kk * 128 + i] * Z[kk * NB + r];
      const double err = fabs(ref - D[i * NB + r]);
      maxerr = fmax(maxerr, err);
      if (err > 1e-3 && bad++ < 4) printf("  D[%d][%d] = %g ref %g\n", i, r, D[i * NB + r], ref);
    }
  printf("NMB=%d mode=%d: %s, bad %d / %d, max err %g, desc %llx idesc %llx tmem %llx\n", NMB, mode, cudaGetErrorString(e), bad,
         128 * NB, maxerr, hd[0], hd[1], hd[2]);
}
int main() {
  run<1>(32); run<1>(33); run<2>(32); run<2>(33);
  return 0;
}
