// micro-test of tcgen05.mma kind::tf32 with the A operand in TMEM (".ts" form): each thread of a
// warp quadrant writes its row m of A (K = 32 tf32 values) with tcgen05.st.32x32b, B is K-major
// SW128 in shared memory.  D[128 x NB] = X[128 x K] * Z[K x NB], compared to CPU.  Also times
// 96 back-to-back MMAs (M=128, N=56, K=8) in SS and TS form.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2103_04081_b200/csrc/gupdate_tc.cuh"
using namespace cps;

__device__ __forceinline__ void umma_tf32_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int NB>
__global__ void k(const float* X /* [K][128] */, const float* Z /* [K][NB] */, float* D, int reps,
                  long long* cyc) {
  constexpr int K = 32;
  extern __shared__ __align__(16) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  unsigned char* A = sm;             // K-major SW128 copy of A (for the SS timing)
  unsigned char* B = sm + 128 * 128;  // NB rows x 128 B
  __shared__ uint32_t s_tmem;
  __shared__ uint64_t bar;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  for (int e = tid; e < K * 128; e += blockDim.x) {
    const int kk = e / 128, m = e % 128;
    *reinterpret_cast<float*>(A + kmaj_off(m, kk)) = X[kk * 128 + m];
  }
  for (int e = tid; e < K * NB; e += blockDim.x) {
    const int kk = e / NB, n = e % NB;
    *reinterpret_cast<float*>(B + kmaj_off(n, kk)) = Z[kk * NB + n];
  }
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t acol = 448;  // A at TMEM columns [448, 480)
  {
    const int m = 32 * wid + lane;
    uint32_t v[32];
    for (int kk = 0; kk < K; ++kk) v[kk] = __float_as_uint(X[kk * 128 + m]);
    const uint32_t ta = tmem + ((uint32_t)(32 * wid) << 16) + acol;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t IDESC = umma_idesc_tf32_mn(128, NB) & ~((1u << 15) | (1u << 16));
  const uint64_t db0 = umma_desc_sw128(smem_u32(B), 16, 1024);
  const uint64_t da0 = umma_desc_sw128(smem_u32(A), 16, 1024);
  uint32_t ph = 0;
  if (tid == 0) {
    for (int k = 0; k < K / 8; ++k) umma_tf32_ts(tmem, tmem + acol + 8 * k, db0 + 2 * k, IDESC, k > 0 ? 1u : 0u);
    umma_commit(&bar);
  }
  mbar_wait(&bar, ph); ph ^= 1;
  tc_fence_after();
  const int row = 32 * wid + lane;
  for (int cb = 0; cb < NB && cb < 64; cb += 8) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(32 * wid) << 16) + (uint32_t)cb, v);
    for (int j = 0; j < 8 && cb + j < NB; ++j) D[row * NB + cb + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // timing: reps x 4 MMAs, SS then TS, into nacc rotating accumulators (columns 0, 64, 128 / N=112: 0, 112 wraps)
  for (int mode = 0; mode < 6; ++mode) {
    const int nacc = (mode >> 1) + 1;
    if (tid == 0) {
      const long long t0 = clock64();
      int q = 0;
      for (int r = 0; r < reps; ++r)
        for (int k = 0; k < K / 8; ++k) {
          const uint32_t d = tmem + (NB <= 64 ? 64u * q : 0u);
          if (++q == nacc) q = 0;
          if ((mode & 1) == 0) umma_tf32(d, da0 + 2 * k, db0 + 2 * k, IDESC, 1u);
          else umma_tf32_ts(d, tmem + acol + 8 * k, db0 + 2 * k, IDESC, 1u);
        }
      umma_commit(&bar);
      const long long t1 = clock64();
      cyc[2 * mode] = t1 - t0;
      mbar_wait(&bar, ph);
      cyc[2 * mode + 1] = clock64() - t0;
    }
    __syncthreads();
    ph ^= 1;
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

template <int NB>
void run() {
  const int K = 32;
  std::vector<float> X(K * 128), Z(K * NB), D(128 * NB);
  unsigned s = 7;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (int)((s >> 16) % 7) - 3; };
  for (auto& x : X) x = (float)rnd();
  for (auto& z : Z) z = (float)rnd();
  float *dX, *dZ, *dD; long long* dc; long long hc[12];
  cudaMalloc(&dX, 4 * X.size()); cudaMalloc(&dZ, 4 * Z.size()); cudaMalloc(&dD, 4 * D.size()); cudaMalloc(&dc, 128);
  cudaMemcpy(dX, X.data(), 4 * X.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dZ, Z.data(), 4 * Z.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xff, 4 * D.size());
  const size_t smem = 1024 + 128 * 128 + 256 * 128;
  cudaFuncSetAttribute(k<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 24;
  k<NB><<<1, 128, smem>>>(dX, dZ, dD, reps, dc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, 4 * D.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(hc, dc, 96, cudaMemcpyDeviceToHost);
  int bad = 0; double maxerr = 0;
  for (int i = 0; i < 128; ++i)
    for (int r = 0; r < NB && r < 64; ++r) {
      double ref = 0;
      for (int kk = 0; kk < K; ++kk) ref += (double)X[kk * 128 + i] * Z[kk * NB + r];
      const double err = fabs(ref - D[i * NB + r]);
      maxerr = fmax(maxerr, err);
      if (err > 1e-3 && bad++ < 4) printf("  D[%d][%d] = %g ref %g\n", i, r, D[i * NB + r], ref);
    }
  printf("TS NB=%d: %s, bad %d / %d, max err %g | %d MMAs (done cyc):", NB, cudaGetErrorString(e), bad, 128 * NB, maxerr, reps * 4);
  for (int m = 0; m < 6; ++m) printf(" %s nacc=%d %lld", m & 1 ? "TS" : "SS", (m >> 1) + 1, hc[2 * m + 1]);
  printf("\n");
}
int main() {
  run<56>(); run<128>(); run<192>(); run<256>();
  return 0;
}
