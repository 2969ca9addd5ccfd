// Which load path sustains random 512-byte fiber-segment gathers on B200?  1 CTA per SM (148 CTAs),
// each CTA streams `nseg` random 512 B segments (8 KB rows of a 32 GB buffer) through:
//   mode 0: LDG.128 into registers (U segments in flight per warp), no shared memory
//   mode 1: cp.async 16 B into a shared ring of NS stages x 32 segments
//   mode 2: cp.async.bulk (TMA 1D, 512 B per op) into the same ring, mbarrier completion
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33; return x;
}
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int SEG = 512, KS = 32;
template <int MODE, int NS>
__global__ void __launch_bounds__(256, 1) k(const float* __restrict__ X, uint64_t nrows, int nseg, uint64_t seed, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  float acc = 0.f;
  auto rowof = [&](int s) { return mix(seed ^ (blockIdx.x * 1000003ULL + s)) % nrows; };
  if (MODE == 0) {
    // warp w handles segments s = w, w+8, ...; 8 in flight per warp (lane: 16 B each)
    for (int s0 = wid; s0 < nseg; s0 += 8 * 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int s = s0 + 8 * u;
        v[u] = s < nseg ? __ldg(reinterpret_cast<const float4*>(X + rowof(s) * 2048 + 128 * (s & 15)) + lane) : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].w;
    }
  } else {
    const int nst = nseg / KS;
    if (tid == 0) { for (int i = 0; i < NS; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[i]))); }
    __syncthreads();
    auto issue = [&](int st) {
      unsigned char* dst = sm + (st % NS) * KS * SEG;
      if (MODE == 1) {
        for (int e = tid; e < KS * 32; e += 256) {
          const int kk = e >> 5, j = e & 31;
          const float* src = X + rowof(st * KS + kk) * 2048 + 128 * ((st * KS + kk) & 15) + 4 * j;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(su32(dst + kk * SEG + 16 * j)), "l"(src));
        }
        asm volatile("cp.async.commit_group;");
      } else if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar[st % NS])), "r"(KS * SEG));
        for (int kk = 0; kk < KS; ++kk) {
          const float* src = X + rowof(st * KS + kk) * 2048 + 128 * ((st * KS + kk) & 15);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(su32(dst + kk * SEG)), "l"(src), "r"(SEG), "r"(su32(&bar[st % NS])));
        }
      }
    };
    for (int s = 0; s < NS - 1 && s < nst; ++s) issue(s);
    for (int st = 0; st < nst; ++st) {
      if (MODE == 1) {
        asm volatile("cp.async.wait_group %0;" :: "n"(NS - 2));
      } else {
        uint32_t ok = 0;
        do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(su32(&bar[st % NS])), "r"((uint32_t)((st / NS) & 1))); } while (!ok);
      }
      __syncthreads();
      const float* buf = reinterpret_cast<const float*>(sm + (st % NS) * KS * SEG);
      for (int e = tid; e < KS * 128; e += 256) acc += buf[e];
      __syncthreads();
      if (st + NS - 1 < nst) issue(st + NS - 1);
      else if (MODE == 1) asm volatile("cp.async.commit_group;");
    }
  }
  if (acc == 12345.f) out[0] = acc;
}
template <int MODE, int NS>
void run(const float* X, uint64_t nrows, float* out, const char* name) {
  const int nseg = 32 * 64;  // 64 stages of 32 segments = 1 MB per CTA
  const size_t smem = MODE ? (size_t)NS * KS * SEG : 0;
  cudaFuncSetAttribute(k<MODE, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<MODE, NS><<<148, 256, smem>>>(X, nrows, nseg, 1, out);
  cudaEventRecord(a);
  for (int r = 0; r < 3; ++r) k<MODE, NS><<<148, 256, smem>>>(X, nrows, nseg, 5 + r, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-34s %7.1f GB/s  (%s)\n", name, 3.0 * 148 * nseg * SEG / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const size_t S = (size_t)32 << 30;
  float* X; float* out;
  cudaMalloc(&X, S); cudaMemset(X, 0, S); cudaMalloc(&out, 64);
  const uint64_t nrows = S / 8192;
  run<0, 1>(X, nrows, out, "LDG.128, 8 segs/warp in flight");
  run<1, 4>(X, nrows, out, "cp.async 16B, 4 x 16KB stages");
  run<1, 8>(X, nrows, out, "cp.async 16B, 8 x 16KB stages");
  run<1, 12>(X, nrows, out, "cp.async 16B, 12 x 16KB stages");
  run<2, 4>(X, nrows, out, "TMA bulk 512B, 4 x 16KB stages");
  run<2, 8>(X, nrows, out, "TMA bulk 512B, 8 x 16KB stages");
  run<2, 12>(X, nrows, out, "TMA bulk 512B, 12 x 16KB stages");
  return 0;
}
