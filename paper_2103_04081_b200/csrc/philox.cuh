// philox.cuh -- counter-based Philox4x32-10 of the sampling contract (DESIGN.md "Sampling
// contract"): counter (x0, purpose<<24 | slot, r_lo, r_hi), key (seed_lo, seed_hi),
// 64-bit word u = y1 << 32 | y0.  Host and device (the host copy draws the random mode order).
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define CPS_HD __host__ __device__ __forceinline__
#else
#define CPS_HD inline
#endif

namespace cps {

enum : uint32_t { kPurposeRow = 0u, kPurposeWindow = 1u, kPurposeMode = 2u };

CPS_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

struct U4 {
  uint32_t x, y, z, w;
};

CPS_HD U4 philox10(U4 c, uint32_t k0, uint32_t k1) {
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int i = 0; i < 10; ++i) {
    const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

CPS_HD uint64_t draw_word(uint64_t seed, uint64_t iter, uint32_t x0, uint32_t purpose, uint32_t slot) {
  U4 y = philox10(U4{x0, (purpose << 24) | slot, (uint32_t)iter, (uint32_t)(iter >> 32)}, (uint32_t)seed,
                  (uint32_t)(seed >> 32));
  return ((uint64_t)y.y << 32) | (uint64_t)y.x;
}

// floor(u * T / 2^64)
CPS_HD uint64_t scale_draw(uint64_t u, uint64_t T) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(u, T);
#else
  return (uint64_t)(((unsigned __int128)u * T) >> 64);
#endif
}

CPS_HD int random_mode(uint64_t seed, uint64_t iter, int N) {
  U4 y = philox10(U4{0u, kPurposeMode << 24, (uint32_t)iter, (uint32_t)(iter >> 32)}, (uint32_t)seed,
                  (uint32_t)(seed >> 32));
  return (int)(((uint64_t)y.x * (uint64_t)N) >> 32);
}

}  // namespace cps
