// sweep_wide_params.cuh -- the host-visible part of k_sweep_wide (sweep_wide.cuh): the launch parameters,
// the unit counts and the shared-memory plan.  The host code includes only this; the kernel body lives
// in sweep_wide.cuh, compiled in k_pw.cu.
#pragma once
#include "gupdate_tc.cuh"
#include "wide.cuh"

namespace cps {

constexpr int kPWThreads = kTCThreads;  // 448: the tcgen05 gather's warp roles
constexpr int kPWFib = 32;              // fibers per sampling unit (one tcgen05 stage)
constexpr int kPWRows = 16;             // rows per update / table unit
constexpr int kPWUpdKG = 8;             // k groups of the update's G = A Gamma - M (short chains vs. partial traffic)

struct PWParams {
  int N, R, strategy, rule;
  int nsteps, first_mode, order;
  int64_t B;
  int64_t dims[kMaxOrder], lstride[kMaxOrder];
  const float* Xg[kMaxOrder];      // gather base of mode n: mode-major copy (n >= 1) or X (mode 0)
  int64_t rowlen[kMaxOrder];       // readable elements per fiber row (pitch, or I_0)
  int64_t pitch[kMaxOrder];        // 0: native (mode 0)
  float* factors[kMaxOrder];
  float* S[kMaxOrder];
  uint64_t* cdf[kMaxOrder];
  double* pprob[kMaxOrder];
  uint64_t* Ttot;
  int32_t window[kMaxOrder][kMaxOrder];
  int64_t bmax[kMaxOrder];
  int CK[kMaxOrder];
  int64_t KB[kMaxOrder];
  uint64_t seed;
  uint64_t* iter;
  int* status;
  int* last_mode;
  double alpha, eta, b, eps;
  const double* alpha_dev;         // constant step on the device (graph-free replays), or NULL
  const double* alphas;            // per-iteration steps (fixed rule), or NULL
  // workspace
  int32_t* idx;
  double* w;
  int64_t* fbase;
  int64_t* beff;
  float* zimg;
  float* gcl;                      // [G][R][R] per-CTA partials of Gamma
  float* gam;                      // [R][R]
  float* Mpart;                    // [tiles][CK][R][128]
  double* gpart;                   // [row units][P] (leverage) or [row units] (Euclidean)
  double* gram;                    // [P] the Gram's pairs
  double* rownorm;                 // [I_max]
  unsigned long long* agg;         // [row units] q sums
  unsigned* aggf;                  // [row units][2]: {bad bits, tag}
  unsigned* bar;                   // grid-barrier arrivals (zero at launch)
  unsigned* pcnt;                  // pair-sum arrivals (zero at launch)
  unsigned* qcnt;                  // table-unit arrivals (zero at launch)
  uint64_t* qraw;                  // [I_max padded to 16]: raw q rows of the table being rebuilt
  uint64_t* coarse[kMaxOrder];     // per mode [units]: the inclusive CDF at the end of each 16-row block
  int64_t gstride;                 // gpart: [P][gstride] (leverage pair partials, unit fastest)
  uint32_t tag0;                   // tag of iteration 0 of this launch (unique per handle)
  float* Gout;
  float* Gam_out;
  TraceParams tr;
  const int* chg;                  // cp_sgd_steps_host: per-mode "staged host factor differs" flags, or NULL; any set
                                   // -> the launch does nothing but report kPWTakeOver (the host takes over, re-runs)
  long long* dbg;
  // timing experiments only (CPSGD_PW_ABLATE_MASK; results are garbage): 1 skip the sweep inverse (W = diag(1 / G_jj)), 2 skip the
  // fiber loads of the gather, 4 skip the pair sums and the Gram load, 8 skip the update's Gram partials,
  // 16 skip the scores, 0x100 never stop on a bad status, 0x200 the CUDA-core forms of the R > 32 tensor-core
  // phases (scores, Gram partials, Gamma partials, G, inverse: timing comparison)
  unsigned ablate;
};

constexpr int kPWTakeOver = -99;  // device status: the optimistic cp_sgd_steps_host launch found changed host factors

__host__ __device__ inline int pw_units_rows(int64_t In) { return (int)((In + kPWRows - 1) / kPWRows); }
__host__ __device__ inline int pw_units_fib(int64_t bmax) { return (int)((bmax + kPWFib - 1) / kPWFib); }

// dynamic shared memory: the gather's ring (tc_smem_bytes) covers every other phase's working set
__host__ __device__ inline size_t pw_other_bytes(int N, int R, int64_t cdf_elems) {
  const int RP = zg_rp(R);
  const size_t sample = 16 * 8 + sizeof(uint64_t) * (cdf_elems + kMaxOrder) + sizeof(int32_t) * kPWFib * (N - 1) +
                        sizeof(double) * kPWFib * (N - 1) + sizeof(double) * kPWFib + sizeof(float) * kPWFib * RP +
                        sizeof(float) * (size_t)zg_groups(R, kPWThreads) * R * R + sizeof(float) * R * R;
  const size_t scratch_g = sizeof(float) * 8 * kPWRows * (size_t)R;
  const size_t scratch_p = sizeof(double) * ((size_t)kPWRows * ut_rd(R) + 4 * (size_t)(R * (R + 1) / 2));
  const size_t upd = uw_step_bytes(R, 4) + 16 * 8 + (scratch_g > scratch_p ? scratch_g : scratch_p) + 64;
  // the inverse / table phases (k_sweep_wide's layout): Gm, the sweep buffer, diag and swept past the update's step
  // area; W and the unit rows from offW; then the tensor-core inverse's buffers (dmma_sweep_inverse: block rows,
  // diagonal tiles, -B^-1, F, scratch; RMAX of k_pw.cu)
  const int rmax = R <= 16 ? 16 : R <= 32 ? 32 : R <= 56 ? 56 : 64;
  const size_t dinv = sizeof(double) * ((size_t)(rmax / 8) * 8 * (rmax + 2) + 2 * (size_t)(rmax / 8) * 64 + 8 * (size_t)(rmax + 2) + 64);
  const size_t offW = (uw_step_bytes(R, 4) + 256 + sizeof(double) * ((size_t)R * (R + 1) + kSweepBuf + kMaxRank) +
                       sizeof(int) * kMaxRank + 16 + 15) / 16 * 16;
  const size_t inv = (offW + sizeof(double) * ((size_t)(R + kPWRows) * ut_rd(R) + 4 * (size_t)kPWRows * ((R + 3) / 4)) + 15) / 16 * 16 +
                     (R > 32 ? dinv : 0) + 64;
  if (upd > inv) return sample > upd ? sample : upd;
  size_t m = sample > inv ? sample : inv;
  return m;
}
__host__ __device__ inline size_t pw_smem_bytes(int N, int R, int64_t KBmax, int64_t cdf_elems) {
  const size_t g = tc_smem_bytes(KBmax);
  const size_t o = pw_other_bytes(N, R, cdf_elems) + 1024;
  return g > o ? g : o;
}

}  // namespace cps
