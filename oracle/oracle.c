/*
 * oracle/oracle.c -- the CPU ORACLE for the importance-sampled mini-batch SGD step of
 * arXiv 2103.04081 (BrawsCPD / AdawsCPD).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2103_04081_b200/) never imports, links or executes anything under oracle/,
 * and this file shares no code, header, table or constant generator with it.
 *
 * Style: plain, slow, obviously correct.  Single thread, IEEE fp64 throughout, compiled
 * with -O2 -ffp-contract=off (no FMA contraction), no BLAS, no SIMD intrinsics.  Every
 * function follows the paper's definition or algorithm in the paper's order; citations
 * are "PAPER.md:<lines> (<label>)".  Where the paper is silent or garbled the reading
 * taken is the one listed in DESIGN.md "Readings" (R-numbers below refer to it).
 *
 * Indices are 0-based (the paper is 1-based; reading R16).  Storage of the dense tensor
 * is first-index-fastest (PAPER.md:47-50 eq:map; reading R17).  Factor matrices are
 * row-major I_n x R.
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions without a pin say so in their
 * comment ("parity unpinned"); at present every exported function has at least one pin.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ERANGE (-2)
#define ORC_EDEGENERATE (-3)
#define ORC_ENOMEM (-4)

/* sampling strategies (PAPER.md:494-504 naming; uniform = Alg. 2 BrasCPD) */
#define ORC_UNIFORM 0
#define ORC_LEVERAGE 1
#define ORC_EUCLIDEAN 2
#define ORC_BLOCK_LEVERAGE 3
#define ORC_BLOCK_EUCLIDEAN 4

#define ORC_STEP_FIXED 0    /* eq:proposed (4.3) */
#define ORC_STEP_ADAPTIVE 1 /* eq:etaada/eq:Aada (4.4) */
#define ORC_STEP_ALS 2      /* sampled least squares: A = M Gamma^+ (eq:lsq_krp) */

#define ORC_ORDER_CYCLIC 0
#define ORC_ORDER_RANDOM 1 /* "uniformly sample n" */

/* ------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11), the counter-based generator of the sampling
 * contract (reading R21).  Round function and key schedule
 * as published: 10 rounds, key bumped between rounds.
 * ---------------------------------------------------------------------------------- */
static uint32_t orc_mulhi32(uint32_t a, uint32_t b) { return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32); }

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0 = orc_mulhi32(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = orc_mulhi32(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* One 64-bit uniform word of the contract: counter (x0, purpose<<24 | slot, r_lo, r_hi),
 * key (seed_lo, seed_hi); u = y1 << 32 | y0. */
static uint64_t orc_word(uint64_t seed, uint64_t iter, uint32_t x0, uint32_t purpose, uint32_t slot) {
  uint32_t ctr[4] = {x0, (purpose << 24) | slot, (uint32_t)iter, (uint32_t)(iter >> 32)};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t y[4];
  orc_philox4x32_10(ctr, key, y);
  return ((uint64_t)y[1] << 32) | (uint64_t)y[0];
}

/* floor(u * T / 2^64), exact */
static uint64_t orc_scale(uint64_t u, uint64_t T) { return (uint64_t)(((unsigned __int128)u * (unsigned __int128)T) >> 64); }

/* ------------------------------------------------------------------------------------
 * Index map, PAPER.md:47-50 (eq:map, Eq. 1.2), 0-based:
 *   j = sum_{k != n} i_k J'_k,  J'_k = prod_{m < k, m != n} I_m.
 * tuple[] holds the N-1 indices of the modes k != n in ascending k (eq:idx).
 * ---------------------------------------------------------------------------------- */
int64_t orc_linear_index(int N, const int64_t* dims, int n, const int32_t* tuple) {
  int64_t j = 0;
  int pos = 0;
  for (int k = 0; k < N; ++k) {
    if (k == n) continue;
    int64_t Jp = 1;
    for (int m = 0; m < k; ++m)
      if (m != n) Jp *= dims[m];
    if (tuple[pos] < 0 || tuple[pos] >= dims[k]) return -1;
    j += (int64_t)tuple[pos] * Jp;
    ++pos;
  }
  return j;
}

/* element (i, j) of the mode-n unfolding X_(n): decode j into the tuple by
 * the inverse of eq:map (mixed radix, first remaining mode fastest), then read the tensor
 * at the first-index-fastest offset sum_k i_k S_k, S_k = prod_{m<k} I_m. */
/* The dense tensor is read through this one accessor: fp64 storage, or fp32 storage (xf32 != 0) whose
 * element is converted to fp64 exactly on read -- the fp32 entry points (orc_run_f32) let the
 * baseline run on a 32 GB fp32 tensor without an fp64 copy; the arithmetic is unchanged. */
static double orc_x(const void* X, int xf32, int64_t off) {
  return xf32 ? (double)((const float*)X)[off] : ((const double*)X)[off];
}

static double orc_unfold_elem(int N, const int64_t* dims, const void* X, int xf32, int n, int64_t i, int64_t j) {
  int64_t off = 0, stride = 1, rem = j;
  for (int k = 0; k < N; ++k) {
    int64_t ik;
    if (k == n) {
      ik = i;
    } else {
      ik = rem % dims[k];
      rem /= dims[k];
    }
    off += ik * stride;
    stride *= dims[k];
  }
  return orc_x(X, xf32, off);
}

/* Alg. 5 TensorSamp: j_b from eq:map, then X_(n)(:, j_b).
 * out is I_n x B, column b contiguous (out[b*I_n + i]). */
static int orc_tensor_samp_x(int N, const int64_t* dims, const void* X, int xf32, int n, int64_t B,
                             const int32_t* idx, double* out) {
  for (int64_t b = 0; b < B; ++b) {
    int64_t j = orc_linear_index(N, dims, n, idx + b * (N - 1));
    if (j < 0) return ORC_ERANGE;
    for (int64_t i = 0; i < dims[n]; ++i) out[b * dims[n] + i] = orc_unfold_elem(N, dims, X, xf32, n, i, j);
  }
  return ORC_OK;
}
int orc_tensor_samp(int N, const int64_t* dims, const double* X, int n, int64_t B, const int32_t* idx, double* out) {
  return orc_tensor_samp_x(N, dims, X, 0, n, B, idx, out);
}

/* Alg. 1 SKR: Z <- 1; for m != n: Z <- Z (*) A^(m)(idx(:,m), :).
 * Z is B x R row-major. */
int orc_skr(int N, const int64_t* dims, int R, const double* const* factors, int n, int64_t B, const int32_t* idx,
            double* Z) {
  for (int64_t b = 0; b < B; ++b)
    for (int r = 0; r < R; ++r) Z[b * R + r] = 1.0;
  int pos = 0;
  for (int m = 0; m < N; ++m) {
    if (m == n) continue;
    for (int64_t b = 0; b < B; ++b) {
      int32_t i = idx[b * (N - 1) + pos];
      if (i < 0 || i >= dims[m]) return ORC_ERANGE;
      for (int r = 0; r < R; ++r) Z[b * R + r] = Z[b * R + r] * factors[m][(int64_t)i * R + r];
    }
    ++pos;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * Leverage scores, Def. 2.3: l_i = ||Q(i,:)||^2 with Q an orthonormal
 * basis of range(A).  Q from a Householder QR with column pivoting (Golub & Van Loan
 * Alg. 5.4.1); numerical rank = #{j : |R_jj| > max(m,R) * eps * |R_00|} (reading R4).
 * A is m x R row-major, not modified.  ell has m entries.
 * ---------------------------------------------------------------------------------- */
int orc_leverage_scores(int64_t m, int R, const double* A, double* ell, int* rank_out) {
  double* W = (double*)malloc(sizeof(double) * (size_t)(m * R)); /* working copy, becomes R + Householder vectors */
  double* V = (double*)malloc(sizeof(double) * (size_t)(m * R)); /* Householder vectors, column k in V[:,k] */
  double* beta = (double*)malloc(sizeof(double) * (size_t)R);
  double* colnorm = (double*)malloc(sizeof(double) * (size_t)R);
  double* Q = (double*)malloc(sizeof(double) * (size_t)(m * R));
  if (!W || !V || !beta || !colnorm || !Q) {
    free(W); free(V); free(beta); free(colnorm); free(Q);
    return ORC_ENOMEM;
  }
  memcpy(W, A, sizeof(double) * (size_t)(m * R));
  memset(V, 0, sizeof(double) * (size_t)(m * R));
  int kmax = (int)(m < R ? m : R);
  double r00 = 0.0;
  int rank = 0;
  for (int k = 0; k < kmax; ++k) {
    /* pivot: remaining column with the largest norm over rows k..m-1 (recomputed, no downdating) */
    int piv = k;
    double best = -1.0;
    for (int c = k; c < R; ++c) {
      double s = 0.0;
      for (int64_t i = k; i < m; ++i) s += W[i * R + c] * W[i * R + c];
      colnorm[c] = s;
      if (s > best) { best = s; piv = c; }
    }
    if (piv != k)
      for (int64_t i = 0; i < m; ++i) {
        double t = W[i * R + k]; W[i * R + k] = W[i * R + piv]; W[i * R + piv] = t;
      }
    /* Householder vector v for column k, rows k..m-1: x - alpha e_1, alpha = -sign(x0)||x|| */
    double norm = sqrt(best);
    if (k == 0) r00 = norm;
    double tol = (double)(m > R ? m : R) * 2.220446049250313e-16 * r00;
    if (!(norm > tol) || norm == 0.0) break;
    double x0 = W[k * R + k];
    double alpha = (x0 >= 0.0) ? -norm : norm;
    for (int64_t i = k; i < m; ++i) V[i * R + k] = W[i * R + k];
    V[k * R + k] = x0 - alpha;
    double vtv = 0.0;
    for (int64_t i = k; i < m; ++i) vtv += V[i * R + k] * V[i * R + k];
    beta[k] = (vtv > 0.0) ? 2.0 / vtv : 0.0;
    /* apply H_k = I - beta v v^T to columns k..R-1 of W */
    for (int c = k; c < R; ++c) {
      double s = 0.0;
      for (int64_t i = k; i < m; ++i) s += V[i * R + k] * W[i * R + c];
      s *= beta[k];
      for (int64_t i = k; i < m; ++i) W[i * R + c] -= s * V[i * R + k];
    }
    ++rank;
  }
  /* explicit Q(:, 0:rank) = H_0 H_1 ... H_{rank-1} [e_0 .. e_{rank-1}] */
  memset(Q, 0, sizeof(double) * (size_t)(m * R));
  for (int c = 0; c < rank; ++c) Q[(int64_t)c * R + c] = 1.0;
  for (int k = rank - 1; k >= 0; --k) {
    for (int c = 0; c < rank; ++c) {
      double s = 0.0;
      for (int64_t i = k; i < m; ++i) s += V[i * R + k] * Q[i * R + c];
      s *= beta[k];
      for (int64_t i = k; i < m; ++i) Q[i * R + c] -= s * V[i * R + k];
    }
  }
  for (int64_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int c = 0; c < rank; ++c) s += Q[i * R + c] * Q[i * R + c];
    ell[i] = s;
  }
  if (rank_out) *rank_out = rank;
  free(W); free(V); free(beta); free(colnorm); free(Q);
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * Per-mode row probabilities p (PAPER.md:271 p_k = l(A^(k))/R; Def. 2.4 :191-193; Def. 2.5
 * :197-199; block variants use the same per-row masses, Defs. 3.1-3.2 :344-390).
 *   uniform   : 1/I
 *   leverage  : l_i / rank               (reading R4: rank = R for full-rank factors)
 *   euclidean : ||A(i,:)||^2 / ||A||_F^2 (Def. 2.5 with beta = 1)
 * ---------------------------------------------------------------------------------- */
int orc_row_probs(int strategy, int64_t I, int R, const double* A, double* p, int* rank_out) {
  if (I < 1 || R < 1) return ORC_EINVAL;
  if (rank_out) *rank_out = R;
  if (strategy == ORC_UNIFORM) {
    for (int64_t i = 0; i < I; ++i) p[i] = 1.0 / (double)I;
    return ORC_OK;
  }
  if (strategy == ORC_LEVERAGE || strategy == ORC_BLOCK_LEVERAGE) {
    int rank = 0;
    int st = orc_leverage_scores(I, R, A, p, &rank);
    if (st) return st;
    if (rank_out) *rank_out = rank;
    if (rank == 0) return ORC_EDEGENERATE;
    for (int64_t i = 0; i < I; ++i) p[i] = p[i] / (double)rank;
    return ORC_OK;
  }
  if (strategy == ORC_EUCLIDEAN || strategy == ORC_BLOCK_EUCLIDEAN) {
    double fro = 0.0;
    for (int64_t i = 0; i < I; ++i)
      for (int r = 0; r < R; ++r) fro += A[i * R + r] * A[i * R + r];
    if (!(fro > 0.0)) return ORC_EDEGENERATE;
    for (int64_t i = 0; i < I; ++i) {
      double s = 0.0;
      for (int r = 0; r < R; ++r) s += A[i * R + r] * A[i * R + r];
      p[i] = s / fro;
    }
    return ORC_OK;
  }
  return ORC_EINVAL;
}

/* Fixed-point realisation of p (sampling contract step 3): q_i = p_i > 0 ? max(1, rint(p_i 2^32)) : 0,
 * uniform q_i = 1; T = sum q.  The sampler draws from q/T, and the weights use q/T (the
 * realised law), which keeps Theorem 5.1 exact. */
int orc_quantize(int strategy, int64_t I, const double* p, uint64_t* q, uint64_t* T_out) {
  uint64_t T = 0;
  for (int64_t i = 0; i < I; ++i) {
    if (strategy == ORC_UNIFORM) {
      q[i] = 1;
    } else if (!(p[i] == p[i]) || p[i] > 2.0) {
      return ORC_EDEGENERATE; /* non-finite or nonsense probability */
    } else if (p[i] > 0.0) {
      double s = rint(p[i] * 4294967296.0);
      q[i] = (s < 1.0) ? 1u : (uint64_t)s;
    } else {
      q[i] = 0;
    }
    T += q[i];
  }
  if (T == 0) return ORC_EDEGENERATE;
  *T_out = T;
  return ORC_OK;
}

/* table = probs + quantisation; p may be NULL */
int orc_build_table(int strategy, int64_t I, int R, const double* A, double* p_out, uint64_t* q, uint64_t* T) {
  double* p = p_out ? p_out : (double*)malloc(sizeof(double) * (size_t)I);
  if (!p) return ORC_ENOMEM;
  int st = orc_row_probs(strategy, I, R, A, p, NULL);
  if (!st) st = orc_quantize(strategy, I, p, q, T);
  if (!p_out) free(p);
  return st;
}

/* #{i : cdf[i] <= r} with cdf the inclusive prefix sums of q (plain linear scan) */
static int64_t orc_count_le(const uint64_t* q, int64_t I, uint64_t r) {
  uint64_t cdf = 0;
  int64_t cnt = 0;
  for (int64_t i = 0; i < I; ++i) {
    cdf += q[i];
    if (cdf <= r) ++cnt;
  }
  return cnt;
}

/* Default block windows (reading R6): for position p of the N-1 remaining modes, b_p is the
 * smallest divisor d of the remaining batch with d^(N-1-p) >= remaining batch; then clamp
 * to I_k. */
int orc_default_windows(int N, const int64_t* dims, int n, int64_t B, int32_t* window) {
  int64_t rem = B;
  int pos = 0;
  for (int k = 0; k < N; ++k) {
    if (k == n) continue;
    int left = N - 1 - pos;
    int64_t d = 1;
    for (d = 1; d <= rem; ++d) {
      if (rem % d) continue;
      double pw = 1.0;
      for (int t = 0; t < left; ++t) pw *= (double)d;
      if (pw >= (double)rem) break;
    }
    if (d > rem) d = rem;
    rem /= d;
    window[pos] = (int32_t)(d < dims[k] ? d : dims[k]);
    ++pos;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * KrpSamp1 / KrpSamp2 index draws (Alg. 3, Alg. 4 :412-428; eq:ik :272-277,
 * eq:bik :364-370) with the realised probabilities (eq:block_lev_prob :279-285,
 * eq:block_norm_prob :299-306 read as products, R3; eq:block_lev_prob2 / eq:block_norm_prob2
 * :372-408 read as Cartesian products of windows, R2/R6).
 *   q[k], T[k] : tables of every mode (mode n ignored)
 *   idx        : out, B_max x (N-1) int32 (B_max = B, or prod(window) for block)
 *   w          : out, per-row weight omega_b (contract step 7)
 *   pj         : out, per-row probability of the drawn row of Z (row-wise), or the batch
 *                probability p_S repeated (block)
 * ---------------------------------------------------------------------------------- */
int orc_sample(int N, const int64_t* dims, int n, int strategy, int64_t B, const int32_t* window_in,
               const uint64_t* const* q, const uint64_t* T, uint64_t seed, uint64_t iter, int32_t* idx, double* w,
               double* pj, int64_t* B_eff_out) {
  if (N < 3 || n < 0 || n >= N || B < 1) return ORC_EINVAL;
  if (strategy == ORC_UNIFORM || strategy == ORC_LEVERAGE || strategy == ORC_EUCLIDEAN) {
    for (int64_t b = 0; b < B; ++b) {
      double prod = 1.0, pprod = 1.0;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == n) continue;
        uint64_t u = orc_word(seed, iter, (uint32_t)b, 0, (uint32_t)pos);
        uint64_t r = orc_scale(u, T[k]);
        int64_t i = orc_count_le(q[k], dims[k], r);
        idx[b * (N - 1) + pos] = (int32_t)i;
        double pt = (double)((uint64_t)dims[k] * q[k][i]) / (double)T[k];
        prod = (pos == 0) ? pt : prod * pt;
        double pk = (double)q[k][i] / (double)T[k];
        pprod = (pos == 0) ? pk : pprod * pk;
        ++pos;
      }
      w[b] = 1.0 / ((double)B * prod);
      if (pj) pj[b] = pprod;
    }
    if (B_eff_out) *B_eff_out = B;
    return ORC_OK;
  }
  if (strategy == ORC_BLOCK_LEVERAGE || strategy == ORC_BLOCK_EUCLIDEAN) {
    int32_t win[16], start[16], len[16];
    if (N - 1 > 16) return ORC_EINVAL;
    if (window_in)
      for (int p = 0; p < N - 1; ++p) win[p] = window_in[p];
    else
      orc_default_windows(N, dims, n, B, win);
    double prod = 1.0, pprod = 1.0;
    int64_t Beff = 1;
    int pos = 0;
    for (int k = 0; k < N; ++k) {
      if (k == n) continue;
      int64_t bk = win[pos];
      if (bk < 1) return ORC_EINVAL;
      if (bk > dims[k]) bk = dims[k];
      int64_t D = (dims[k] + bk - 1) / bk; /* ceil(I_k / b_k) windows; the last one is ragged */
      /* window masses Q_d = sum_{i in tau_d} q_i (Defs. 3.1-3.2 in fixed point) */
      uint64_t* Qw = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)D);
      if (!Qw) return ORC_ENOMEM;
      for (int64_t d = 0; d < D; ++d) {
        Qw[d] = 0;
        for (int64_t i = d * bk; i < dims[k] && i < (d + 1) * bk; ++i) Qw[d] += q[k][i];
      }
      uint64_t u = orc_word(seed, iter, 0u, 1, (uint32_t)pos);
      uint64_t r = orc_scale(u, T[k]);
      int64_t d = orc_count_le(Qw, D, r);
      start[pos] = (int32_t)(d * bk);
      len[pos] = (int32_t)((d + 1) * bk <= dims[k] ? bk : dims[k] - d * bk);
      double pt = (double)((uint64_t)dims[k] * Qw[d]) / (double)T[k];
      prod = (pos == 0) ? pt : prod * pt;
      double pk = (double)Qw[d] / (double)T[k];
      pprod = (pos == 0) ? pk : pprod * pk;
      Beff *= len[pos];
      free(Qw);
      ++pos;
    }
    /* tuples of the Cartesian product in index-map order (first remaining position fastest) */
    for (int64_t t = 0; t < Beff; ++t) {
      int64_t rem = t;
      for (int p = 0; p < N - 1; ++p) {
        idx[t * (N - 1) + p] = start[p] + (int32_t)(rem % len[p]);
        rem /= len[p];
      }
      w[t] = 1.0 / prod;
      if (pj) pj[t] = pprod;
    }
    if (B_eff_out) *B_eff_out = Beff;
    return ORC_OK;
  }
  return ORC_EINVAL;
}

/* ------------------------------------------------------------------------------------
 * Stratified per-slab sampling (reading R26 in DESIGN.md): the row-wise draws of
 * eq:ik with the batch split into P strata, one per slab of the LAST mode.
 *   slabs    : P contiguous ranges [lo_g, hi_g) of the last mode's index, lo[0] = 0, lo[P] = I_{N-1}
 *   strata   : stratum g = batch rows [off_g, off_g + B_g), B_g = floor(B/P) + (g < B mod P), B >= P
 *   draws    : every remaining mode k < N-1 exactly as orc_sample (same Philox counter of row b and
 *              position); the last mode from the slab's conditional law q_i / Q_g (i in slab g,
 *              Q_g = sum of q over the slab): r = (q_0 + ... + q_{lo_g - 1}) + floor(u Q_g / 2^64), i =
 *              #{i : cdf_i <= r}, which lies in the slab.
 *   estimator: unbiased stratum by stratum (the argument of Theorem 5.1, applied
 *              to each stratum: E over stratum g of (1/B_g) sum_b g_{j_b} / P_g(j_b) = sum_{j in g} g_j),
 *              so w_b = 1/(B_g prod_k ptilde_k) with ptilde_k = I_k q_k/T_k (k < N-1) and
 *              ptilde_{N-1} = I_{N-1} q_i / Q_g, in that order (contract of DESIGN.md section 4);
 *              pj_b = (B_g / B) prod_k (q_k/T_k or q_i/Q_g), so that orc_gradient's 1/(B J_n pj_b) = w_b.
 *   Q_g = 0  : the slab has probability 0 (no fibers of it could be drawn unstratified either): the
 *              stratum's rows take i = lo_g, w = 0, pj = +inf (they contribute nothing).
 * Mode n == N-1 (every fiber spans all slabs): no strata, identical to orc_sample.  Row-wise
 * strategies only (uniform / leverage / Euclidean); ORC_EINVAL otherwise, or when B < P.
 * ---------------------------------------------------------------------------------- */
int orc_sample_stratified(int N, const int64_t* dims, int n, int strategy, int64_t B, const uint64_t* const* q,
                          const uint64_t* T, uint64_t seed, uint64_t iter, int P, const int64_t* slab_lo,
                          int32_t* idx, double* w, double* pj) {
  if (N < 3 || n < 0 || n >= N || B < 1 || P < 1) return ORC_EINVAL;
  if (!(strategy == ORC_UNIFORM || strategy == ORC_LEVERAGE || strategy == ORC_EUCLIDEAN)) return ORC_EINVAL;
  if (n == N - 1 || P == 1) return orc_sample(N, dims, n, strategy, B, NULL, q, T, seed, iter, idx, w, pj, NULL);
  if (B < P || slab_lo[0] != 0 || slab_lo[P] != dims[N - 1]) return ORC_EINVAL;
  for (int g = 0; g < P; ++g)
    if (slab_lo[g + 1] <= slab_lo[g]) return ORC_EINVAL;
  const int64_t IL = dims[N - 1];
  int64_t b = 0;
  for (int g = 0; g < P; ++g) {
    const int64_t Bg = B / P + (g < B % P ? 1 : 0);
    const int64_t lo = slab_lo[g], hi = slab_lo[g + 1];
    uint64_t base = 0, Qg = 0;
    for (int64_t i = 0; i < lo; ++i) base += q[N - 1][i];
    for (int64_t i = lo; i < hi; ++i) Qg += q[N - 1][i];
    for (int64_t t = 0; t < Bg; ++t, ++b) {
      double prod = 1.0, pprod = 1.0;
      int pos = 0;
      for (int k = 0; k < N; ++k) {
        if (k == n) continue;
        uint64_t u = orc_word(seed, iter, (uint32_t)b, 0, (uint32_t)pos);
        int64_t i;
        double pt, pk;
        if (k < N - 1) {
          uint64_t r = orc_scale(u, T[k]);
          i = orc_count_le(q[k], dims[k], r);
          pt = (double)((uint64_t)dims[k] * q[k][i]) / (double)T[k];
          pk = (double)q[k][i] / (double)T[k];
        } else if (Qg > 0) {
          uint64_t r = base + orc_scale(u, Qg);
          i = orc_count_le(q[k], IL, r);
          pt = (double)((uint64_t)IL * q[k][i]) / (double)Qg;
          pk = (double)q[k][i] / (double)Qg;
        } else {
          i = lo;
          pt = 0.0;
          pk = 0.0;
        }
        idx[b * (N - 1) + pos] = (int32_t)i;
        prod = (pos == 0) ? pt : prod * pt;
        pprod = (pos == 0) ? pk : pprod * pk;
        ++pos;
      }
      if (Qg > 0) {
        w[b] = 1.0 / ((double)Bg * prod);
        if (pj) pj[b] = ((double)Bg / (double)B) * pprod;
      } else {
        w[b] = 0.0;
        if (pj) pj[b] = INFINITY;
      }
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------------------
 * Stochastic gradient, literally as eq:gradient1 (4.1) for the row-wise
 * strategies and uniform (BrasCPD, :155, reading R1) and eq:gradient2 (4.2, :450-457) for the
 * block strategies; D placed as Z^T D Z and X D Z (reading R2 of the garbled :442):
 *   row-wise: G = 1/(B J_n) (A (Z^T D Z) - (X_F D) Z),   D = diag(1/p_{j_b})
 *   block   : G = 1/(p_S J_n) (A (Z^T Z) - X_S Z)
 * Outputs (any may be NULL): G (I_n x R), Gamma = scale * Z^T D Z (R x R), M = scale * X_F D Z.
 * pj[] are the per-row probabilities from orc_sample (block: p_S in every entry).
 * ---------------------------------------------------------------------------------- */
static int orc_gradient_x(int N, const int64_t* dims, int R, const void* X, int xf32, const double* const* factors,
                          int n, int strategy, int64_t B, int64_t B_eff, const int32_t* idx, const double* pj,
                          double* G_out, double* Gamma_out, double* M_out) {
  int64_t In = dims[n];
  int64_t Jn = 1;
  for (int k = 0; k < N; ++k)
    if (k != n) Jn *= dims[k];
  double* Z = (double*)malloc(sizeof(double) * (size_t)(B_eff * R));
  double* XF = (double*)malloc(sizeof(double) * (size_t)(B_eff * In));
  double* C1 = (double*)malloc(sizeof(double) * (size_t)(R * R));
  double* C2 = (double*)malloc(sizeof(double) * (size_t)(In * R));
  if (!Z || !XF || !C1 || !C2) {
    free(Z); free(XF); free(C1); free(C2);
    return ORC_ENOMEM;
  }
  int st = orc_skr(N, dims, R, factors, n, B_eff, idx, Z);
  if (!st) st = orc_tensor_samp_x(N, dims, X, xf32, n, B_eff, idx, XF);
  if (st) {
    free(Z); free(XF); free(C1); free(C2);
    return st;
  }
  int block = (strategy == ORC_BLOCK_LEVERAGE || strategy == ORC_BLOCK_EUCLIDEAN);
  double scale;
  /* C1 = Z^T D Z, C2 = (X_F D) Z with D = diag(1/p_j) (row-wise) or I (block); b ascending */
  for (int r1 = 0; r1 < R; ++r1)
    for (int r2 = 0; r2 < R; ++r2) {
      double s = 0.0;
      for (int64_t b = 0; b < B_eff; ++b) {
        double d = block ? 1.0 : 1.0 / pj[b];
        s += Z[b * R + r1] * (d * Z[b * R + r2]);
      }
      C1[r1 * R + r2] = s;
    }
  for (int64_t i = 0; i < In; ++i)
    for (int r = 0; r < R; ++r) {
      double s = 0.0;
      for (int64_t b = 0; b < B_eff; ++b) {
        double d = block ? 1.0 : 1.0 / pj[b];
        s += (XF[b * In + i] * d) * Z[b * R + r];
      }
      C2[i * R + r] = s;
    }
  if (block)
    scale = 1.0 / (pj[0] * (double)Jn);
  else
    scale = 1.0 / ((double)B * (double)Jn);
  if (Gamma_out)
    for (int t = 0; t < R * R; ++t) Gamma_out[t] = scale * C1[t];
  if (M_out)
    for (int64_t t = 0; t < In * R; ++t) M_out[t] = scale * C2[t];
  if (G_out) {
    const double* A = factors[n];
    for (int64_t i = 0; i < In; ++i)
      for (int r = 0; r < R; ++r) {
        double s = 0.0;
        for (int c = 0; c < R; ++c) s += A[i * R + c] * C1[c * R + r];
        G_out[i * R + r] = scale * (s - C2[i * R + r]);
      }
  }
  free(Z); free(XF); free(C1); free(C2);
  return ORC_OK;
}

int orc_gradient(int N, const int64_t* dims, int R, const double* X, const double* const* factors, int n,
                 int strategy, int64_t B, int64_t B_eff, const int32_t* idx, const double* pj, double* G_out,
                 double* Gamma_out, double* M_out) {
  return orc_gradient_x(N, dims, R, X, 0, factors, n, strategy, B, B_eff, idx, pj, G_out, Gamma_out, M_out);
}

/* Gamma^+ of a symmetric R x R matrix on its numerically full-rank pivot set: the symmetric sweep
 * operator in natural order, pivot k swept when its current diagonal exceeds
 * tol = R * eps * max_i Gam_ii (reading R25: the rank rule of the sampled-ALS solve); on the swept
 * set S, W_SS = (Gam_SS)^{-1}, zero elsewhere.  Plain O(R^3) loops.  Returns |S|. */
int orc_sym_pinv(int R, const double* Gam, double* W) {
  double* M = (double*)malloc(sizeof(double) * (size_t)(R * R));
  double* rk = (double*)malloc(sizeof(double) * (size_t)R);
  int* swept = (int*)calloc((size_t)R, sizeof(int));
  if (!M || !rk || !swept) {
    free(M); free(rk); free(swept);
    return -1;
  }
  double dmax = 0.0;
  for (int i = 0; i < R * R; ++i) M[i] = Gam[i];
  for (int i = 0; i < R; ++i)
    if (M[i * R + i] > dmax) dmax = M[i * R + i];
  const double tol = (double)R * 2.220446049250313e-16 * dmax;
  int rank = 0;
  for (int k = 0; k < R; ++k) {
    const double d = M[k * R + k];
    if (!(d > tol)) continue;
    for (int j = 0; j < R; ++j) rk[j] = M[k * R + j];  /* row k before the step (= column k) */
    for (int i = 0; i < R; ++i) {
      if (i == k) continue;
      for (int j = 0; j < R; ++j) {
        if (j == k) continue;
        M[i * R + j] -= rk[i] * rk[j] / d;
      }
    }
    for (int j = 0; j < R; ++j)
      if (j != k) {
        M[k * R + j] = rk[j] / d;
        M[j * R + k] = rk[j] / d;
      }
    M[k * R + k] = -1.0 / d;
    swept[k] = 1;
    ++rank;
  }
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) W[i * R + j] = (swept[i] && swept[j]) ? -M[i * R + j] : 0.0;
  free(M); free(rk); free(swept);
  return rank;
}

/* The sampled least-squares step of eq:lsq_krp: the sampled normal equations
 * A Gamma = M (Gamma, M of eq:gradient1/2, scaled alike) solved as A = M Gamma^+. */
int orc_update_als(int64_t I, int R, double* A, const double* M, const double* Gam) {
  double* W = (double*)malloc(sizeof(double) * (size_t)(R * R));
  if (!W) return ORC_ENOMEM;
  if (orc_sym_pinv(R, Gam, W) < 0) {
    free(W);
    return ORC_ENOMEM;
  }
  for (int64_t i = 0; i < I; ++i)
    for (int r = 0; r < R; ++r) {
      double s = 0.0;
      for (int c = 0; c < R; ++c) s += M[i * R + c] * W[c * R + r];
      A[i * R + r] = s;
    }
  free(W);
  return ORC_OK;
}

/* eq:proposed (4.3): A <- A - alpha G */
void orc_update_fixed(int64_t I, int R, double* A, const double* G, double alpha) {
  for (int64_t t = 0; t < I * R; ++t) A[t] = A[t] - alpha * G[t];
}

/* eq:etaada / eq:Aada (4.4a/b), with S the running sum of G^2 over this
 * mode's updates including the current one (reading R12); entries with S = 0 are left
 * unchanged (their G is 0). */
void orc_update_adaptive(int64_t I, int R, double* A, double* S, const double* G, double eta, double b, double eps) {
  for (int64_t t = 0; t < I * R; ++t) {
    S[t] = S[t] + G[t] * G[t];
    if (S[t] > 0.0) {
      double step = eta / pow(b + S[t], 0.5 + eps);
      A[t] = A[t] - step * G[t];
    }
  }
}

/* fit = 1 - ||X - [[A]]||_F / ||X||_F by direct loops (objective PAPER.md:118-127; reading R14) */
int orc_fit(int N, const int64_t* dims, const double* X, int R, const double* const* factors, double* fit,
            double* resid2_out, double* xnorm2_out) {
  int64_t total = 1;
  for (int k = 0; k < N; ++k) total *= dims[k];
  int64_t sub[32];
  if (N > 32) return ORC_EINVAL;
  for (int k = 0; k < N; ++k) sub[k] = 0;
  double res2 = 0.0, x2 = 0.0;
  for (int64_t off = 0; off < total; ++off) {
    double xhat = 0.0;
    for (int r = 0; r < R; ++r) {
      double prod = 1.0;
      for (int k = 0; k < N; ++k) prod *= factors[k][sub[k] * R + r];
      xhat += prod;
    }
    double d = X[off] - xhat;
    res2 += d * d;
    x2 += X[off] * X[off];
    for (int k = 0; k < N; ++k) { /* first index fastest */
      if (++sub[k] < dims[k]) break;
      sub[k] = 0;
    }
  }
  if (resid2_out) *resid2_out = res2;
  if (xnorm2_out) *xnorm2_out = x2;
  if (!(x2 > 0.0)) return ORC_EDEGENERATE;
  *fit = 1.0 - sqrt(res2) / sqrt(x2);
  return ORC_OK;
}

/* mode of iteration r under random order: floor(y0 * N / 2^32) from purpose 2 */
int orc_random_mode(uint64_t seed, uint64_t iter, int N) {
  uint32_t ctr[4] = {0u, (2u << 24) | 0u, (uint32_t)iter, (uint32_t)(iter >> 32)};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t y[4];
  orc_philox4x32_10(ctr, key, y);
  return (int)(((uint64_t)y[0] * (uint64_t)N) >> 32);
}

/* ------------------------------------------------------------------------------------
 * Alg. 6 BrawsCPD / Alg. 7 AdawsCPD (:548-568) main loop, `iters`
 * iterations starting at iteration counter r0.  Per iteration: choose n (cyclic i mod N
 * within this call, or random), sample with tables of the current factors, TensorSamp,
 * gradient, update A^(n), rebuild table n (reading R9).  factors and S (may be NULL for the
 * fixed rule) are updated in place.  alpha: per-iteration array (fixed rule) or NULL ->
 * alpha0.  Workspace is allocated here.  modes_out (optional) records n per iteration.
 * ---------------------------------------------------------------------------------- */
static int orc_run_x(int N, const int64_t* dims, int R, const void* X, int xf32, double* const* factors,
                     double* const* S, int strategy, int rule, int order, int first_mode, int64_t B,
                     const int32_t* window, double alpha0, const double* alpha, double eta, double bpar, double eps,
                     uint64_t seed, uint64_t r0, int64_t iters, int32_t* modes_out) {
  if (N < 3 || N > 16 || R < 1 || B < 1) return ORC_EINVAL;
  uint64_t* q[16];
  uint64_t T[16];
  int64_t Imax = 0, Bmax = B;
  for (int k = 0; k < N; ++k) {
    if (dims[k] > Imax) Imax = dims[k];
    q[k] = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)dims[k]);
    if (!q[k]) return ORC_ENOMEM;
  }
  if (strategy == ORC_BLOCK_LEVERAGE || strategy == ORC_BLOCK_EUCLIDEAN) {
    /* the Cartesian batch is at most prod(window) <= B (windows clamp to I_k) */
    Bmax = B;
    if (window) {
      Bmax = 1;
      for (int p = 0; p < N - 1; ++p) Bmax *= window[p];
    }
  }
  int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(Bmax * (N - 1)));
  double* w = (double*)malloc(sizeof(double) * (size_t)Bmax);
  double* pj = (double*)malloc(sizeof(double) * (size_t)Bmax);
  double* G = (double*)malloc(sizeof(double) * (size_t)(Imax * R));
  double* Gam = (double*)malloc(sizeof(double) * (size_t)(R * R));
  double* Mm = (double*)malloc(sizeof(double) * (size_t)(Imax * R));
  int st = (!idx || !w || !pj || !G || !Gam || !Mm) ? ORC_ENOMEM : ORC_OK;
  for (int k = 0; k < N && !st; ++k) st = orc_build_table(strategy, dims[k], R, factors[k], NULL, q[k], &T[k]);
  for (int64_t it = 0; it < iters && !st; ++it) {
    uint64_t r = r0 + (uint64_t)it;
    int n = (order == ORC_ORDER_RANDOM) ? orc_random_mode(seed, r, N) : (int)((first_mode + it) % N);
    if (modes_out) modes_out[it] = n;
    int64_t Beff = 0;
    st = orc_sample(N, dims, n, strategy, B, window, (const uint64_t* const*)q, T, seed, r, idx, w, pj, &Beff);
    if (st) break;
    st = orc_gradient_x(N, dims, R, X, xf32, (const double* const*)factors, n, strategy, B, Beff, idx, pj, G, Gam, Mm);
    if (st) break;
    if (rule == ORC_STEP_ADAPTIVE)
      orc_update_adaptive(dims[n], R, factors[n], S[n], G, eta, bpar, eps);
    else if (rule == ORC_STEP_ALS)
      st = orc_update_als(dims[n], R, factors[n], Mm, Gam);
    else
      orc_update_fixed(dims[n], R, factors[n], G, alpha ? alpha[it] : alpha0);
    if (st) break;
    st = orc_build_table(strategy, dims[n], R, factors[n], NULL, q[n], &T[n]);
  }
  for (int k = 0; k < N; ++k) free(q[k]);
  free(idx); free(w); free(pj); free(G); free(Gam); free(Mm);
  return st;
}

int orc_run(int N, const int64_t* dims, int R, const double* X, double* const* factors, double* const* S,
            int strategy, int rule, int order, int64_t B, const int32_t* window, double alpha0,
            const double* alpha, double eta, double bpar, double eps, uint64_t seed, uint64_t r0, int64_t iters,
            int32_t* modes_out) {
  return orc_run_x(N, dims, R, X, 0, factors, S, strategy, rule, order, 0, B, window, alpha0, alpha, eta, bpar, eps,
                   seed, r0, iters, modes_out);
}

/* orc_run on an fp32-stored tensor (each element converted to fp64 on read; factors, accumulators and
 * every operation fp64 as in orc_run) */
int orc_run_f32(int N, const int64_t* dims, int R, const float* X, double* const* factors, double* const* S,
                int strategy, int rule, int order, int64_t B, const int32_t* window, double alpha0,
                const double* alpha, double eta, double bpar, double eps, uint64_t seed, uint64_t r0, int64_t iters,
                int32_t* modes_out) {
  return orc_run_x(N, dims, R, X, 1, factors, S, strategy, rule, order, 0, B, window, alpha0, alpha, eta, bpar, eps,
                   seed, r0, iters, modes_out);
}

/* orc_run / orc_run_f32 with the cyclic order starting at mode first_mode (iteration it of the call
 * updates mode (first_mode + it) mod N): a run split into calls continues the sweep */
int orc_run_from(int N, const int64_t* dims, int R, const void* X, int xf32, double* const* factors,
                 double* const* S, int strategy, int rule, int order, int first_mode, int64_t B,
                 const int32_t* window, double alpha0, const double* alpha, double eta, double bpar, double eps,
                 uint64_t seed, uint64_t r0, int64_t iters, int32_t* modes_out) {
  if (first_mode < 0 || first_mode >= N) return ORC_EINVAL;
  return orc_run_x(N, dims, R, X, xf32, factors, S, strategy, rule, order, first_mode, B, window, alpha0, alpha, eta,
                   bpar, eps, seed, r0, iters, modes_out);
}
