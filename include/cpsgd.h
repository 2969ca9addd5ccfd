/*
 * cpsgd.h -- C ABI of the B200-native importance-sampled mini-batch SGD step for the
 * Khatri-Rao-structured least-squares subproblem of CP-ALS (arXiv 2103.04081, the
 * BrawsCPD / AdawsCPD methods).  Implemented by libcpsgd.so (hand-written sm_100a CUDA).
 *
 * Citations are PAPER.md:<lines> (<LaTeX label>) of the paper text; "R<k>" refers to the
 * numbered readings in DESIGN.md where the paper is silent, ambiguous or garbled.
 *
 * Conventions (all calls):
 *   - Every call returns cp_status: CP_OK (0) or a negative error code.  No C++ exception,
 *     abort or exit crosses this boundary.  cp_sgd_last_error(h) gives a message.
 *   - Indices are 0-based (the paper is 1-based, R16).  The dense tensor is stored
 *     first-index-fastest: element (i_0..i_{N-1}) at offset sum_k i_k S_k, S_k = prod_{m<k} I_m
 *     (PAPER.md:47-50 eq:map, R17).  Factor matrices are row-major I_n x R.
 *   - Pointers named *_dev are CUDA device pointers, *_host host pointers.
 *   - Ownership: X and the factors are BORROWED from the caller (e.g. torch tensors) and must
 *     outlive the handle; X is never written; factors are written only by step/sweep calls.
 *     The handle OWNS its workspace (tables, samples, partial sums, adaptive accumulators,
 *     optional mode-major copies of X, the NCCL communicator) and frees it in cp_sgd_destroy.
 *   - Asynchrony: work is enqueued on cfg.stream (a cudaStream_t, 0 = legacy default stream).
 *     Calls documented as "synchronises" wait for the stream and report device-side errors
 *     (degenerate or non-finite importance tables) raised by earlier asynchronous calls.
 *   - One host thread per handle.
 */
#ifndef CPSGD_H
#define CPSGD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct cp_sgd_s* cp_sgd_t;

typedef enum {
  CP_OK = 0,
  CP_EINVAL = -1,       /* bad configuration or argument                                  */
  CP_ERANGE = -2,       /* index/mode out of range                                        */
  CP_EDEGENERATE = -3,  /* all-zero factor -> empty distribution, or ||X|| = 0 in cp_fit   */
  CP_ENOMEM = -4,       /* device or host allocation failed                               */
  CP_ECUDA = -5,        /* CUDA runtime error                                             */
  CP_ENCCL = -6,        /* NCCL error (world > 1)                                         */
  CP_ESTATE = -7,       /* call not valid in the handle's state                           */
  CP_ENONFINITE = -8    /* a table rebuild met a NaN/Inf factor (e.g. a diverged step size) */
} cp_status;

typedef enum { CP_F32 = 0, CP_F64 = 1 } cp_dtype;

/* Sampling strategies: uniform = BrasCPD (Alg. 2); leverage / Euclidean =
 * KrpSamp1 (Alg. 3); block-leverage / block-Euclidean = KrpSamp2 (Alg. 4,
 * PAPER.md:412-428; Cartesian windows, R2/R6). */
typedef enum {
  CP_UNIFORM = 0,
  CP_LEVERAGE = 1,
  CP_EUCLIDEAN = 2,
  CP_BLOCK_LEVERAGE = 3,
  CP_BLOCK_EUCLIDEAN = 4
} cp_sampler;

/* fixed step = eq:proposed (BrawsCPD Alg. 6); adaptive = eq:etaada/eq:Aada
 * (AdawsCPD Alg. 7). */
/* CP_STEP_ALS: the sampled least-squares step of eq:lsq_krp on the same batch,
 * A^(n) <- M Gamma^+ (M, Gamma of eq:gradient1/2; Gamma^+ by the natural-order symmetric sweep on its
 * numerically full-rank pivot set, tol = R eps max_i Gamma_ii, reading R25).  Single
 * GPU, fused or wide path only (CP_EINVAL otherwise). */
typedef enum { CP_STEP_FIXED = 0, CP_STEP_ADAPTIVE = 1, CP_STEP_ALS = 2 } cp_step_rule;

/* mode order of a sweep: cyclic 0..N-1, or n drawn uniformly per iteration */
typedef enum { CP_ORDER_CYCLIC = 0, CP_ORDER_RANDOM = 1 } cp_mode_order;

/* flags */
#define CP_FLAG_MODE_MAJOR 0x1u   /* keep mode-major copies X_(n)^T ([J_n][I_n], fiber-contiguous) for
                                     n >= 1 so every sampled fiber is one contiguous row (DESIGN.md
                                     "Data layout"); costs (N-1) extra tensor-sized buffers; a mode whose
                                     copy does not fit the free device memory (less 2 GiB) keeps the native
                                     layout                                                         */
#define CP_FLAG_NO_GRAPH 0x2u     /* never capture CUDA graphs for sweeps                              */
#define CP_FLAG_NO_FUSED 0x8u      /* never use the persistent single-cluster sweep kernel (small problems
                                     otherwise run whole step sequences in one launch)               */
#define CP_FLAG_EXTERNAL_COMM 0x4u /* world > 1 without an internal NCCL communicator: the caller
                                     performs the exchange between the phases of cp_sgd_step_phase  */
#define CP_FLAG_NO_TC 0x20u        /* fp32 wide path: FFMA mainloop instead of tcgen05 3xTF32       */
#define CP_FLAG_FUSED_CU8 0x40u    /* fused path on 8-CTA clusters instead of 16: slower per chain, but
                                      two chains fit one GPC (cp_sgd_sweep_multi throughput mode)   */
#define CP_FLAG_NO_WIDE 0x10u      /* single GPU, split path: never use the fused gather + update kernel
                                     (k_gather_update); use the gather-partials + update-table pair */
#define CP_FLAG_STRATIFIED 0x100u  /* world > 1 (slab sharding), row-wise samplers: stratified per-slab sampling
                                      (reading R26 in DESIGN.md): for modes n < N-1 the batch
                                      is split into world_size strata, B_g = floor(B/P) (+1 for g < B mod P)
                                      rows each, and stratum g draws the last mode from the conditional law
                                      of slab g (q_i / Q_g); weights omega_b = 1/(B_g prod_k ptilde_k) with
                                      ptilde_{N-1} = I_{N-1} q_i / Q_g -- unbiased stratum by stratum
                                      (Theorem 5.1); a zero-mass slab gives its rows
                                      omega = 0.  Every rank then gathers exactly B_g fibers (its own
                                      stratum): balanced owner-computes.  Mode N-1 is unchanged.  Needs
                                      slab_bounds with CP_FLAG_EXTERNAL_COMM; CP_EINVAL for block samplers,
                                      B < world_size or world_size > 16. */
#define CP_FLAG_REPLICA 0x200u     /* world > 1 with the WHOLE tensor on every rank (BASELINE C4 at 2-8 GPUs;
                                      SURVEY 8(e) "C4 alternative"): every rank draws the same global batch and
                                      runs the replicated update / table / next batch, but gathers and contracts
                                      only the wide path's batch chunks c = rank, rank + P, ... (perfect balance,
                                      any strategy); M = the sum over ranks of each rank's chunk sum (ncclAllReduce
                                      on the library stream, or by the caller between phases 0 and 1 with
                                      CP_FLAG_EXTERNAL_COMM: cp_sgd_exchange_info / _copy expose that buffer,
                                      [ceil(I_n/128)][R][128] of cfg.dtype).  slab_begin/end are ignored.  Needs
                                      the wide path for every mode (CP_EINVAL otherwise); excludes STRATIFIED. */
#define CP_FLAG_FORCE_COMM 0x400u  /* test hook: a world_size == 1 handle that still takes the multi-rank code
                                      path (slab sharding, or REPLICA) with a 1-rank NCCL communicator from
                                      nccl_unique_id (or the caller's exchanges with EXTERNAL_COMM), so the
                                      library's NCCL calls run on a one-GPU machine */
#define CP_FLAG_P2P 0x800u        /* with CP_FLAG_REPLICA: M is exchanged over peer memory (NVLink / NVSwitch)
                                      instead of an allreduce -- each rank publishes its chunk sum in its own
                                      symmetric buffer (cp_sgd_p2p_buffer) and the update kernel sums the P
                                      ranks' copies in rank order straight from their memory (the collective
                                      fused into its consumer; bitwise identical M on every rank).  The caller
                                      maps the peers' buffers once (cp_ipc_get_handle + cp_sgd_p2p_open across
                                      processes, or cp_sgd_p2p_peers with pointers it can already address)
                                      before the first step; phases 0 and 1 of cp_sgd_step_phase then need no
                                      exchange in between.                                            */
#define CP_FLAG_NO_PERSIST 0x80u   /* fp32 wide path: never use the persistent cooperative sweep kernel
                                     (k_sweep_wide); run each step as the gather / update+table /
                                     sample kernel chain (graph-captured for cyclic sweeps)        */

typedef struct {
  int32_t order;               /* N >= 3                                                          */
  const int64_t* dims;         /* host, N entries, I_n >= 1 (GLOBAL sizes, also when sharded)      */
  int32_t rank;                /* CP rank R, 1 <= R <= 64                                          */
  int32_t dtype;               /* cp_dtype of X, factors and accumulators                          */
  const void* X;               /* device; local slab X[..., slab_begin:slab_end] when world > 1;   */
                               /* first-index-fastest; BORROWED read-only                          */
  void* const* factors;        /* host array of N device pointers, row-major I_n x R (all rows,    */
                               /* replicated on every rank); BORROWED, updated in place            */
  int64_t batch;               /* B >= 1: fibers per step (row-wise); nominal batch for block      */
  const int32_t* block_window; /* host, N-1 window lengths per remaining-mode position, or NULL    */
                               /* for the default (R6: smallest divisor d of the remaining batch   */
                               /* with d^(positions left) >= remaining batch, clamped to I_k)      */
  int32_t sampler;             /* cp_sampler                                                       */
  int32_t rule;                /* cp_step_rule                                                     */
  double alpha;                /* fixed rule: default step (>= 0) when a call passes none          */
  double eta, b, eps;          /* adaptive rule: eta > 0, b >= 0, eps >= 0      */
  uint64_t seed;               /* Philox key of the sampling contract                              */
  void* stream;                /* cudaStream_t                                                     */
  int32_t world_rank;          /* this process's rank, 0 <= world_rank < world_size                */
  int32_t world_size;          /* 1 = single GPU                                                   */
  const void* nccl_unique_id;  /* 128-byte ncclUniqueId, world_size > 1 without EXTERNAL_COMM      */
  int64_t slab_begin, slab_end;/* local range of the LAST mode's index (slab sharding); ignored
                                  (whole tensor) when world_size == 1                              */
  uint32_t flags;              /* CP_FLAG_*                                                        */
  const int64_t* slab_bounds;  /* host, world_size + 1 entries: slab g = [slab_bounds[g], slab_bounds[g+1])
                                  of the last mode, contiguous in rank order, slab_bounds[0] = 0 and
                                  slab_bounds[world_size] = I_{N-1}, this rank's entry equal to
                                  [slab_begin, slab_end); or NULL (the ranks' ranges are exchanged over the
                                  internal communicator).  Read at init only.                      */
} cp_sgd_config;

/* Create a handle: validates cfg (CP_EINVAL: N < 3 or > 16, R < 1 or > 64, B < 1, eta <= 0,
 * b < 0, eps < 0, alpha < 0, NULL pointers, bad slab range), allocates the workspace, builds
 * the optional mode-major copies and the importance tables of every mode from the current
 * factors (R9).  Iteration counter r = 0. */
cp_status cp_sgd_init(const cp_sgd_config* cfg, cp_sgd_t* out);

/* Destroy a handle and free everything it owns.  NULL is a no-op. */
cp_status cp_sgd_destroy(cp_sgd_t h);

/* Message for the last error of h (or of the last failed cp_sgd_init when h == NULL). */
const char* cp_sgd_last_error(cp_sgd_t h);

/* rows a step of `mode` draws at most: B (row-wise, uniform) or prod(window) (block) */
cp_status cp_sgd_batch_max(cp_sgd_t h, int32_t mode, int64_t* bmax_host);

/* KrpSamp1 / KrpSamp2 index draws for mode `mode` at iteration `iter` (Alg. 3 / Alg. 4 with
 * eq:ik, eq:bik), a pure function of (current tables, seed, iter, mode):
 *   idx_dev : out, device int32 [B_max][N-1] (positions = modes k != mode ascending; B_max = batch,
 *             or prod(window) for block strategies)
 *   w_dev   : out, device fp64 [B_max], omega_b = 1/(B J_n p_{j_b}) (row-wise, eq:gradient1) or
 *             1/(J_n p_S) (block, eq:gradient2), computed in the contract's exact operation order
 *   batch_eff_host : out (may be NULL), number of valid rows; non-NULL synchronises.          */
cp_status cp_sgd_sample(cp_sgd_t h, int32_t mode, uint64_t iter, int32_t* idx_dev, double* w_dev,
                        int64_t* batch_eff_host);

/* One iteration of Alg. 6 (fixed rule, step alpha >= 0; alpha < 0 means cfg.alpha) or Alg. 7
 * (adaptive; alpha ignored) on mode `mode` at iteration r: sample (Alg. 3/4), TensorSamp
 * (Alg. 5) + SKR (Alg. 1), gradient eq:gradient1 / eq:gradient2, update A^(mode) (eq:proposed /
 * eq:Aada), rebuild table `mode` (R9); then r += 1.  Asynchronous. */
cp_status cp_sgd_step(cp_sgd_t h, int32_t mode, double alpha);

/* nsweeps x N iterations of cp_sgd_step with modes in `order` (cyclic: 0..N-1 per sweep;
 * random: n = floor(y0 N / 2^32) of Philox purpose 2 at iteration r).  alpha_per_iter: host,
 * nsweeps*N entries for the fixed rule, or NULL for cfg.alpha / the adaptive rule.  Cyclic
 * sweeps with a constant step are replayed from a captured CUDA graph.  Asynchronous. */
cp_status cp_sgd_sweep(cp_sgd_t h, int32_t nsweeps, int32_t order, const double* alpha_per_iter);

/* Many independent chains in ONE launch: nsweeps cyclic sweeps (constant step:
 * cfg.alpha / the adaptive or ALS rule) of each of the nh handles, one thread-block cluster per
 * chain.  Every handle must be on the fused single-GPU path with the same geometry (dtype, dims, R,
 * fused plan); samplers, rules, seeds, tensors and factors may differ.  Launched on hs[0]'s stream
 * after the other handles' streams are synchronised; their later work is ordered after it.
 * Results equal nh separate cp_sgd_sweep calls bit for bit.  Asynchronous.  CP_EINVAL otherwise. */
cp_status cp_sgd_sweep_multi(cp_sgd_t* hs, int32_t nh, int32_t nsweeps);

/* fit = 1 - ||X - [[A]]||_F / ||X||_F (PAPER.md:118-127 objective, R14), fp64 accumulation,
 * summed over ranks when sharded.  Synchronises.  CP_EDEGENERATE when ||X|| = 0. */
cp_status cp_fit(cp_sgd_t h, double* fit_host);

/* ---- replicas over peer memory (CP_FLAG_P2P) ------------------------------------------------------
 * cp_sgd_p2p_buffer: this handle's symmetric exchange buffer (device pointer, bytes) -- flags, then two
 *   parity copies of the rank's chunk sum of M; owned by the handle.
 * cp_ipc_get_handle: the 64-byte cudaIpcMemHandle of a device allocation (to send to the other ranks).
 * cp_sgd_p2p_open: map the world_size handles (64 bytes each, rank order; this rank's entry ignored) with
 *   cudaIpcOpenMemHandle (peer access enabled) and register them; the mappings are closed by destroy.
 * cp_sgd_p2p_peers: register world_size device pointers the calling process can address directly (rank
 *   order; entry world_rank must be this handle's own buffer).  Errors: CP_ESTATE on a handle without
 *   CP_FLAG_P2P, CP_EINVAL on NULL entries, CP_ECUDA when a mapping fails. */
cp_status cp_sgd_p2p_buffer(cp_sgd_t h, void** buf_dev, int64_t* bytes);
cp_status cp_ipc_get_handle(const void* dev_ptr, void* out64_host);
cp_status cp_sgd_p2p_open(cp_sgd_t h, const void* handles64_host);
cp_status cp_sgd_p2p_peers(cp_sgd_t h, void* const* peer_bufs_dev);
/* A fresh 128-byte ncclUniqueId from the NCCL library this library uses (rank 0 creates it and
 * broadcasts it to the other ranks, e.g. through torch.distributed, before cp_sgd_init). */
cp_status cp_nccl_unique_id(void* out128_host);
/* Squared Frobenius norms of the last-mode slices of a first-index-fastest tensor (or of a rank's local
 * slab): out_dev[i] = sum of x^2 over slice i (fp64, a fixed summation order), i < nslices <= 65535,
 * slice_len = product of the other dims.  No handle; enqueued on `stream` (cudaStream_t).  The data-side
 * proxy of the sampling mass the last factor's rows converge to, for mass-balanced contiguous slabs
 * (SURVEY 8(e) mitigation 2; host logic: paper_2103_04081_b200.parallel.balanced_slab_ranges). */
cp_status cp_slice_sqnorms(const void* X_dev, int32_t dtype, int64_t nslices, int64_t slice_len, double* out_dev,
                           void* stream);
/* Wait for the stream; report device-side errors of earlier asynchronous calls. */
cp_status cp_sgd_sync(cp_sgd_t h);

/* Host-buffer convenience path (the end-to-end call): copy the N factors from host buffers
 * (pinned recommended) to the device, run `nsteps` cyclic iterations starting at mode
 * `first_mode`, copy every factor back to the host buffers.  factors_host: N host pointers,
 * row-major I_n x R of cfg.dtype.  A host factor that differs bitwise from the device copy
 * replaces it and its table is rebuilt before the first iteration (R9: the tables are a function
 * of the factors; an unchanged factor keeps its table).  Synchronises. */
cp_status cp_sgd_steps_host(cp_sgd_t h, int32_t first_mode, int32_t nsteps, double alpha,
                            void* const* factors_host);

/* ---- split-phase step for sharded runs (world > 1) ------------------------------------
 * phase 0: sample + TensorSamp/SKR + local contraction into the exchange buffer
 *          (modes n < N-1: partial M, I_n x R, to be SUMMED over ranks; mode N-1: nothing)
 * phase 1: update A^(n) from the summed M (mode N-1: only the locally owned rows)
 * phase 2: (mode N-1: rows must have been gathered) rebuild table n; r += 1
 * With an internal communicator cp_sgd_step does all three plus the exchanges. */
cp_status cp_sgd_step_phase(cp_sgd_t h, int32_t mode, int32_t phase, double alpha);
/* device pointer / element count of the exchange buffer of `mode` after phase 0 (partial M to
 * be summed) -- and, for the last mode, the owned row range [row_begin, row_end) of A^(N-1)
 * to be gathered after phase 1. */
cp_status cp_sgd_exchange_info(cp_sgd_t h, int32_t mode, void** buf_dev, int64_t* count, int64_t* row_begin,
                               int64_t* row_end);

/* copy the exchange buffer of `mode` (the partial M after phase 0, R x I_n of cfg.dtype, layout
 * [R][I_n]) to (to_lib = 0) or from (to_lib = 1) a caller device buffer, on the handle's stream */
cp_status cp_sgd_exchange_copy(cp_sgd_t h, int32_t mode, void* buf_dev, int32_t to_lib);

/* ---- parity / debug hooks (synchronise) -------------------------------------------------- */
/* integer table of `mode`: q_host[I_mode] (may be NULL), T_host (may be NULL), p_host (fp64
 * probabilities before quantisation, may be NULL) */
cp_status cp_sgd_get_table(cp_sgd_t h, int32_t mode, uint64_t* q_host, uint64_t* T_host, double* p_host);
/* last gradient G (I_n x R of cfg.dtype) of the last step's mode, its mode, and Gamma (R x R) */
cp_status cp_sgd_get_grad(cp_sgd_t h, void* G_host, int32_t* mode_host, void* Gamma_host);
/* adaptive accumulator S^(mode) (I_mode x R of cfg.dtype) */
cp_status cp_sgd_get_accum(cp_sgd_t h, int32_t mode, void* S_host);
cp_status cp_sgd_get_iter(cp_sgd_t h, uint64_t* r_host);
cp_status cp_sgd_set_iter(cp_sgd_t h, uint64_t r);
/* rebuild every table from the current factors (after the caller changed factors) */
cp_status cp_sgd_refresh_tables(cp_sgd_t h);
/* number of kernels the library launched since the handle was created (graph nodes count) */
cp_status cp_sgd_get_launches(cp_sgd_t h, uint64_t* n_host);
/* per-step kernel names and their average device time over the last timed window (profiling):
 * cp_sgd_profile(h, 1) starts recording CUDA events around each kernel of subsequent
 * direct-launch steps, cp_sgd_profile(h, 0) stops; cp_sgd_profile_read returns up to `cap`
 * (kernel id, total ms, count) triples. */
cp_status cp_sgd_profile(cp_sgd_t h, int32_t on);
cp_status cp_sgd_profile_read(cp_sgd_t h, int32_t cap, int32_t* ids, double* total_ms, int64_t* counts,
                              int32_t* n_out);

/* debug trace of the batches the persistent kernels consume (k_sweep_wide, k_sweep_fused; other
 * paths record nothing).  cp_sgd_trace_layout returns the record layout: out[0] = stride (bytes per
 * SGD iteration), out[1..6] = byte offsets of idx (int32 [B_max][N-1]), w (fp64 [B_max]), the
 * updated factor A^(n) (dtype [I_n][R]), its accumulator S^(n) (adaptive rule), the new CDF of mode n
 * (uint64 [I_n]) and meta (int64 {n, r, B_eff, 0}).  cp_sgd_trace(h, buf, cap) starts recording into
 * the caller's device buffer buf (>= cap * stride bytes, BORROWED): the k-th SGD iteration run by a
 * persistent kernel after this call fills record k (k < cap; later ones are dropped); buf = NULL
 * stops.  cp_sgd_trace_count returns the number of iterations recorded since the last cp_sgd_trace. */
cp_status cp_sgd_trace_layout(cp_sgd_t h, int64_t* out7_host);
cp_status cp_sgd_trace(cp_sgd_t h, void* buf_dev, int64_t cap);
cp_status cp_sgd_trace_count(cp_sgd_t h, int64_t* n_host);

/* 1 if the handle runs its sweeps / steps on a persistent kernel (k_sweep_fused: 1, k_sweep_wide: 2),
 * 0 for kernel chains (also after the device refused k_sweep_wide's cooperative launch because its grid could not
 * be co-resident, e.g. with other work holding SMs: the handle then runs the same steps on the chain) */
cp_status cp_sgd_path(cp_sgd_t h, int32_t* path_host);

/* debug: clock64() phase timestamps of the last kernels (4096 kernel-specific entries, then the persistent
 * kernel's per-CTA marks [8 iterations][160 CTAs][32]: out16 holds 4096 + 40960 entries); only when the
 * environment variable CPSGD_DEBUG_TIMERS was set at cp_sgd_init, else CP_ESTATE */
cp_status cp_sgd_debug_timers(cp_sgd_t h, long long* out64_host);

/* library version string */
const char* cp_sgd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CPSGD_H */
