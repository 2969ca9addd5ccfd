// cpsgd.cu -- host side of libcpsgd.so: the C ABI of include/cpsgd.h.
//
// Orchestrates the sm_100a kernels of kernels.cuh on the caller's stream: per step
//   k_sample (a2,a3) -> k_gather (a4,a5,a6) -> [sharded: reduce + NCCL allreduce]
//   -> k_update (a6,a7,a8; r += 1) -> [sharded last mode: NCCL row broadcasts] -> k_table (a1, a9)
// Cyclic constant-step sweeps are captured once into a CUDA graph and replayed.
// NCCL is resolved at run time (dlopen of the libnccl.so.2 torch already loaded), only when
// world_size > 1 with an internal communicator.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/cpsgd.h"
#include "fused.cuh"
#include "gupdate.cuh"
#include "gupdate_tc.cuh"
#include "wide.cuh"
#include "sweep_wide_params.cuh"
#include "kernels.cuh"
#include "kptr.h"

using namespace cps;

namespace {

thread_local std::string g_init_error;

// ---- minimal NCCL surface (types match nccl.h 2.x) -------------------------------------------
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0 };
struct NcclApi {
  void* dl = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (dl) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      dl = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!dl) dl = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (dl) break;
    }
    if (!dl) {
      err = "cannot dlopen libnccl.so.2";
      return false;
    }
#define CPS_SYM(f, s)                                        \
  f = reinterpret_cast<decltype(f)>(dlsym(dl, s));           \
  if (!f) {                                                  \
    err = std::string("NCCL symbol missing: ") + s;          \
    return false;                                            \
  }
    CPS_SYM(CommInitRank, "ncclCommInitRank");
    CPS_SYM(AllReduce, "ncclAllReduce");
    CPS_SYM(Broadcast, "ncclBroadcast");
    CPS_SYM(GroupStart, "ncclGroupStart");
    CPS_SYM(GroupEnd, "ncclGroupEnd");
    CPS_SYM(CommDestroy, "ncclCommDestroy");
    CPS_SYM(GetErrorString, "ncclGetErrorString");
    CPS_SYM(GetUniqueId, "ncclGetUniqueId");
#undef CPS_SYM
    return true;
  }
};
NcclApi g_nccl;

enum KernelId { kKSample = 0, kKGather, kKUpdate, kKTable, kKReduce, kKComm, kKFit, kKFused, kKGatherUpdate, kKZwGamma, kKGatherUpdateTC, kKTableSample, kKUpdateWide, kKScoresWide, kKSampleWide, kKSweepWide, kNumKernelIds };

struct ProfRec {
  int id;
  cudaEvent_t a, b;
};

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// allow the largest dynamic shared memory the device grants this kernel (opt-in max minus its
// static shared memory); returns that size (0 on failure)
template <typename F>
size_t allow_max_dyn_smem(F* func) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, func) != cudaSuccess) return 0;
  const int mx = optin - (int)fa.sharedSizeBytes;
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess) return 0;
  return (size_t)mx;
}

// "first use on this device" for per-launcher one-time kernel attributes (function attributes are
// per device context: a second GPU in the same process needs them too)
struct DevOnce {
  std::atomic<uint64_t> mask{0};
  bool first(int dev) {
    const uint64_t bit = 1ull << (dev & 63);
    return !(mask.fetch_or(bit) & bit);
  }
};

}  // namespace

struct cp_sgd_s {
  // configuration
  int N = 0, R = 0, dtype = 0, sampler = 0, rule = 0;
  int device = 0;                // CUDA device of the handle (cp_sgd_sweep_multi checks it)
  int64_t dims[kMaxOrder] = {}, ldims[kMaxOrder] = {}, lstride[kMaxOrder] = {};
  int64_t lo_last = 0, hi_last = 0;
  int64_t B = 0;
  int32_t window[kMaxOrder][kMaxOrder] = {};  // [mode n][position]
  int64_t bmax[kMaxOrder] = {};               // rows per step for mode n
  double alpha = 0, eta = 0, bpar = 0, eps = 0;
  uint64_t seed = 0;
  cudaStream_t stream = nullptr;     // the caller's stream
  cudaStream_t ls = nullptr;         // stream kernels are launched on (== stream, or cap_stream while capturing)
  cudaStream_t cap_stream = nullptr; // private non-blocking stream used only for graph capture
  int world_rank = 0, world_size = 1;
  uint32_t flags = 0;
  const void* X = nullptr;
  void* factors[kMaxOrder] = {};
  void* fstage[kMaxOrder] = {};    // cp_sgd_steps_host staging of the host factors (fused / wide path)
  int* take_chg = nullptr;         // cp_sgd_steps_host (wide): per-mode "host factor differs" flags
  void* multi_params = nullptr;    // cp_sgd_sweep_multi: the chains' kernel parameters (device)
  size_t multi_cap = 0;
  size_t esz = 4;
  // layout
  void* Xmm[kMaxOrder] = {};
  int64_t pitch[kMaxOrder] = {};
  // per-mode tiling of k_gather
  int64_t In_local[kMaxOrder] = {}, row0[kMaxOrder] = {};
  int ntiles[kMaxOrder] = {}, nchunks[kMaxOrder] = {}, cgather[kMaxOrder] = {}, nparts[kMaxOrder] = {};
  int cu[kMaxOrder] = {};           // cluster size of k_update_table for mode n (0: legacy kernels)
  int64_t ut_rows[kMaxOrder] = {};  // rows per CTA of k_update_table
  size_t ut_smem[kMaxOrder] = {};
  int64_t TB[kMaxOrder] = {};
  // workspace (device)
  uint64_t* cdf[kMaxOrder] = {};
  double* pprob[kMaxOrder] = {};
  void* S[kMaxOrder] = {};
  uint64_t* Ttot = nullptr;
  int32_t* idx = nullptr;
  double* w = nullptr;
  int64_t* beff = nullptr;       // rows of the prefetched batch
  int64_t* beff_api = nullptr;   // rows of the last cp_sgd_sample call
  void* zrow = nullptr;          // prefetched unweighted SKR rows [Bmax][R]
  int64_t* fbase = nullptr;      // prefetched fiber offsets [Bmax]
  long long* dbg = nullptr;      // CPSGD_DEBUG_TIMERS: phase timestamps of k_update_table
  bool pdl = false;              // programmatic dependent launch in the wide path (CPSGD_PDL=1; measured
                                 // slower at C4: 272 vs 265 us/sweep, so off by default)
  int* last_mode_dev = nullptr;  // written by the fused sweep kernel
  void* zwp = nullptr;           // wide path: weighted padded SKR rows [Bmax][ceil8(R)] of the prefetched batch
  void* gam_next = nullptr;      // wide path: Gamma of the prefetched batch [R][R]
  int gu_ck[kMaxOrder] = {};     // wide path: batch chunks (CTAs per I-tile) of k_gather_update, 0 = not eligible
  int64_t gu_kb[kMaxOrder] = {};  // wide path: fibers per chunk
  void* Mpart = nullptr;         // wide path: split-K partial tiles [tiles][chunks][128][R]
  unsigned* gu_cnt = nullptr;    // wide path: per-tile arrival counters (unused)
  double* uw_gpart = nullptr;    // wide path: k_update_wide table partials [CTAs][R(R+1)/2]
  double* uw_rownorm = nullptr;  // wide path: Euclidean row norms [I_max]
  unsigned* uw_cnt = nullptr;    // wide path: k_update_wide CTA arrival counter
  double* tw_W = nullptr;        // wide path: W = swept Gram inverse [R][R] (or ||A||_F^2)
  int* tw_stat = nullptr;        // wide path: rank, bad bits of the table being built
  unsigned long long* sc_q = nullptr;  // wide path: quantised weights of the table being built [I_max]
  unsigned* sc_cnt = nullptr;    // wide path: k_update_wide score-phase CTA arrival counter
  unsigned* uw_flag = nullptr;   // wide path: W-ready epoch (monotonic)
  void* sw_gcl = nullptr;        // wide path: k_sample_wide cluster partials of Gamma
  bool use_tc = false;           // fp32 wide path on tcgen05 (k_gather_update_tc), else the FFMA mainloop
  float* zimg = nullptr;         // tcgen05 path: {zh; zl} A-operand images of the prefetched batch
  // persistent cooperative sweep kernel of the fp32 wide path (k_sweep_wide, sweep_wide.cuh)
  bool pw_ok = false;
  const int* pw_chg = nullptr;     // cp_sgd_steps_host's optimistic persistent launch: the take-over flags
  int pw_grid = 0;
  size_t pw_smem = 0;
  uint32_t pw_tag = 0;           // look-back tags: iteration s of a launch uses pw_tag + 1 + s
  float* pw_gcl = nullptr;       // [grid][R][R] per-CTA partials of Gamma
  double* pw_gram = nullptr;     // [R(R+1)/2]
  uint64_t* pw_qraw = nullptr;   // [I_max rounded to 16]: raw q rows of the table being rebuilt
  uint64_t* pw_coarse[kMaxOrder] = {};  // per mode [units]: coarse CDFs of the persistent kernel
  unsigned long long* pw_agg = nullptr;  // [row units]
  unsigned* pw_aggf = nullptr;   // [row units][2]
  unsigned* pw_bar = nullptr;    // [0] barrier arrivals, [32] pair-sum, [64] table-unit arrivals (zeroed per launch)
  double* pw_alphas = nullptr;   // per-iteration steps of one call (fixed rule schedules)
  int64_t pw_alphas_cap = 0;
  // cp_sgd_trace: the consumed batches of the persistent kernels
  unsigned char* trace_base = nullptr;
  int64_t trace_cap = 0, trace_count = 0;
  int fused_cu = 0, fused_bpc = 0, fused_rpc = 0;  // fused kernel geometry (0: not eligible)
  size_t fused_smem = 0;
  int pref_mode = -1;            // mode whose batch (at the current r) sits in idx/w/zrow/fbase
  uint64_t* iter_dev = nullptr;
  uint64_t* iter_tmp = nullptr;
  int* status_dev = nullptr;
  double* alpha_dev = nullptr;
  void* Mp = nullptr;
  void* Gp = nullptr;
  void* Msum = nullptr;
  void* Gsum = nullptr;
  void* Gout = nullptr;
  void* Gam_out = nullptr;
  void** fac_dev = nullptr;     // device copy of the factor pointer array (k_fit)
  int64_t* ldims_dev = nullptr;
  double* fit_partial = nullptr;
  int fit_blocks = 0;
  // host mirrors / pinned staging
  uint64_t iter_host = 0;
  int last_mode = -1;
  double* pinned = nullptr;  // small pinned staging buffer (alpha, iter)
  int sample_smem = 0;       // dynamic smem bytes of k_sample (0: read CDFs from global)
  // graph of one cyclic sweep (constant step)
  cudaGraphExec_t sweep_exec = nullptr;
  uint64_t sweep_launches = 0;
  int graph_end_pref = -1;
  // NCCL
  ncclComm_t comm = nullptr;
  // diagnostics
  std::string err;
  uint64_t launches = 0;
  bool prof = false;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  std::vector<int64_t> row_ranges;  // [2*world]: slab [lo, hi) of every rank
  void* Mred = nullptr;             // replicas / slab shards on the wide path: this rank's chunk sum of M, [tiles][R][128]
  int* one_dev = nullptr;           // a device 1 (table-only rebuild of the current factor)
  int* chg_host = nullptr;          // pinned: cp_sgd_steps_host's per-mode 'host factor differs' flags
  // CP_FLAG_P2P: this rank's symmetric exchange buffer (flags + 2 parity copies), the peers' buffers
  void* p2p_buf = nullptr;
  int64_t p2p_msz = 0;
  void* peer[kMaxStrata] = {};
  bool peers_set = false;
  std::vector<void*> peer_opened;   // IPC mappings to close
  unsigned long long* p2p_epoch = nullptr;
  unsigned* p2p_cnt = nullptr;      // [0] chunk-sum arrivals, [32] update arrivals
  int64_t strat_lo[kMaxStrata + 1] = {};  // CP_FLAG_STRATIFIED: slab bounds of the ranks (R26)

  cp_status fail(cp_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return st;
  }
};

namespace {

#define CUDA_TRY(h, expr)                                                                        \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess) return (h)->fail(CP_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

cp_status check_launch(cp_sgd_s* h, const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return h->fail(CP_ECUDA, "%s launch: %s", what, cudaGetErrorString(e));
  return CP_OK;
}

// profiling: event pair around one kernel of a direct-launch step
cudaEvent_t next_event(cp_sgd_s* h) {
  if (h->ev_next == h->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h->ev_pool.push_back(e);
  }
  return h->ev_pool[h->ev_next++];
}
struct ProfScope {
  cp_sgd_s* h;
  int id;
  cudaEvent_t b = nullptr;
  ProfScope(cp_sgd_s* h_, int id_) : h(h_), id(id_) {
    if (h->prof) {
      cudaEvent_t a = next_event(h);
      b = next_event(h);
      cudaEventRecord(a, h->ls);
      h->prof_recs.push_back(ProfRec{id, a, b});
    }
  }
  ~ProfScope() {
    if (h->prof) cudaEventRecord(b, h->ls);
  }
};

int rpt_for(int R) { return R <= 8 ? 4 : R <= 16 ? 8 : R <= 32 ? 16 : 32; }

// ---- kernel launchers ---------------------------------------------------------------------
template <typename T>
cp_status launch_table(cp_sgd_s* h, int k) {
  if (h->sampler == CP_UNIFORM) return CP_OK;  // q = 1, T = I_k: nothing depends on the factors
  ProfScope ps(h, kKTable);
  const int P = h->R * (h->R + 1) / 2;
  const int groups = std::max(1, kTableThreads / P);
  const size_t smem = sizeof(double) * (kMaxRank * kMaxRank + std::max(kTableThreads, P * groups));
  k_table<T><<<1, kTableThreads, smem, h->ls>>>((const T*)h->factors[k], h->dims[k], h->R, h->sampler,
                                                    h->pprob[k], h->cdf[k], h->Ttot + k, h->status_dev);
  h->launches++;
  return check_launch(h, "k_table");
}

cp_status launch_ut(cp_sgd_s* h, int n, int do_update, int do_table, int64_t row0, int64_t In, double alpha,
                    const double* alpha_dev, bool use_sum, int next_mode);
bool ut_fits(const cp_sgd_s* h, int64_t In);
bool wide_mode(const cp_sgd_s* h, int n);
bool multi(const cp_sgd_s* h);
bool sharded(const cp_sgd_s* h);
bool replica(const cp_sgd_s* h);

cp_status launch_table_any(cp_sgd_s* h, int k) {
  if (h->sampler == CP_UNIFORM) return CP_OK;
  if (ut_fits(h, h->dims[k])) return launch_ut(h, k, 0, 1, 0, h->dims[k], 0.0, nullptr, false, -1);
  return h->dtype == CP_F64 ? launch_table<double>(h, k) : launch_table<float>(h, k);
}

void fill_sample_params(cp_sgd_s* h, SampleParams& p, int n, const uint64_t* iter_ptr, uint64_t iter_add,
                        int32_t* idx, double* w, int64_t* beff, bool prefetch) {
  memset(&p, 0, sizeof p);
  p.N = h->N;
  p.n = n;
  p.R = h->R;
  p.strategy = h->sampler;
  p.B = h->B;
  for (int k = 0; k < h->N; ++k) {
    p.dims[k] = h->dims[k];
    p.cdf[k] = h->cdf[k];
    p.factors[k] = h->factors[k];
    p.ldims[k] = h->ldims[k];
    p.lstride[k] = h->lstride[k];
  }
  for (int q = 0; q < h->N - 1; ++q) p.window[q] = h->window[n][q];
  p.Ttot = h->Ttot;
  p.seed = h->seed;
  p.iter = iter_ptr;
  p.iter_add = iter_add;
  p.idx = idx;
  p.w = w;
  p.beff = beff;
  p.bmax = h->bmax[n];
  p.lo_last = h->lo_last;
  p.mode_major = h->Xmm[n] ? 1 : 0;
  p.pitch = h->pitch[n];
  if (h->flags & CP_FLAG_STRATIFIED) {  // R26: one stratum per rank's slab
    p.strat_P = h->world_size;
    for (int g = 0; g <= h->world_size; ++g) p.strat_lo[g] = h->strat_lo[g];
  }
  if (prefetch) {
    p.zrow = h->zrow;
    p.fbase = h->fbase;
    p.zimg = h->zimg;
  }
}

size_t sample_cdf_bytes(const cp_sgd_s* h, int n) {
  if (h->sampler == CP_UNIFORM) return 0;
  int64_t need = 0;
  for (int k = 0; k < h->N; ++k)
    if (k != n) need += h->dims[k];
  return (size_t)need * sizeof(uint64_t);
}

cp_status launch_sample(cp_sgd_s* h, int n, const uint64_t* iter_ptr, int32_t* idx, double* w, int64_t* beff,
                        bool prefetch) {
  ProfScope ps(h, kKSample);
  SampleParams p;
  fill_sample_params(h, p, n, iter_ptr, 0, idx, w, beff, prefetch);
  size_t smem = sample_cdf_bytes(h, n);
  p.stage_smem = (smem > 0 && smem <= (size_t)h->sample_smem) ? 1 : 0;
  if (!p.stage_smem) smem = 0;
  const int threads = 256;
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(h->bmax[n], threads), 148));
  if (h->dtype == CP_F64)
    k_sample<double><<<(unsigned)blocks, threads, smem, h->ls>>>(p);
  else
    k_sample<float><<<(unsigned)blocks, threads, smem, h->ls>>>(p);
  h->launches++;
  return check_launch(h, "k_sample");
}

template <typename T, int RPT>
cp_status launch_gather_t(cp_sgd_s* h, int n) {
  ProfScope ps(h, kKGather);
  GatherParams<T> p;
  memset(&p, 0, sizeof p);
  p.N = h->N;
  p.n = n;
  p.R = h->R;
  for (int k = 0; k < h->N; ++k) {
    p.ldims[k] = h->ldims[k];
    p.lstride[k] = h->lstride[k];
  }
  p.lo_last = h->lo_last;
  if (h->Xmm[n]) {
    p.X = (const T*)h->Xmm[n];
    p.mode_major = 1;
    p.pitch = h->pitch[n];
  } else {
    p.X = (const T*)h->X;
    p.mode_major = 0;
    p.pitch = 0;
  }
  p.fbase = h->fbase;
  p.zrow = (const T*)h->zrow;
  p.w = h->w;
  p.beff = h->beff;
  p.TB = h->TB[n];
  p.In_local = h->In_local[n];
  p.Mp = (T*)h->Mp;
  p.Gp = (T*)h->Gp;
  const size_t smem = gather_smem_bytes<T, RPT>(h->R);
  static DevOnce attr_once;  // per device: the attribute is per context
  if (attr_once.first(h->device)) {
    allow_max_dyn_smem(k_gather<T, RPT>);
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(h->ntiles[n], h->nchunks[n], 1);
  lc.blockDim = dim3(kGatherThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = h->ls;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = h->cgather[n];
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, k_gather<T, RPT>, p);
  h->launches++;
  if (e != cudaSuccess) return h->fail(CP_ECUDA, "k_gather launch: %s", cudaGetErrorString(e));
  return check_launch(h, "k_gather");
}

template <typename T>
cp_status launch_gather(cp_sgd_s* h, int n) {
  switch (rpt_for(h->R)) {
    case 4: return launch_gather_t<T, 4>(h, n);
    case 8: return launch_gather_t<T, 8>(h, n);
    case 16: return launch_gather_t<T, 16>(h, n);
    default: return launch_gather_t<T, 32>(h, n);
  }
}

// fused update + table (cluster kernel).  rows: [row0, row0 + In) of A^(n).
template <typename T>
cp_status launch_ut_t(cp_sgd_s* h, int n, int do_update, int do_table, int64_t row0, int64_t In, double alpha,
                      const double* alpha_dev, bool use_sum, int next_mode) {
  ProfScope ps(h, do_update ? kKUpdate : kKTable);
  UTParams<T> p;
  memset(&p, 0, sizeof p);
  p.R = h->R;
  p.strategy = h->sampler;
  p.rule = h->rule;
  p.do_update = do_update;
  p.do_table = do_table;
  p.In = In;
  int CU = 1;
  while (CU < 16 && CU * 32 < In) CU *= 2;
  p.rows_per = ceil_div(In, CU);
  p.nparts = h->nparts[n];
  p.Mp = (const T*)h->Mp;
  p.Gp = (const T*)h->Gp;
  p.Msum = use_sum ? (const T*)h->Msum : nullptr;
  p.Gsum = use_sum ? (const T*)h->Gsum : nullptr;
  p.A = (T*)h->factors[n] + row0 * h->R;
  p.S = h->S[n] ? (T*)h->S[n] + row0 * h->R : nullptr;
  p.Gout = (T*)h->Gout + row0 * h->R;
  p.Gam_out = (T*)h->Gam_out;
  p.alpha = alpha;
  p.alpha_dev = alpha_dev;
  p.eta = h->eta;
  p.b = h->bpar;
  p.eps = h->eps;
  p.iter = h->iter_dev;
  p.p_out = h->pprob[n];
  p.cdf = h->cdf[n];
  p.Tout = h->Ttot + n;
  p.status = h->status_dev;
  p.dbg = h->dbg;
  size_t smem = ut_smem_bytes(h->R, p.rows_per, sizeof(T));
  if (next_mode >= 0) {
    p.sample_next = 1;
    fill_sample_params(h, p.sp, next_mode, h->iter_dev, 0, h->idx, h->w, h->beff, true);
    const size_t cb = sample_cdf_bytes(h, next_mode);
    p.sp.stage_smem = (cb > 0 && smem + cb <= (size_t)h->sample_smem) ? 1 : 0;
    if (p.sp.stage_smem) smem += cb;
  }
  // one CTA per SM: the cluster's CTAs each run the serial table stages; co-residing CTAs would
  // share one SM's issue slots (claim more than half of the SM's shared memory)
  smem = std::max(smem, (size_t)h->sample_smem / 2 + 1024);
  static DevOnce attr_once;  // per device: the attribute is per context
  if (attr_once.first(h->device)) {
    const size_t mx = allow_max_dyn_smem(k_update_table<T>);
    cudaError_t eb = cudaFuncSetAttribute(k_update_table<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (mx == 0 || eb != cudaSuccess)
      return h->fail(CP_ECUDA, "k_update_table attributes: %s", cudaGetErrorString(eb));
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(CU, 1, 1);
  lc.blockDim = dim3(kUTThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = h->ls;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CU;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, k_update_table<T>, p);
  h->launches++;
  if (e != cudaSuccess)
    return h->fail(CP_ECUDA, "k_update_table launch (cluster %d, smem %zu B, params %zu B): %s", CU, smem,
                   sizeof(p), cudaGetErrorString(e));
  return check_launch(h, "k_update_table");
}

cp_status launch_ut(cp_sgd_s* h, int n, int do_update, int do_table, int64_t row0, int64_t In, double alpha,
                    const double* alpha_dev, bool use_sum, int next_mode) {
  return h->dtype == CP_F64
             ? launch_ut_t<double>(h, n, do_update, do_table, row0, In, alpha, alpha_dev, use_sum, next_mode)
             : launch_ut_t<float>(h, n, do_update, do_table, row0, In, alpha, alpha_dev, use_sum, next_mode);
}

bool ut_fits(const cp_sgd_s* h, int64_t In) {
  int CU = 1;
  while (CU < 16 && CU * 32 < In) CU *= 2;
  return ut_smem_bytes(h->R, ceil_div(In, CU), h->esz) <= (size_t)h->sample_smem;
}

template <typename T>
cp_status launch_update(cp_sgd_s* h, int n, double alpha, const double* alpha_dev, bool use_sum) {
  ProfScope ps(h, kKUpdate);
  UpdateParams<T> p;
  memset(&p, 0, sizeof p);
  p.R = h->R;
  p.In_local = h->In_local[n];
  p.row0 = h->row0[n];
  p.nchunks = h->nparts[n];
  p.Mp = (const T*)h->Mp;
  p.Gp = (const T*)h->Gp;
  p.Msum = use_sum ? (const T*)h->Msum : nullptr;
  p.Gsum = use_sum ? (const T*)h->Gsum : nullptr;
  p.A = (T*)h->factors[n];
  p.S = (T*)h->S[n];
  p.Gout = (T*)h->Gout;
  p.Gam_out = (T*)h->Gam_out;
  p.rule = h->rule;
  p.alpha = alpha;
  p.alpha_dev = alpha_dev;
  p.eta = h->eta;
  p.b = h->bpar;
  p.eps = h->eps;
  p.iter = h->iter_dev;
  const size_t smem = sizeof(T) * (h->R * h->R + kUR * (h->R + 1));
  const int64_t blocks = std::max<int64_t>(1, ceil_div(h->In_local[n], kUR));
  k_update<T><<<(unsigned)blocks, kUpdThreads, smem, h->ls>>>(p);
  h->launches++;
  return check_launch(h, "k_update");
}

template <typename T>
cp_status launch_reduce(cp_sgd_s* h, int n) {
  ProfScope ps(h, kKReduce);
  const int64_t tot = std::max<int64_t>((int64_t)h->R * h->In_local[n], (int64_t)h->R * h->R);
  k_reduce_partials<T><<<(unsigned)ceil_div(tot, 256), 256, 0, h->ls>>>(
      (const T*)h->Mp, (const T*)h->Gp, h->nparts[n], h->R, h->In_local[n], (T*)h->Msum, (T*)h->Gsum);
  h->launches++;
  return check_launch(h, "k_reduce_partials");
}

// several ranks (or one rank forced onto the multi-rank path with a 1-rank communicator: a test hook)
bool multi(const cp_sgd_s* h) { return h->world_size > 1 || (h->flags & CP_FLAG_FORCE_COMM); }
// slab sharding of the tensor along the last mode
bool sharded(const cp_sgd_s* h) { return multi(h) && !(h->flags & CP_FLAG_REPLICA); }
// whole-tensor replicas with a batch split of the wide path (CP_FLAG_REPLICA)
bool replica(const cp_sgd_s* h) { return multi(h) && (h->flags & CP_FLAG_REPLICA); }

// ---- wide single-GPU path: k_gather_update (gather + split-K + update) and the zw / Gamma epilogue ----
bool wide_mode(const cp_sgd_s* h, int n) { return n >= 0 && h->gu_ck[n] > 0; }

// the batch chunks this launch covers: all CK of them, or (replicas with a batch split) chunks rank, rank + P, ...
template <typename PP>
int gu_set_chunks(const cp_sgd_s* h, int n, PP& p) {
  p.CK = h->gu_ck[n];
  p.c_first = replica(h) ? h->world_rank : 0;
  p.c_step = replica(h) ? h->world_size : 1;
  return (int)ceil_div(p.CK - p.c_first, p.c_step);
}

// replicas: this rank's chunk partials summed in chunk order -> Mred [tiles][R][TI] (the exchange buffer)
template <typename T>
__global__ void k_chunk_sum(const T* __restrict__ Mpart, int CK, int c_first, int c_step, int R, int64_t tiles,
                            T* __restrict__ Mred) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)R * kGUTI;
  if (e >= tiles * per) return;
  const int64_t tile = e / per, o = e % per;
  T acc = T(0);
  for (int c = c_first; c < CK; c += c_step) acc += Mpart[(tile * CK + c) * per + o];
  Mred[e] = acc;
}

// replicas over peer memory (CP_FLAG_P2P, wide.cuh "replicas exchanging M over peer memory"): the chunk
// sum into this rank's symmetric buffer (parity of epoch e), published by the last CTA (ready = e)
template <typename T>
__global__ void k_chunk_sum_p2p(const T* __restrict__ Mpart, int CK, int c_first, int c_step, int R, int64_t tiles,
                                void* buf, int64_t msz, int npeer, const unsigned long long* epoch, unsigned* cnt) {
  __shared__ unsigned long long s_e;
  if (threadIdx.x == 0) {
    const unsigned long long e = *reinterpret_cast<const volatile unsigned long long*>(epoch) + 1;
    s_e = e;
    if (e > 2)  // this parity was published at e - 2: every reader must be done with it
      for (int r = 0; r < npeer; ++r)
        while (ld_acquire_sys_u64(p2p_done_flag(buf, r)) < e - 2) {
        }
  }
  __syncthreads();
  T* dst = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(buf) + kP2PHead) + (int64_t)(s_e & 1ull) * msz;
  const int64_t per = (int64_t)R * kGUTI;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tiles * per; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tile = e / per, o = e % per;
    T acc = T(0);
    for (int c = c_first; c < CK; c += c_step) acc += Mpart[(tile * CK + c) * per + o];
    dst[e] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(cnt, 1u) == gridDim.x - 1) {  // every CTA's part written: publish
      *cnt = 0;
      __threadfence_system();
      st_release_sys_u64(reinterpret_cast<unsigned long long*>(buf), s_e);
    }
  }
}

template <typename T, int CPT>
cp_status launch_gu_t(cp_sgd_s* h, int n, double alpha, const double* alpha_dev) {
  ProfScope ps(h, kKGatherUpdate);
  GUParams<T> p;
  memset(&p, 0, sizeof p);
  p.R = h->R;
  p.In = h->In_local[n];  // slab shards, last mode: the rank's rows
  if (h->Xmm[n]) {
    p.X = (const T*)h->Xmm[n];
    p.es = 1;
    p.vec = 1;
  } else {
    p.X = (const T*)h->X;
    p.es = h->lstride[n];
    p.vec = (n == 0 && (h->dims[0] * (int64_t)sizeof(T)) % 16 == 0) ? 1 : 0;
  }
  p.fbase = h->fbase;
  p.zwp = (const T*)h->zwp;
  p.bmax = h->bmax[n];
  const int CK = h->gu_ck[n];
  p.KB = h->gu_kb[n];
  p.Mpart = (T*)h->Mpart;
  p.cnt = h->gu_cnt;
  p.Gam = (const T*)h->gam_next;
  p.gcl = (decltype(p.gcl))h->sw_gcl;
  p.ncl = (int)ceil_div(ceil_div(h->bmax[n], kSWFibers), kSWCluster);
  p.gam_sum = (decltype(p.gam_sum))h->gam_next;
  p.A = (T*)h->factors[n];
  p.S = (T*)h->S[n];
  p.Gout = (T*)h->Gout;
  p.Gam_out = (T*)h->Gam_out;
  p.rule = h->rule;
  p.alpha = alpha;
  p.alpha_dev = alpha_dev;
  p.eta = h->eta;
  p.b = h->bpar;
  p.eps = h->eps;
  p.iter = h->iter_dev;
  const int ny = gu_set_chunks(h, n, p);
  const size_t smem = gu_smem_bytes<T, CPT>(p.KB);
  static DevOnce attr_once;  // per device: the attribute is per context
  if (attr_once.first(h->device)) {
    allow_max_dyn_smem(k_gather_update<T, CPT>);
    cudaFuncSetAttribute(k_gather_update<T, CPT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)ceil_div(h->In_local[n], kGUTI), (unsigned)ny, 1);
  lc.blockDim = dim3(kGUThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = h->ls;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, k_gather_update<T, CPT>, p);
  h->launches++;
  if (e != cudaSuccess) return h->fail(CP_ECUDA, "k_gather_update launch: %s", cudaGetErrorString(e));
  return check_launch(h, "k_gather_update");
}

cp_status launch_gu_tc(cp_sgd_s* h, int n, double alpha, const double* alpha_dev) {
  ProfScope ps(h, kKGatherUpdateTC);
  GUParams<float> p;
  memset(&p, 0, sizeof p);
  p.R = h->R;
  p.In = h->In_local[n];  // slab shards, last mode: the rank's rows
  p.X = h->Xmm[n] ? (const float*)h->Xmm[n] : (const float*)h->X;
  p.es = 1;
  p.vec = 1;
  p.rowlen = h->Xmm[n] ? h->pitch[n] : h->dims[n];
  p.fbase = h->fbase;
  p.zwp = (const float*)h->zwp;
  p.zimg = h->zimg;
  p.bmax = h->bmax[n];
  const int CK = h->gu_ck[n];
  p.KB = h->gu_kb[n];
  p.Mpart = (float*)h->Mpart;
  p.cnt = h->gu_cnt;
  p.Gam = (const float*)h->gam_next;
  p.gcl = (decltype(p.gcl))h->sw_gcl;
  p.ncl = (int)ceil_div(ceil_div(h->bmax[n], kSWFibers), kSWCluster);
  p.gam_sum = (decltype(p.gam_sum))h->gam_next;
  p.A = (float*)h->factors[n];
  p.S = (float*)h->S[n];
  p.Gout = (float*)h->Gout;
  p.Gam_out = (float*)h->Gam_out;
  p.rule = h->rule;
  p.alpha = alpha;
  p.alpha_dev = alpha_dev;
  p.eta = h->eta;
  p.b = h->bpar;
  p.eps = h->eps;
  p.iter = h->iter_dev;
  p.dbg = h->dbg;
  const int ny = gu_set_chunks(h, n, p);
  const size_t smem = tc_smem_bytes(p.KB);
  static DevOnce attr_once;  // per device: the attribute is per context
  if (attr_once.first(h->device)) {
    allow_max_dyn_smem(k_gather_update_tc<0>);
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)ceil_div(h->In_local[n], kGUTI), (unsigned)ny, 1);
  lc.blockDim = dim3(kTCThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = h->ls;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, k_gather_update_tc<0>, p);
  h->launches++;
  if (e != cudaSuccess)
    return h->fail(CP_ECUDA, "k_gather_update_tc launch (chunks %d, smem %zu): %s", CK, smem, cudaGetErrorString(e));
  return check_launch(h, "k_gather_update_tc");
}

template <typename T>
cp_status launch_gu(cp_sgd_s* h, int n, double alpha, const double* alpha_dev) {
  // tensor-core mainloop needs fiber-contiguous, 16-byte aligned fibers (mode-major copy, or mode 0)
  const bool tc_ok = sizeof(T) == 4 && h->use_tc && (h->Xmm[n] || (n == 0 && h->dims[0] % 4 == 0));
  if (tc_ok) return launch_gu_tc(h, n, alpha, alpha_dev);
  switch ((h->R + 7) / 8) {
    case 1: return launch_gu_t<T, 1>(h, n, alpha, alpha_dev);
    case 2: return launch_gu_t<T, 2>(h, n, alpha, alpha_dev);
    case 3: return launch_gu_t<T, 3>(h, n, alpha, alpha_dev);
    case 4: return launch_gu_t<T, 4>(h, n, alpha, alpha_dev);
    case 5: return launch_gu_t<T, 5>(h, n, alpha, alpha_dev);
    case 6: return launch_gu_t<T, 6>(h, n, alpha, alpha_dev);
    case 7: return launch_gu_t<T, 7>(h, n, alpha, alpha_dev);
    default: return launch_gu_t<T, 8>(h, n, alpha, alpha_dev);
  }
}

int64_t ts_cdf_elems(const cp_sgd_s* h, int next_mode) {
  if (next_mode < 0 || h->sampler == CP_UNIFORM) return 0;
  int64_t c = 0;
  for (int k = 0; k < h->N; ++k)
    if (k != next_mode) c += h->dims[k];
  return c;
}

// ---- wide path: k_update_wide (+ the Gram inverse in its last cluster, the scores, the scan) -> k_sample_wide (wide.cuh) ----
// k_update_wide's CTAs wait for one another (the Gram inverse of its last cluster): every cluster
// of the grid must be resident at once.  True when the occupancy calculator says so for the
// launch's configuration (clusters of kUWCluster, its dynamic shared memory).
template <typename T>
bool uw_coresident(int R, int64_t In) {
  const int64_t ncl = ceil_div(ceil_div(In, kUWRows), kUWCluster);
  const size_t smem = uw_smem_bytes(R, sizeof(T), std::min<int64_t>(In, 4096));
  if (cudaFuncSetAttribute(k_update_wide<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return false;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(ncl * kUWCluster), 1, 1);
  lc.blockDim = dim3(kWThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kUWCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  int act = 0;
  const cudaError_t eo = cudaOccupancyMaxActiveClusters(&act, k_update_wide<T>, &lc);
  // leave the attribute at the opt-in maximum: launches of other handles / modes (larger R or
  // I_n) need more than this mode's size, and the launcher sets it only once per device
  allow_max_dyn_smem(k_update_wide<T>);
  if (eo != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (int64_t)act >= ncl;
}

template <typename T>
cp_status launch_uw_t(cp_sgd_s* h, int n, double alpha, const double* alpha_dev, const int* take_chg = nullptr,
                      bool from_self = false) {
  ProfScope ps(h, kKUpdateWide);
  UWParams<T> p;
  memset(&p, 0, sizeof p);
  p.R = h->R;
  p.strategy = h->sampler;
  p.rule = h->rule;
  // slab shards, last mode: the update of the rank's rows only (the table follows the row exchange: phase 2)
  const bool own_rows = sharded(h) && n == h->N - 1 && !take_chg;
  const int64_t r0 = own_rows ? h->row0[n] : 0;
  p.In = own_rows ? h->In_local[n] : h->dims[n];
  const bool red = replica(h) || (sharded(h) && n < h->N - 1);  // the rank-summed M, one "chunk"
  p.Mpart = (const T*)(red ? h->Mred : h->Mpart);
  p.CK = red ? 1 : h->gu_ck[n];
  p.update_only = own_rows ? 1 : 0;
  if (replica(h) && (h->flags & CP_FLAG_P2P) && !take_chg) {  // M summed from the peers' buffers
    p.npeer = h->world_size;
    p.rank = h->world_rank;
    for (int g = 0; g < h->world_size; ++g) p.peer[g] = h->peer[g];
    p.p2p_msz = h->p2p_msz;
    p.p2p_epoch = h->p2p_epoch;
    p.p2p_cnt = h->p2p_cnt + 32;
  }
  p.Gam = (const T*)h->gam_next;
  p.A = (T*)h->factors[n] + r0 * h->R;
  p.S = h->S[n] ? (T*)h->S[n] + r0 * h->R : nullptr;
  p.Gout = (T*)h->Gout + r0 * h->R;
  p.Gam_out = (T*)h->Gam_out;
  p.alpha = alpha;
  p.alpha_dev = alpha_dev;
  p.eta = h->eta;
  p.b = h->bpar;
  p.eps = h->eps;
  p.gpart = h->uw_gpart;
  p.rownorm = h->uw_rownorm;
  p.W = h->tw_W;
  p.tstat = h->tw_stat;
  p.cnt = h->uw_cnt;
  p.flag = h->uw_flag;
  p.cnt2 = h->sc_cnt;
  p.qbuf = h->sc_q;
  p.p_out = h->pprob[n];
  p.cdf = h->cdf[n];
  p.Tout = h->Ttot + n;
  p.status = h->status_dev;
  p.qch = std::min<int64_t>(h->dims[n], 4096);
  p.table_only = take_chg ? 1 : 0;  // cp_sgd_steps_host: take over the staged factor, rebuild its table
  p.fstage = from_self ? (const T*)h->factors[n] : (const T*)h->fstage[n];  // from_self: the factor as it is
  p.chg = take_chg;
  p.dbg = h->dbg;
  const size_t smem = uw_smem_bytes(h->R, sizeof(T), p.qch);
  static DevOnce attr_once;  // per device: the attribute is per context
  if (attr_once.first(h->device)) {
    allow_max_dyn_smem(k_update_wide<T>);
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)(ceil_div(ceil_div(p.In, kUWRows), kUWCluster) * kUWCluster), 1, 1);
  lc.blockDim = dim3(kWThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = h->ls;
  cudaLaunchAttribute at[3];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kUWCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  // every CTA waits for the Gram inverse of the last cluster: a cooperative launch, so the runtime
  // guarantees co-residency (or refuses the launch) even with other work on the device (init also
  // checked the occupancy: uw_coresident); CPSGD_PW_NONCOOP=1 drops the attribute for profilers that
  // cannot replay cooperative launches
  at[2].id = cudaLaunchAttributeCooperative;
  at[2].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = getenv("CPSGD_PW_NONCOOP") ? 2 : 3;
  cudaError_t e = cudaLaunchKernelEx(&lc, k_update_wide<T>, p);
  h->launches++;
  if (e != cudaSuccess) return h->fail(CP_ECUDA, "k_update_wide launch: %s", cudaGetErrorString(e));
  return check_launch(h, "k_update_wide");
}

template <typename T>
cp_status launch_sw_t(cp_sgd_s* h, int n) {
  ProfScope ps(h, kKSampleWide);
  SWParams p;
  memset(&p, 0, sizeof p);
  fill_sample_params(h, p.sp, n, h->iter_dev, 0, h->idx, h->w, h->beff, true);
  p.sp.zwp = h->zwp;
  p.sp.gam_next = h->gam_next;
  p.gcl = h->sw_gcl;
  p.dbg = h->dbg;
  p.cdf_elems = ts_cdf_elems(h, n);
  const size_t smem = sw_smem_bytes(h->N, h->R, p.cdf_elems, sizeof(T));
  static DevOnce attr_once;  // per device: the attribute is per context
  if (attr_once.first(h->device)) {
    allow_max_dyn_smem(k_sample_wide<T>);
  }
  const int64_t ctas = ceil_div(ceil_div(h->bmax[n], kSWFibers), kSWCluster) * kSWCluster;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)ctas, 1, 1);
  lc.blockDim = dim3(kWThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = h->ls;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kSWCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = h->pdl ? 1 : 0;
  lc.attrs = at;
  lc.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&lc, k_sample_wide<T>, p);
  h->launches++;
  if (e != cudaSuccess) return h->fail(CP_ECUDA, "k_sample_wide launch (smem %zu): %s", smem, cudaGetErrorString(e));
  return check_launch(h, "k_sample_wide");
}

// the batch of mode n at the current r into the prefetch buffers (k_sample [+ k_zw_gamma])
cp_status launch_prefetch(cp_sgd_s* h, int n) {
  if (wide_mode(h, n)) return h->dtype == CP_F64 ? launch_sw_t<double>(h, n) : launch_sw_t<float>(h, n);
  return launch_sample(h, n, h->iter_dev, h->idx, h->w, h->beff, true);
}

TraceParams trace_params(cp_sgd_s* h, int nsteps);

// ---- persistent single-cluster sweep kernel (fused.cuh) ----------------------------------------
template <typename T>
void fill_fused_params(cp_sgd_s* h, FusedParams<T>& p, int nsteps, int first_mode, int order, double alpha,
                       const double* alpha_dev, int rebuild) {
  memset(&p, 0, sizeof p);
  p.N = h->N;
  p.R = h->R;
  p.strategy = h->sampler;
  p.rule = h->rule;
  p.CU = h->fused_cu;
  for (int k = 0; k < h->N; ++k) {
    p.dims[k] = h->dims[k];
    p.stride[k] = h->lstride[k];
    if (h->Xmm[k]) {
      p.Xg[k] = (const T*)h->Xmm[k];
      p.estride[k] = 1;
      p.pitch[k] = h->pitch[k];
    } else {
      p.Xg[k] = (const T*)h->X;
      p.estride[k] = h->lstride[k];
      p.pitch[k] = 0;
    }
    p.factors[k] = (T*)h->factors[k];
    p.S[k] = (T*)h->S[k];
    p.cdf[k] = h->cdf[k];
    p.pprob[k] = h->pprob[k];
    p.bmax[k] = h->bmax[k];
    for (int j = 0; j < h->N - 1; ++j) p.window[k][j] = h->window[k][j];
  }
  p.Ttot = h->Ttot;
  p.status = h->status_dev;
  p.iter = h->iter_dev;
  p.seed = h->seed;
  p.B = h->B;
  p.alpha = alpha;
  p.alpha_dev = alpha_dev;
  p.eta = h->eta;
  p.b = h->bpar;
  p.eps = h->eps;
  p.nsteps = nsteps;
  p.first_mode = first_mode;
  p.order = order;
  p.rebuild = rebuild;
  for (int k = 0; k < h->N; ++k) p.fstage[k] = (const T*)h->fstage[k];
  p.Gout = (T*)h->Gout;
  p.Gam_out = (T*)h->Gam_out;
  p.last_mode = h->last_mode_dev;
  p.BPC = h->fused_bpc;
  p.RPC = h->fused_rpc;
  int64_t imax = 0;
  for (int k = 0; k < h->N; ++k) imax = std::max(imax, h->dims[k]);
  p.Imax = imax;
  p.tr = trace_params(h, nsteps);
  p.dbg = h->dbg;
}

template <typename T, int ROWS>
cp_status launch_fused_t(cp_sgd_s* h, int nsteps, int first_mode, int order, double alpha, const double* alpha_dev,
                         int rebuild) {
  ProfScope ps(h, kKFused);
  FusedParams<T> p;
  fill_fused_params<T>(h, p, nsteps, first_mode, order, alpha, alpha_dev, rebuild);
  static DevOnce attr_once;  // per device: the attribute is per context
  if (attr_once.first(h->device)) {
    allow_max_dyn_smem(fused_k<T, ROWS>());
    cudaFuncSetAttribute(fused_k<T, ROWS>(), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(h->fused_cu, 1, 1);
  lc.blockDim = dim3(kFThreads, 1, 1);
  lc.dynamicSmemBytes = h->fused_smem;
  lc.stream = h->ls;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = h->fused_cu;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, fused_k<T, ROWS>(), p);
  h->launches++;
  if (e != cudaSuccess)
    return h->fail(CP_ECUDA, "k_sweep_fused launch (cluster %d, smem %zu): %s", h->fused_cu, h->fused_smem,
                   cudaGetErrorString(e));
  return check_launch(h, "k_sweep_fused");
}

template <typename T>
cp_status launch_fused_r(cp_sgd_s* h, int nsteps, int first_mode, int order, double alpha, const double* alpha_dev,
                         int rebuild) {
  int64_t imax = 0;
  for (int k = 0; k < h->N; ++k) imax = std::max(imax, h->dims[k]);
  return imax > kFThreads ? launch_fused_t<T, 2>(h, nsteps, first_mode, order, alpha, alpha_dev, rebuild)
                          : launch_fused_t<T, 1>(h, nsteps, first_mode, order, alpha, alpha_dev, rebuild);
}

cp_status launch_fused(cp_sgd_s* h, int nsteps, int first_mode, int order, double alpha, const double* alpha_dev,
                       int rebuild = 0) {
  cp_status st = h->dtype == CP_F64 ? launch_fused_r<double>(h, nsteps, first_mode, order, alpha, alpha_dev, rebuild)
                                    : launch_fused_r<float>(h, nsteps, first_mode, order, alpha, alpha_dev, rebuild);
  h->pref_mode = -1;
  return st;
}

// many independent chains in one launch: cluster c runs nsteps cyclic iterations of
// handle hs[c] (same geometry for all: dtype, dims, R, fused plan; samplers, rules, seeds may differ)
template <typename T, int ROWS>
cp_status launch_fused_multi_t(cp_sgd_s* const* hs, int nh, int nsteps) {
  cp_sgd_s* h0 = hs[0];
  ProfScope ps(h0, kKFused);
  std::vector<FusedParams<T>> prm(nh);
  for (int i = 0; i < nh; ++i) fill_fused_params<T>(hs[i], prm[i], nsteps, 0, CP_ORDER_CYCLIC, hs[i]->alpha, nullptr, 0);
  const size_t bytes = sizeof(FusedParams<T>) * (size_t)nh;
  if (h0->multi_cap < bytes) {
    cudaFree(h0->multi_params);
    h0->multi_params = nullptr;
    h0->multi_cap = 0;
    CUDA_TRY(h0, cudaMalloc(&h0->multi_params, bytes));
    h0->multi_cap = bytes;
  }
  for (int i = 1; i < nh; ++i) CUDA_TRY(h0, cudaStreamSynchronize(hs[i]->stream));  // their earlier work first
  CUDA_TRY(h0, cudaMemcpyAsync(h0->multi_params, prm.data(), bytes, cudaMemcpyHostToDevice, h0->stream));
  static DevOnce attr_once;  // per device: the attribute is per context
  if (attr_once.first(h0->device)) {
    allow_max_dyn_smem(fused_multi_k<T, ROWS>());
    cudaFuncSetAttribute(fused_multi_k<T, ROWS>(), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  cudaLaunchConfig_t lc = {};
  size_t smem = 0;  // each cluster lays out its own shared memory (the CDF area depends on the sampler)
  for (int i = 0; i < nh; ++i) smem = std::max(smem, (size_t)hs[i]->fused_smem);
  lc.gridDim = dim3((unsigned)(nh * h0->fused_cu), 1, 1);
  lc.blockDim = dim3(kFThreads, 1, 1);
  lc.dynamicSmemBytes = smem;
  lc.stream = h0->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = h0->fused_cu;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&lc, fused_multi_k<T, ROWS>(), (const FusedParams<T>*)h0->multi_params,
                                     h0->fused_cu);
  h0->launches++;
  if (e != cudaSuccess) return h0->fail(CP_ECUDA, "k_sweep_fused_multi launch (%d chains): %s", nh, cudaGetErrorString(e));
  cp_status st = check_launch(h0, "k_sweep_fused_multi");
  if (st) return st;
  cudaEvent_t ev;  // the other handles' later work after this launch
  CUDA_TRY(h0, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_TRY(h0, cudaEventRecord(ev, h0->stream));
  for (int i = 1; i < nh; ++i) CUDA_TRY(h0, cudaStreamWaitEvent(hs[i]->stream, ev, 0));
  cudaEventDestroy(ev);
  for (int i = 0; i < nh; ++i) {
    hs[i]->iter_host += nsteps;
    hs[i]->last_mode = hs[i]->N - 1;
    hs[i]->pref_mode = -1;
  }
  return CP_OK;
}

// geometry + eligibility of the fused kernel: one GPU, R <= 32, I_n <= 512, fits shared memory
void plan_fused(cp_sgd_s* h) {
  h->fused_cu = 0;
  if (multi(h) || (h->flags & CP_FLAG_NO_FUSED)) return;
  if (fused_rp(h->R, h->esz) / (h->esz == 8 ? 2 : 4) > 8) return;  // gather_contract supports <= 8 vector groups
  int64_t imax = 0, bmx = 0, cdfmax = 0;  // cdfmax: the resident CDFs of every mode
  for (int n = 0; n < h->N; ++n) {
    imax = std::max(imax, h->dims[n]);
    bmx = std::max(bmx, h->bmax[n]);
    cdfmax += h->dims[n];
  }
  if (imax > 2 * kFThreads) return;
  const int CU = (h->flags & CP_FLAG_FUSED_CU8) ? 8 : 16;
  const int bpc = (int)ceil_div(bmx, CU);
  const int rpc = (int)ceil_div(imax, CU);
  if (bpc > 256 || rpc > kFThreads) return;
  const FusedLayout L = fused_layout(h->N, h->R, bpc, rpc, imax, h->sampler == CP_UNIFORM ? 0 : cdfmax, h->esz);
  if (L.total + 2048 > (size_t)h->sample_smem) return;
  h->fused_cu = CU;
  h->fused_bpc = bpc;
  h->fused_rpc = rpc;
  h->fused_smem = L.total;
}

// ---- cp_sgd_trace record layout ------------------------------------------------------------------
struct TraceLayout {
  int64_t stride, o_idx, o_w, o_A, o_S, o_cdf, o_meta;
};
TraceLayout trace_layout(const cp_sgd_s* h) {
  int64_t bm = 0, im = 0;
  for (int k = 0; k < h->N; ++k) {
    bm = std::max(bm, h->bmax[k]);
    im = std::max(im, h->dims[k]);
  }
  TraceLayout L;
  int64_t off = 0;
  auto take = [&](int64_t bytes) {
    off = (off + 15) / 16 * 16;
    const int64_t at = off;
    off += bytes;
    return at;
  };
  L.o_idx = take(4 * bm * (h->N - 1));
  L.o_w = take(8 * bm);
  L.o_A = take((int64_t)h->esz * im * h->R);
  L.o_S = take((int64_t)h->esz * im * h->R);
  L.o_cdf = take(8 * im);
  L.o_meta = take(8 * 4);
  L.stride = (off + 255) / 256 * 256;
  return L;
}
TraceParams trace_params(cp_sgd_s* h, int nsteps) {
  TraceParams t;
  memset(&t, 0, sizeof t);
  if (!h->trace_base) return t;
  const TraceLayout L = trace_layout(h);
  t.base = h->trace_base;
  t.stride = L.stride;
  t.o_idx = L.o_idx;
  t.o_w = L.o_w;
  t.o_A = L.o_A;
  t.o_S = L.o_S;
  t.o_cdf = L.o_cdf;
  t.o_meta = L.o_meta;
  t.first = h->trace_count;
  t.cap = h->trace_cap;
  h->trace_count = std::min<int64_t>(h->trace_cap, h->trace_count + nsteps);
  return t;
}

// ---- persistent cooperative sweep kernel of the fp32 wide path (sweep_wide.cuh) -------------------
// row units of the largest mode (the stride of the persistent kernel's unit-fastest pair partials)
int64_t units_max_of(const cp_sgd_s* h) {
  int64_t u = 1;
  for (int k = 0; k < h->N; ++k) u = std::max<int64_t>(u, pw_units_rows(h->dims[k]));
  return u;
}
// pw_kernel(R): k_pw.cu (its own translation unit)

// SMs one handle's persistent / wide launches are planned for: the B200's 148, or CPSGD_SMS (read at init) so that
// several handles can run their cooperative launches side by side on disjoint SMs (independent chains)
int sm_budget() {
  const char* e = getenv("CPSGD_SMS");
  const int v = e ? atoi(e) : 148;
  return v >= 8 && v <= 148 ? v : 148;
}

// eligible: one GPU, fp32 on the tcgen05 gather for every mode, gradient rules (the sampled-ALS rule
// stays on the kernel chain), cooperative launch supported, one 448-thread CTA per SM co-resident
bool plan_pw(cp_sgd_s* h) {
  h->pw_ok = false;
  if (multi(h) || h->dtype != CP_F32 || !h->use_tc || h->rule == CP_STEP_ALS ||
      (h->flags & CP_FLAG_NO_PERSIST))
    return true;
  int64_t kbmax = 0, cdfmax = 0, units = 0;
  for (int n = 0; n < h->N; ++n) {
    if (!wide_mode(h, n)) return true;
    if (!(h->Xmm[n] || (n == 0 && h->dims[0] % 4 == 0))) return true;
    kbmax = std::max(kbmax, h->gu_kb[n]);
    cdfmax = std::max(cdfmax, ts_cdf_elems(h, n));
    units = std::max<int64_t>(units, pw_units_rows(h->dims[n]));
  }
  int coop = 0, sms = 0, optin = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
  if (!coop || sms < 1) return true;
  const size_t smem = pw_smem_bytes(h->N, h->R, kbmax, cdfmax);
  if (smem + 1024 > (size_t)optin) return true;
  allow_max_dyn_smem(pw_kernel(h->R));
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pw_kernel(h->R), kPWThreads, smem) != cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return true;
  }
  h->pw_grid = std::min(sms, sm_budget());  // one CTA per SM (of the handle's SM budget)
  h->pw_smem = smem;
  const int P = h->R * (h->R + 1) / 2;
  auto alloc = [&](void** ptr, size_t bytes) {
    if (cudaMalloc(ptr, bytes) != cudaSuccess) return false;
    cudaMemsetAsync(*ptr, 0, bytes, h->stream);
    return true;
  };
  if (!alloc((void**)&h->pw_gcl, sizeof(float) * (size_t)h->pw_grid * h->R * h->R) ||
      !alloc((void**)&h->pw_gram, sizeof(double) * ((P + 1) & ~1)) ||  // even: whole 16-byte bulk copies
      !alloc((void**)&h->pw_qraw, sizeof(uint64_t) * (size_t)(units_max_of(h) * kPWRows)) ||
      !alloc((void**)&h->pw_coarse[0], sizeof(uint64_t) * (size_t)(units_max_of(h) * h->N)) ||
      !alloc((void**)&h->pw_agg, sizeof(unsigned long long) * units) ||
      !alloc((void**)&h->pw_aggf, sizeof(unsigned) * 2 * units) ||
      !alloc((void**)&h->pw_bar, sizeof(unsigned) * 128)) {
    cudaGetLastError();
    return false;
  }
  h->pw_ok = true;
  return true;
}

cp_status launch_pw(cp_sgd_s* h, int nsteps, int first_mode, int order, double alpha, const double* alpha_dev,
                    const double* alphas_dev) {
  ProfScope ps(h, kKSweepWide);
  PWParams p;
  memset(&p, 0, sizeof p);
  p.N = h->N;
  p.R = h->R;
  p.strategy = h->sampler;
  p.rule = h->rule;
  p.nsteps = nsteps;
  p.first_mode = first_mode;
  p.order = order;
  p.B = h->B;
  for (int k = 0; k < h->N; ++k) {
    p.dims[k] = h->dims[k];
    p.lstride[k] = h->lstride[k];
    p.Xg[k] = h->Xmm[k] ? (const float*)h->Xmm[k] : (const float*)h->X;
    p.rowlen[k] = h->Xmm[k] ? h->pitch[k] : h->dims[k];
    p.pitch[k] = h->Xmm[k] ? h->pitch[k] : 0;
    p.factors[k] = (float*)h->factors[k];
    p.S[k] = (float*)h->S[k];
    p.cdf[k] = h->cdf[k];
    p.pprob[k] = h->pprob[k];
    for (int j = 0; j < h->N - 1; ++j) p.window[k][j] = h->window[k][j];
    p.bmax[k] = h->bmax[k];
    p.CK[k] = h->gu_ck[k];
    p.KB[k] = h->gu_kb[k];
  }
  p.Ttot = h->Ttot;
  p.seed = h->seed;
  p.iter = h->iter_dev;
  p.status = h->status_dev;
  p.last_mode = h->last_mode_dev;
  p.alpha = alpha;
  p.alpha_dev = alpha_dev;
  p.alphas = alphas_dev;
  p.eta = h->eta;
  p.b = h->bpar;
  p.eps = h->eps;
  p.idx = h->idx;
  p.w = h->w;
  p.fbase = h->fbase;
  p.beff = h->beff;
  p.zimg = h->zimg;
  p.gcl = h->pw_gcl;
  p.gam = (float*)h->gam_next;
  p.Mpart = (float*)h->Mpart;
  p.gpart = h->uw_gpart;
  p.gram = h->pw_gram;
  p.rownorm = h->uw_rownorm;
  p.agg = h->pw_agg;
  p.aggf = h->pw_aggf;
  p.bar = h->pw_bar;
  p.pcnt = h->pw_bar + 32;  // another 128-byte line
  p.qcnt = h->pw_bar + 64;  // another 128-byte line
  p.qraw = h->pw_qraw;
  for (int k = 0; k < h->N; ++k) p.coarse[k] = h->pw_coarse[0] + (size_t)k * units_max_of(h);
  p.gstride = units_max_of(h);
  p.tag0 = h->pw_tag + 1;
  p.Gout = (float*)h->Gout;
  p.Gam_out = (float*)h->Gam_out;
  p.tr = trace_params(h, nsteps);
  p.dbg = h->dbg;
  p.chg = h->pw_chg;
  p.ablate = getenv("CPSGD_PW_ABLATE_MASK") ? (unsigned)strtoul(getenv("CPSGD_PW_ABLATE_MASK"), nullptr, 0) : 0u;
  h->pw_tag += (uint32_t)nsteps;
  static DevOnce attr_once[4];
  if (attr_once[h->R <= 16 ? 0 : h->R <= 32 ? 1 : h->R <= 56 ? 2 : 3].first(h->device)) allow_max_dyn_smem(pw_kernel(h->R));
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)h->pw_grid, 1, 1);
  lc.blockDim = dim3(kPWThreads, 1, 1);
  lc.dynamicSmemBytes = h->pw_smem;
  lc.stream = h->ls;
  cudaLaunchAttribute at[1];
  // every CTA waits for the others (grid barriers, look-back): the launch must be co-resident
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  lc.attrs = at;
  lc.numAttrs = getenv("CPSGD_PW_NONCOOP") ? 0 : 1;  // profilers that cannot replay cooperative launches
  CUDA_TRY(h, cudaMemsetAsync(h->pw_bar, 0, sizeof(unsigned) * 128, h->ls));
  cudaError_t e = getenv("CPSGD_PW_FORCE_FALLBACK") ? cudaErrorCooperativeLaunchTooLarge
                                                    : cudaLaunchKernelEx(&lc, pw_kernel(h->R), p);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    // the grid cannot be co-resident right now (other work holds SMs, e.g. another process under MPS): this and
    // every later call of the handle run the same steps on the kernel chain instead (cp_sgd_path reports it)
    cudaGetLastError();
    h->pw_ok = false;
    h->pw_tag -= (uint32_t)nsteps;
    return CP_OK;
  }
  h->launches++;
  h->pref_mode = -1;
  if (e != cudaSuccess)
    return h->fail(CP_ECUDA, "k_sweep_wide launch (grid %d, smem %zu): %s", h->pw_grid, h->pw_smem, cudaGetErrorString(e));
  return check_launch(h, "k_sweep_wide");
}

// ---- one step, by phases ------------------------------------------------------------------------
cp_status phase0(cp_sgd_s* h, int n, double alpha, const double* alpha_dev) {
  cp_status st = CP_OK;
  if (h->pref_mode != n) {  // no prefetched batch for this mode: sample it now
    st = launch_prefetch(h, n);
    if (st) return st;
    h->pref_mode = n;
  }
  if (wide_mode(h, n)) {  // gather + contraction + split-K partials (replicas: this rank's chunks)
    st = h->dtype == CP_F64 ? launch_gu<double>(h, n, alpha, alpha_dev) : launch_gu<float>(h, n, alpha, alpha_dev);
    h->pref_mode = -1;
    if (!st && replica(h) && (h->flags & CP_FLAG_P2P)) {  // -> this rank's symmetric buffer, published
      if (!h->peers_set) return h->fail(CP_ESTATE, "CP_FLAG_P2P: the peers' buffers were not set (cp_sgd_p2p_peers)");
      const int64_t tiles = ceil_div(h->dims[n], kGUTI), tot = tiles * h->R * kGUTI;
      const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(tot, 256), 296);
      if (h->dtype == CP_F64)
        k_chunk_sum_p2p<double><<<blocks, 256, 0, h->ls>>>((const double*)h->Mpart, h->gu_ck[n], h->world_rank,
                                                           h->world_size, h->R, tiles, h->p2p_buf, h->p2p_msz,
                                                           h->world_size, h->p2p_epoch, h->p2p_cnt);
      else
        k_chunk_sum_p2p<float><<<blocks, 256, 0, h->ls>>>((const float*)h->Mpart, h->gu_ck[n], h->world_rank,
                                                          h->world_size, h->R, tiles, h->p2p_buf, h->p2p_msz,
                                                          h->world_size, h->p2p_epoch, h->p2p_cnt);
      h->launches++;
      return check_launch(h, "k_chunk_sum_p2p");
    }
    if (!st && (replica(h) || (sharded(h) && n < h->N - 1))) {  // -> Mred, summed over ranks before phase 1
      const int64_t tiles = ceil_div(h->dims[n], kGUTI), tot = tiles * h->R * kGUTI;
      const int CK = h->gu_ck[n];
      const int c0 = replica(h) ? h->world_rank : 0, cs = replica(h) ? h->world_size : 1;
      if (h->dtype == CP_F64)
        k_chunk_sum<double><<<(unsigned)ceil_div(tot, 256), 256, 0, h->ls>>>(
            (const double*)h->Mpart, CK, c0, cs, h->R, tiles, (double*)h->Mred);
      else
        k_chunk_sum<float><<<(unsigned)ceil_div(tot, 256), 256, 0, h->ls>>>(
            (const float*)h->Mpart, CK, c0, cs, h->R, tiles, (float*)h->Mred);
      h->launches++;
      st = check_launch(h, "k_chunk_sum");
    }
    return st;
  }
  st = h->dtype == CP_F64 ? launch_gather<double>(h, n) : launch_gather<float>(h, n);
  if (st) return st;
  h->pref_mode = -1;  // consumed
  if (sharded(h)) st = h->dtype == CP_F64 ? launch_reduce<double>(h, n) : launch_reduce<float>(h, n);
  return st;
}

// update (+ table + next batch when the rows are all local)
cp_status phase1(cp_sgd_s* h, int n, double alpha, const double* alpha_dev, int next_mode) {
  if (wide_mode(h, n)) {  // update, table of the updated A^(n), the next batch (+ its zw rows and Gamma)
    const bool f64 = h->dtype == CP_F64;
    cp_status st = f64 ? launch_uw_t<double>(h, n, alpha, alpha_dev) : launch_uw_t<float>(h, n, alpha, alpha_dev);
    if (sharded(h) && n == h->N - 1) return st;  // the rank's rows only: the table waits for the row exchange
    if (!st && next_mode >= 0) {
      st = launch_prefetch(h, next_mode);
      if (!st) h->pref_mode = next_mode;
    }
    return st;
  }
  const bool last_sharded = sharded(h) && n == h->N - 1;
  if (ut_fits(h, h->In_local[n])) {
    cp_status st;
    if (!last_sharded) {
      st = launch_ut(h, n, 1, 1, 0, h->dims[n], alpha, alpha_dev, sharded(h), next_mode);
      if (!st && next_mode >= 0) h->pref_mode = next_mode;
      return st;
    }
    return launch_ut(h, n, 1, 0, h->row0[n], h->In_local[n], alpha, alpha_dev, true, -1);
  }
  return h->dtype == CP_F64 ? launch_update<double>(h, n, alpha, alpha_dev, sharded(h))
                            : launch_update<float>(h, n, alpha, alpha_dev, sharded(h));
}

// table refresh of mode n when it could not be fused into phase 1 (rows gathered first / legacy)
cp_status phase2(cp_sgd_s* h, int n, int next_mode) {
  if (wide_mode(h, n)) {
    if (!(sharded(h) && n == h->N - 1)) return CP_OK;
    // slab shards, last mode: the rows of every rank are in place -- the table of the whole A^(N-1) (a
    // table-only k_update_wide taking over the factor from itself), then the next batch
    const bool f64 = h->dtype == CP_F64;
    cp_status st = f64 ? launch_uw_t<double>(h, n, 0.0, nullptr, h->one_dev, true)
                       : launch_uw_t<float>(h, n, 0.0, nullptr, h->one_dev, true);
    if (!st && next_mode >= 0) {
      st = launch_prefetch(h, next_mode);
      if (!st) h->pref_mode = next_mode;
    }
    return st;
  }
  const bool last_sharded = sharded(h) && n == h->N - 1;
  if (ut_fits(h, h->In_local[n])) {
    if (!last_sharded) return CP_OK;
    cp_status st = launch_ut(h, n, 0, 1, 0, h->dims[n], 0.0, nullptr, false, next_mode);
    if (!st && next_mode >= 0) h->pref_mode = next_mode;
    return st;
  }
  return launch_table_any(h, n);
}

cp_status nccl_check(cp_sgd_s* h, ncclResult_t r, const char* what) {
  if (r != 0) return h->fail(CP_ENCCL, "%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
  return CP_OK;
}

cp_status exchange_after0(cp_sgd_s* h, int n) {
  if (replica(h) && (h->flags & CP_FLAG_P2P)) return CP_OK;  // summed by k_update_wide from peer memory
  if (replica(h) && !(h->flags & CP_FLAG_EXTERNAL_COMM)) {  // M = sum over ranks of the chunk sums
    ProfScope ps(h, kKComm);
    const int dt = h->dtype == CP_F64 ? kNcclFloat64 : kNcclFloat32;
    const size_t cnt = (size_t)ceil_div(h->dims[n], kGUTI) * h->R * kGUTI;
    return nccl_check(h, g_nccl.AllReduce(h->Mred, h->Mred, cnt, dt, kNcclSum, h->comm, h->ls), "ncclAllReduce(M)");
  }
  if (!sharded(h) || (h->flags & CP_FLAG_EXTERNAL_COMM) || n == h->N - 1) return CP_OK;
  ProfScope ps(h, kKComm);
  const int dt = h->dtype == CP_F64 ? kNcclFloat64 : kNcclFloat32;
  if (wide_mode(h, n))  // the wide path's rank chunk sums (owned fibers only)
    return nccl_check(h, g_nccl.AllReduce(h->Mred, h->Mred, (size_t)ceil_div(h->dims[n], kGUTI) * h->R * kGUTI, dt,
                                          kNcclSum, h->comm, h->ls),
                      "ncclAllReduce(M)");
  return nccl_check(h, g_nccl.AllReduce(h->Msum, h->Msum, (size_t)h->R * h->In_local[n], dt, kNcclSum, h->comm,
                                        h->ls),
                    "ncclAllReduce(M)");
}

// every rank broadcasts its owned rows of A^(N-1); slab ranges are exchanged at init
cp_status exchange_after1(cp_sgd_s* h, int n, const std::vector<int64_t>& row_ranges) {
  if (!sharded(h) || (h->flags & CP_FLAG_EXTERNAL_COMM) || n != h->N - 1) return CP_OK;
  ProfScope ps(h, kKComm);
  const int dt = h->dtype == CP_F64 ? kNcclFloat64 : kNcclFloat32;
  cp_status st = nccl_check(h, g_nccl.GroupStart(), "ncclGroupStart");
  if (st) return st;
  for (int r = 0; r < h->world_size; ++r) {
    const int64_t a = row_ranges[2 * r], b = row_ranges[2 * r + 1];
    if (b <= a) continue;
    char* base = (char*)h->factors[n] + (size_t)a * h->R * h->esz;
    st = nccl_check(h, g_nccl.Broadcast(base, base, (size_t)(b - a) * h->R, dt, r, h->comm, h->ls),
                    "ncclBroadcast(rows)");
    if (st) break;
  }
  cp_status st2 = nccl_check(h, g_nccl.GroupEnd(), "ncclGroupEnd");
  return st ? st : st2;
}

}  // namespace

namespace {

cp_status do_step(cp_sgd_s* h, int n, int next_mode, double alpha, const double* alpha_dev,
                  const std::vector<int64_t>& rr) {
  cp_status st = phase0(h, n, alpha, alpha_dev);
  if (!st) st = exchange_after0(h, n);
  if (!st) st = phase1(h, n, alpha, alpha_dev, next_mode);
  if (!st) st = exchange_after1(h, n, rr);
  if (!st) st = phase2(h, n, next_mode);
  return st;
}

}  // namespace

// =================================================================================================
// C ABI
// =================================================================================================
extern "C" {

const char* cp_sgd_version(void) { return "cpsgd 0.1 (sm_100a)"; }

const char* cp_sgd_last_error(cp_sgd_t h) { return h ? h->err.c_str() : g_init_error.c_str(); }

static cp_status init_fail(cp_sgd_s* h, cp_status st) {
  g_init_error = h->err;
  cp_sgd_destroy(h);
  return st;
}

// row ranges [lo, hi) of every rank's slab of the last mode (owned rows exchanged after phase 1)
static std::vector<int64_t>* rr_store(cp_sgd_s* h, bool create) {
  if (h->row_ranges.empty() && !create) return nullptr;
  return &h->row_ranges;
}

cp_status cp_sgd_init(const cp_sgd_config* cfg, cp_sgd_t* out) {
  g_init_error.clear();
  if (!cfg || !out) {
    g_init_error = "NULL config or output";
    return CP_EINVAL;
  }
  *out = nullptr;
  cp_sgd_s* h = new (std::nothrow) cp_sgd_s();
  if (!h) {
    g_init_error = "host allocation failed";
    return CP_ENOMEM;
  }
  // ---- validation ----
  if (cfg->order < 3 || cfg->order > kMaxOrder) return init_fail(h, h->fail(CP_EINVAL, "order N=%d not in [3,16]", cfg->order));
  if (!cfg->dims || !cfg->factors || !cfg->X) return init_fail(h, h->fail(CP_EINVAL, "NULL dims/factors/X"));
  if (cfg->rank < 1 || cfg->rank > kMaxRank) return init_fail(h, h->fail(CP_EINVAL, "rank R=%d not in [1,64]", cfg->rank));
  if (cfg->dtype != CP_F32 && cfg->dtype != CP_F64) return init_fail(h, h->fail(CP_EINVAL, "bad dtype"));
  if (cfg->batch < 1) return init_fail(h, h->fail(CP_EINVAL, "batch B=%lld < 1", (long long)cfg->batch));
  if (cfg->sampler < 0 || cfg->sampler > 4) return init_fail(h, h->fail(CP_EINVAL, "bad sampler"));
  if (cfg->rule != CP_STEP_FIXED && cfg->rule != CP_STEP_ADAPTIVE && cfg->rule != CP_STEP_ALS)
    return init_fail(h, h->fail(CP_EINVAL, "bad rule"));
  if (!(cfg->alpha >= 0.0)) return init_fail(h, h->fail(CP_EINVAL, "alpha < 0"));
  if (cfg->rule == CP_STEP_ADAPTIVE && !(cfg->eta > 0.0)) return init_fail(h, h->fail(CP_EINVAL, "eta <= 0"));
  if (!(cfg->b >= 0.0) || !(cfg->eps >= 0.0)) return init_fail(h, h->fail(CP_EINVAL, "b or eps < 0"));
  if (cfg->world_size < 1 || cfg->world_rank < 0 || cfg->world_rank >= cfg->world_size)
    return init_fail(h, h->fail(CP_EINVAL, "bad world rank/size"));
  h->N = cfg->order;
  h->R = cfg->rank;
  h->dtype = cfg->dtype;
  h->esz = cfg->dtype == CP_F64 ? 8 : 4;
  h->sampler = cfg->sampler;
  h->rule = cfg->rule;
  cudaGetDevice(&h->device);
  h->B = cfg->batch;
  h->alpha = cfg->alpha;
  h->eta = cfg->eta;
  h->bpar = cfg->b;
  h->eps = cfg->eps;
  h->seed = cfg->seed;
  h->stream = (cudaStream_t)cfg->stream;
  h->ls = h->stream;
  if (cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
    return init_fail(h, h->fail(CP_ECUDA, "cudaStreamCreate failed"));
  h->world_rank = cfg->world_rank;
  h->world_size = cfg->world_size;
  h->flags = cfg->flags;
  h->X = cfg->X;
  for (int k = 0; k < h->N; ++k) {
    if (cfg->dims[k] < 1 || cfg->dims[k] > (int64_t)1 << 31)
      return init_fail(h, h->fail(CP_EINVAL, "dims[%d]=%lld out of range", k, (long long)cfg->dims[k]));
    if (!cfg->factors[k]) return init_fail(h, h->fail(CP_EINVAL, "factor %d is NULL", k));
    h->dims[k] = cfg->dims[k];
    h->factors[k] = cfg->factors[k];
    h->ldims[k] = cfg->dims[k];
  }
  if ((h->flags & CP_FLAG_P2P) && !(h->flags & CP_FLAG_REPLICA))
    return init_fail(h, h->fail(CP_EINVAL, "CP_FLAG_P2P is the replicas' exchange: it needs CP_FLAG_REPLICA"));
  if ((h->flags & CP_FLAG_REPLICA) && (h->flags & CP_FLAG_STRATIFIED))
    return init_fail(h, h->fail(CP_EINVAL, "CP_FLAG_REPLICA and CP_FLAG_STRATIFIED exclude each other"));
  if (sharded(h)) {
    if (cfg->slab_begin < 0 || cfg->slab_end > h->dims[h->N - 1] || cfg->slab_begin >= cfg->slab_end)
      return init_fail(h, h->fail(CP_EINVAL, "bad slab range [%lld,%lld)", (long long)cfg->slab_begin,
                                  (long long)cfg->slab_end));
    h->lo_last = cfg->slab_begin;
    h->hi_last = cfg->slab_end;
    h->ldims[h->N - 1] = cfg->slab_end - cfg->slab_begin;
  } else {
    h->lo_last = 0;
    h->hi_last = h->dims[h->N - 1];
  }
  int64_t st_ = 1;
  for (int k = 0; k < h->N; ++k) {
    h->lstride[k] = st_;
    st_ *= h->ldims[k];
  }
  const int64_t local_numel = st_;
  // ---- block windows and per-mode batch sizes (R6) ----
  const bool block = (h->sampler == CP_BLOCK_LEVERAGE || h->sampler == CP_BLOCK_EUCLIDEAN);
  for (int n = 0; n < h->N; ++n) {
    int pos = 0;
    int64_t rem = h->B, prod = 1;
    for (int k = 0; k < h->N; ++k) {
      if (k == n) continue;
      int64_t bk;
      if (cfg->block_window) {
        bk = cfg->block_window[pos];
        if (bk < 1) return init_fail(h, h->fail(CP_EINVAL, "block_window[%d] < 1", pos));
      } else {
        const int left = h->N - 1 - pos;
        int64_t d = 1;
        for (d = 1; d <= rem; ++d) {
          if (rem % d) continue;
          double pw = 1.0;
          for (int t = 0; t < left; ++t) pw *= (double)d;
          if (pw >= (double)rem) break;
        }
        if (d > rem) d = rem;
        rem /= d;
        bk = d;
      }
      bk = std::min<int64_t>(bk, h->dims[k]);
      h->window[n][pos] = (int32_t)bk;
      prod *= bk;
      ++pos;
    }
    h->bmax[n] = block ? prod : h->B;
  }
  // ---- tiling of k_gather per mode ----
  int64_t Bmax_all = 0, Mp_elems = 0, Gp_elems = 0, Imax = 0, Msum_elems = 0;
  for (int n = 0; n < h->N; ++n) {
    const bool last = (n == h->N - 1);
    h->In_local[n] = last ? h->ldims[n] : h->dims[n];
    h->row0[n] = last ? h->lo_last : 0;
    h->ntiles[n] = (int)ceil_div(h->In_local[n], kTI);
    const int64_t bm = h->bmax[n];
    int64_t nch = std::max<int64_t>(1, 296 / h->ntiles[n]);
    nch = std::min<int64_t>(nch, std::max<int64_t>(1, ceil_div(bm, 8)));
    int CG = 1;
    while (CG * 2 <= nch && CG < 8) CG *= 2;
    h->TB[n] = ceil_div(bm, nch);
    h->nchunks[n] = (int)(ceil_div(ceil_div(bm, h->TB[n]), CG) * CG);
    h->cgather[n] = CG;
    h->nparts[n] = h->nchunks[n] / CG;
    Bmax_all = std::max(Bmax_all, bm);
    Mp_elems = std::max(Mp_elems, (int64_t)h->nparts[n] * h->R * h->In_local[n]);
    Gp_elems = std::max(Gp_elems, (int64_t)h->nparts[n] * h->R * h->R);
    Msum_elems = std::max(Msum_elems, (int64_t)h->R * h->In_local[n]);
    Imax = std::max(Imax, h->dims[n]);
  }
  // ---- allocations ----
#define ALLOC(ptr, bytes)                                                                        \
  do {                                                                                           \
    cudaError_t e_ = cudaMalloc((void**)&(ptr), (bytes));                                        \
    if (e_ != cudaSuccess)                                                                       \
      return init_fail(h, h->fail(CP_ENOMEM, "cudaMalloc(%zu): %s", (size_t)(bytes), cudaGetErrorString(e_))); \
  } while (0)
  for (int k = 0; k < h->N; ++k) {
    ALLOC(h->cdf[k], sizeof(uint64_t) * ((h->dims[k] + 15) & ~15));  // whole 16-row blocks (two-level search)
    ALLOC(h->pprob[k], sizeof(double) * h->dims[k]);
    if (h->rule == CP_STEP_ADAPTIVE) {
      ALLOC(h->S[k], h->esz * h->dims[k] * h->R);
      cudaMemsetAsync(h->S[k], 0, h->esz * h->dims[k] * h->R, h->stream);
    }
  }
  ALLOC(h->Ttot, sizeof(uint64_t) * h->N);
  ALLOC(h->idx, sizeof(int32_t) * Bmax_all * (h->N - 1));
  ALLOC(h->w, sizeof(double) * Bmax_all);
  ALLOC(h->beff, sizeof(int64_t));
  ALLOC(h->beff_api, sizeof(int64_t));
  ALLOC(h->last_mode_dev, sizeof(int));
  if (getenv("CPSGD_PDL")) h->pdl = true;
  if (getenv("CPSGD_DEBUG_TIMERS")) {
    ALLOC(h->dbg, sizeof(long long) * kDbgEntries);
    cudaMemsetAsync(h->dbg, 0, sizeof(long long) * kDbgEntries, h->stream);
  }
  ALLOC(h->zrow, h->esz * Bmax_all * h->R);
  ALLOC(h->fbase, sizeof(int64_t) * Bmax_all);
  ALLOC(h->iter_dev, sizeof(uint64_t));
  ALLOC(h->iter_tmp, sizeof(uint64_t));
  ALLOC(h->status_dev, sizeof(int));
  ALLOC(h->alpha_dev, sizeof(double));
  ALLOC(h->Mp, h->esz * Mp_elems);
  ALLOC(h->Gp, h->esz * Gp_elems);
  ALLOC(h->Msum, h->esz * Msum_elems);
  ALLOC(h->Gsum, h->esz * h->R * h->R);
  ALLOC(h->Gout, h->esz * Imax * h->R);
  ALLOC(h->Gam_out, h->esz * h->R * h->R);
  ALLOC(h->fac_dev, sizeof(void*) * h->N);
  ALLOC(h->ldims_dev, sizeof(int64_t) * h->N);
  h->fit_blocks = 148 * 4;
  ALLOC(h->fit_partial, sizeof(double) * 2 * h->fit_blocks);
  if (cudaMallocHost((void**)&h->pinned, 64) != cudaSuccess)
    return init_fail(h, h->fail(CP_ENOMEM, "cudaMallocHost failed"));
  cudaMemsetAsync(h->iter_dev, 0, sizeof(uint64_t), h->stream);
  cudaMemsetAsync(h->status_dev, 0, sizeof(int), h->stream);
  cudaMemsetAsync(h->Gout, 0, h->esz * Imax * h->R, h->stream);
  cudaMemsetAsync(h->beff, 0, sizeof(int64_t), h->stream);
  cudaMemcpyAsync(h->fac_dev, h->factors, sizeof(void*) * h->N, cudaMemcpyHostToDevice, h->stream);
  cudaMemcpyAsync(h->ldims_dev, h->ldims, sizeof(int64_t) * h->N, cudaMemcpyHostToDevice, h->stream);
  // uniform tables are constant: q = 1, cdf[i] = i + 1, T = I (materialised for get_table)
  {
    std::vector<uint64_t> hc;
    std::vector<uint64_t> Th(h->N);
    for (int k = 0; k < h->N; ++k) Th[k] = (uint64_t)h->dims[k];
    if (h->sampler == CP_UNIFORM) {
      for (int k = 0; k < h->N; ++k) {
        hc.resize(h->dims[k]);
        std::vector<double> hp(h->dims[k], 1.0 / (double)h->dims[k]);
        for (int64_t i = 0; i < h->dims[k]; ++i) hc[i] = (uint64_t)(i + 1);
        cudaMemcpy(h->cdf[k], hc.data(), sizeof(uint64_t) * h->dims[k], cudaMemcpyHostToDevice);
        cudaMemcpy(h->pprob[k], hp.data(), sizeof(double) * h->dims[k], cudaMemcpyHostToDevice);
      }
      cudaMemcpy(h->Ttot, Th.data(), sizeof(uint64_t) * h->N, cudaMemcpyHostToDevice);
    }
  }
  // ---- kernel attributes ----
  {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // dynamic shared-memory budget of the sampler / fused kernels (opt-in max less 4 KB of statics)
    h->sample_smem = (int)std::min(allow_max_dyn_smem(k_sample<float>), allow_max_dyn_smem(k_sample<double>));
    h->sample_smem = std::min(h->sample_smem, optin - 4096);
    allow_max_dyn_smem(k_table<float>);
    allow_max_dyn_smem(k_table<double>);
    cudaGetLastError();
  }
  plan_fused(h);
  // ---- wide single-GPU path (k_gather_update) eligibility and buffers ----
  if (!(h->flags & CP_FLAG_NO_WIDE)) {  // single GPU, replicas, and slab shards (the last mode on the rank's rows)
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    bool any = false;
    const bool tc = h->dtype == CP_F32 && !(h->flags & CP_FLAG_NO_TC);
    h->use_tc = tc;
    int64_t mpart = 0;
    for (int n = 0; n < h->N; ++n) {
      const int64_t nt = ceil_div(h->In_local[n], kGUTI);
      // chunks per I-tile: one wave of CTAs (tcgen05 kernel: one CTA per SM; FFMA kernel: two)
      const int64_t slots = tc ? sm_budget() : 2 * sm_budget();
      int64_t CK = std::max<int64_t>(1, std::min<int64_t>(slots / nt, 64));
      // replicas: P times as many chunks, every rank one wave of its own (chunks rank, rank + P, ...)
      if (replica(h)) CK *= h->world_size;
      const int64_t gran = tc ? kTCKS : 8;
      int64_t KB = ceil_div(ceil_div(h->bmax[n], CK), gran) * gran;
      CK = ceil_div(h->bmax[n], KB);  // no empty chunk
      size_t gs = h->esz == 8 ? gu_smem_bytes<double, 8>(KB) : gu_smem_bytes<float, 8>(KB);
      if (tc) gs = std::max(gs, tc_smem_bytes(KB));
      int64_t bmx = 0, cdfmax = 0;
      for (int k = 0; k < h->N; ++k) {
        bmx = std::max(bmx, h->bmax[k]);
        cdfmax = std::max(cdfmax, ts_cdf_elems(h, k));
      }
      const size_t us = std::max(uw_smem_bytes(h->R, h->esz, std::min<int64_t>(h->dims[n], 4096)),
                                 sw_smem_bytes(h->N, h->R, cdfmax, h->esz));
      const bool cores = h->esz == 8 ? uw_coresident<double>(h->R, h->dims[n]) : uw_coresident<float>(h->R, h->dims[n]);
      if (gs + 1024 <= (size_t)optin && us <= (size_t)h->sample_smem && cores && (!replica(h) || CK >= h->world_size)) {
        h->gu_ck[n] = (int)CK;
        h->gu_kb[n] = KB;
        mpart = std::max(mpart, nt * CK * kGUTI * h->R);
        any = true;
      }
    }
    if (any) {
      const int P = h->R * (h->R + 1) / 2;
      ALLOC(h->uw_gpart, sizeof(double) * ceil_div(Imax, kUWRows) * P);
      ALLOC(h->uw_rownorm, sizeof(double) * Imax);
      ALLOC(h->uw_cnt, sizeof(unsigned));
      ALLOC(h->sc_cnt, sizeof(unsigned));
      cudaMemsetAsync(h->uw_cnt, 0, sizeof(unsigned), h->stream);
      cudaMemsetAsync(h->sc_cnt, 0, sizeof(unsigned), h->stream);
      ALLOC(h->uw_flag, sizeof(unsigned));
      cudaMemsetAsync(h->uw_flag, 0, sizeof(unsigned), h->stream);
      ALLOC(h->tw_W, sizeof(double) * h->R * h->R);
      ALLOC(h->tw_stat, sizeof(int) * 2);
      ALLOC(h->sc_q, sizeof(unsigned long long) * Imax);
      int64_t ncl = 0;
      for (int n = 0; n < h->N; ++n) ncl = std::max(ncl, ceil_div(ceil_div(h->bmax[n], kSWFibers), kSWCluster));
      ALLOC(h->sw_gcl, h->esz * ncl * h->R * h->R);
      ALLOC(h->Mpart, h->esz * mpart);
      if (multi(h)) ALLOC(h->Mred, h->esz * ceil_div(Imax, kGUTI) * kGUTI * h->R);
      if (sharded(h)) {
        ALLOC(h->one_dev, sizeof(int));
        const int one = 1;
        cudaMemcpy(h->one_dev, &one, sizeof(int), cudaMemcpyHostToDevice);
      }
      if (replica(h) && (h->flags & CP_FLAG_P2P)) {
        h->p2p_msz = ceil_div(Imax, kGUTI) * kGUTI * h->R;
        const size_t bytes = kP2PHead + 2 * h->esz * (size_t)h->p2p_msz;
        ALLOC(h->p2p_buf, bytes);
        cudaMemsetAsync(h->p2p_buf, 0, bytes, h->stream);
        ALLOC(h->p2p_epoch, sizeof(unsigned long long));
        cudaMemsetAsync(h->p2p_epoch, 0, sizeof(unsigned long long), h->stream);
        ALLOC(h->p2p_cnt, sizeof(unsigned) * 64);
        cudaMemsetAsync(h->p2p_cnt, 0, sizeof(unsigned) * 64, h->stream);
      }
      ALLOC(h->gu_cnt, sizeof(unsigned) * ceil_div(Imax, kGUTI));
      cudaMemsetAsync(h->gu_cnt, 0, sizeof(unsigned) * ceil_div(Imax, kGUTI), h->stream);
      ALLOC(h->zwp, h->esz * Bmax_all * zg_rp(h->R));
      ALLOC(h->gam_next, (h->esz * h->R * h->R + 15) / 16 * 16);  // whole 16-byte bulk copies
      cudaMemsetAsync(h->zwp, 0, h->esz * Bmax_all * zg_rp(h->R), h->stream);
      if (h->use_tc) {  // A images: every chunk rounded up to whole stages; rows r >= R stay zero
        int64_t rows = 0;
        for (int n = 0; n < h->N; ++n)
          if (h->gu_ck[n]) rows = std::max(rows, (int64_t)h->gu_ck[n] * h->gu_kb[n]);
        const size_t bytes = (size_t)ceil_div(rows, kTCKS) * kTCZBytes;
        ALLOC(h->zimg, bytes);
        cudaMemsetAsync(h->zimg, 0, bytes, h->stream);
      }
    } else {
      h->use_tc = false;
    }
  }
  if (replica(h)) {  // the batch split lives in the wide path's gather launch
    bool ok = true;
    for (int n = 0; n < h->N; ++n) ok = ok && wide_mode(h, n);
    if (!ok) return init_fail(h, h->fail(CP_EINVAL, "CP_FLAG_REPLICA needs the wide path for every mode (and a batch of "
                                                    "at least world_size chunks)"));
  }
  if (h->rule == CP_STEP_ALS) {  // the ALS step is implemented by the fused and wide kernels only
    bool ok = h->fused_cu > 0;
    if (!ok) {
      ok = !sharded(h);
      for (int n = 0; n < h->N; ++n) ok = ok && wide_mode(h, n);
    }
    if (!ok) return init_fail(h, h->fail(CP_EINVAL, "rule=als needs one GPU and the fused or wide path"));
  }
  // ---- optional mode-major copies (n >= 1; mode 0 fibers are already contiguous) ----
  if (h->flags & CP_FLAG_MODE_MAJOR) {
    for (int n = 1; n < h->N; ++n) {
      const int64_t In = h->ldims[n];
      int64_t inner = 1, outer = 1;
      for (int k = 0; k < n; ++k) inner *= h->ldims[k];
      for (int k = n + 1; k < h->N; ++k) outer *= h->ldims[k];
      const int64_t align = 16 / (int64_t)h->esz;
      h->pitch[n] = ceil_div(In, align) * align;
      // only where it fits (e.g. C5 slabs at P < 8): a mode without a copy gathers from the native layout
      size_t mem_free = 0, mem_tot = 0;
      const size_t bytes = h->esz * h->pitch[n] * inner * outer;
      if (cudaMemGetInfo(&mem_free, &mem_tot) != cudaSuccess || bytes + ((size_t)2 << 30) > mem_free) {
        cudaGetLastError();
        h->pitch[n] = 0;
        continue;
      }
      ALLOC(h->Xmm[n], bytes);
      dim3 tb(32, 8);
      dim3 grid((unsigned)ceil_div(inner, 32), (unsigned)ceil_div(In, 32), (unsigned)std::min<int64_t>(outer, 65535));
      if (h->dtype == CP_F64)
        k_transpose<double><<<grid, tb, 0, h->ls>>>((const double*)h->X, (double*)h->Xmm[n], In, inner, outer,
                                                        h->pitch[n]);
      else
        k_transpose<float><<<grid, tb, 0, h->ls>>>((const float*)h->X, (float*)h->Xmm[n], In, inner, outer,
                                                       h->pitch[n]);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return init_fail(h, h->fail(CP_ECUDA, "k_transpose: %s", cudaGetErrorString(e)));
    }
  }
#undef ALLOC
  // ---- persistent cooperative sweep kernel of the fp32 wide path ----
  if (!plan_pw(h)) return init_fail(h, h->fail(CP_ENOMEM, "persistent sweep kernel workspace"));
  // ---- NCCL communicator ----
  if (multi(h)) {
    auto* rr = rr_store(h, true);
    rr->assign(2 * h->world_size, 0);
    // no communicator for external-comm handles, nor for replicas exchanging over peer memory
    if (!(h->flags & CP_FLAG_EXTERNAL_COMM) && !(h->flags & CP_FLAG_P2P)) {
      if (!cfg->nccl_unique_id) return init_fail(h, h->fail(CP_EINVAL, "world_size > 1 needs nccl_unique_id"));
      std::string e;
      if (!g_nccl.load(e)) return init_fail(h, h->fail(CP_ENCCL, "%s", e.c_str()));
      ncclUniqueId id;
      memcpy(&id, cfg->nccl_unique_id, sizeof id);
      // replicas stay bitwise identical only if every run reduces in the same order: pin the ring
      // algorithm and one protocol unless the caller chose
      setenv("NCCL_ALGO", "Ring", 0);
      setenv("NCCL_PROTO", "LL128", 0);
      ncclResult_t r = g_nccl.CommInitRank(&h->comm, h->world_size, id, h->world_rank);
      if (r != 0) return init_fail(h, h->fail(CP_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r)));
      // exchange the slab ranges (allreduce of a one-hot vector)
      int64_t* d_rr = nullptr;
      if (cudaMalloc((void**)&d_rr, sizeof(int64_t) * 2 * h->world_size) != cudaSuccess)
        return init_fail(h, h->fail(CP_ENOMEM, "cudaMalloc(rr)"));
      std::vector<double> one(2 * h->world_size, 0.0);
      one[2 * h->world_rank] = (double)h->lo_last;
      one[2 * h->world_rank + 1] = (double)h->hi_last;
      double* d_one = nullptr;
      cudaMalloc((void**)&d_one, sizeof(double) * one.size());
      cudaMemcpy(d_one, one.data(), sizeof(double) * one.size(), cudaMemcpyHostToDevice);
      r = g_nccl.AllReduce(d_one, d_one, one.size(), kNcclFloat64, kNcclSum, h->comm, h->stream);
      cudaStreamSynchronize(h->stream);
      cudaMemcpy(one.data(), d_one, sizeof(double) * one.size(), cudaMemcpyDeviceToHost);
      cudaFree(d_one);
      cudaFree(d_rr);
      if (r != 0) return init_fail(h, h->fail(CP_ENCCL, "slab exchange: %s", g_nccl.GetErrorString(r)));
      for (size_t i = 0; i < one.size(); ++i) (*rr)[i] = (int64_t)one[i];
    }
  }
  // ---- stratified per-slab sampling (R26): the slab bounds of every rank ----
  if (h->flags & CP_FLAG_STRATIFIED) {
    const int P = h->world_size;
    const int64_t IL = h->dims[h->N - 1];
    if (P < 2 || P > kMaxStrata || block || h->B < P)
      return init_fail(h, h->fail(CP_EINVAL, "CP_FLAG_STRATIFIED needs 2 <= world_size <= %d, a row-wise sampler and "
                                             "batch >= world_size", kMaxStrata));
    if (cfg->slab_bounds) {
      for (int g = 0; g <= P; ++g) h->strat_lo[g] = cfg->slab_bounds[g];
    } else if (!(h->flags & CP_FLAG_EXTERNAL_COMM)) {
      const auto& rr = h->row_ranges;
      for (int g = 0; g < P; ++g) {
        if (g > 0 && rr[2 * g] != rr[2 * g - 1])
          return init_fail(h, h->fail(CP_EINVAL, "stratified sampling needs contiguous slabs in rank order"));
        h->strat_lo[g] = rr[2 * g];
      }
      h->strat_lo[P] = rr[2 * P - 1];
    } else {
      return init_fail(h, h->fail(CP_EINVAL, "CP_FLAG_STRATIFIED with CP_FLAG_EXTERNAL_COMM needs slab_bounds"));
    }
    bool ok = h->strat_lo[0] == 0 && h->strat_lo[P] == IL && h->strat_lo[h->world_rank] == h->lo_last &&
              h->strat_lo[h->world_rank + 1] == h->hi_last;
    for (int g = 0; g < P; ++g) ok = ok && h->strat_lo[g + 1] > h->strat_lo[g];
    if (!ok) return init_fail(h, h->fail(CP_EINVAL, "slab_bounds: not a contiguous rank-order cover of [0, I_last) "
                                                    "matching this rank's slab"));
  }
  // ---- initial tables of every mode ----
  for (int k = 0; k < h->N; ++k) {
    cp_status st = launch_table_any(h, k);
    if (st) return init_fail(h, st);
  }
  if (cudaStreamSynchronize(h->stream) != cudaSuccess)
    return init_fail(h, h->fail(CP_ECUDA, "init: %s", cudaGetErrorString(cudaGetLastError())));
  int status = 0;
  cudaMemcpy(&status, h->status_dev, sizeof(int), cudaMemcpyDeviceToHost);
  if (status != 0) return init_fail(h, h->fail((cp_status)status, "initial table build failed (status %d)", status));
  *out = h;
  return CP_OK;
}

cp_status cp_sgd_destroy(cp_sgd_t h) {
  if (!h) return CP_OK;
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->sweep_exec) cudaGraphExecDestroy(h->sweep_exec);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  for (int k = 0; k < kMaxOrder; ++k) {
    cudaFree(h->cdf[k]);
    cudaFree(h->pprob[k]);
    cudaFree(h->S[k]);
    cudaFree(h->Xmm[k]);
  }
  cudaFree(h->Ttot);
  cudaFree(h->idx);
  cudaFree(h->w);
  cudaFree(h->beff);
  cudaFree(h->beff_api);
  cudaFree(h->last_mode_dev);
  cudaFree(h->dbg);
  cudaFree(h->zrow);
  cudaFree(h->fbase);
  cudaFree(h->zwp);
  cudaFree(h->fstage[0]);  // one block for every mode (cp_sgd_steps_host)
  cudaFree(h->take_chg);
  cudaFree(h->multi_params);
  cudaFree(h->zimg);
  cudaFree(h->gam_next);
  cudaFree(h->Mpart);
  cudaFree(h->Mred);
  cudaFree(h->one_dev);
  if (h->chg_host) cudaFreeHost(h->chg_host);
  for (void* q : h->peer_opened) cudaIpcCloseMemHandle(q);
  cudaFree(h->p2p_buf);
  cudaFree(h->p2p_epoch);
  cudaFree(h->p2p_cnt);
  cudaFree(h->gu_cnt);
  cudaFree(h->uw_gpart);
  cudaFree(h->uw_rownorm);
  cudaFree(h->uw_cnt);
  cudaFree(h->sc_cnt);
  cudaFree(h->uw_flag);
  cudaFree(h->tw_W);
  cudaFree(h->tw_stat);
  cudaFree(h->sc_q);
  cudaFree(h->sw_gcl);
  cudaFree(h->iter_dev);
  cudaFree(h->iter_tmp);
  cudaFree(h->status_dev);
  cudaFree(h->alpha_dev);
  cudaFree(h->Mp);
  cudaFree(h->Gp);
  cudaFree(h->Msum);
  cudaFree(h->Gsum);
  cudaFree(h->Gout);
  cudaFree(h->Gam_out);
  cudaFree(h->fac_dev);
  cudaFree(h->ldims_dev);
  cudaFree(h->fit_partial);
  if (h->pinned) cudaFreeHost(h->pinned);
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  cudaFree(h->pw_gcl);
  cudaFree(h->pw_gram);
  cudaFree(h->pw_qraw);
  cudaFree(h->pw_coarse[0]);
  cudaFree(h->pw_agg);
  cudaFree(h->pw_aggf);
  cudaFree(h->pw_bar);
  cudaFree(h->pw_alphas);
  if (h->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(h->comm);
  cudaGetLastError();
  delete h;
  return CP_OK;
}

static cp_status check_mode(cp_sgd_t h, int mode) {
  if (!h) return CP_EINVAL;
  if (mode < 0 || mode >= h->N) return h->fail(CP_ERANGE, "mode %d out of range", mode);
  return CP_OK;
}

cp_status cp_sgd_sync(cp_sgd_t h) {
  if (!h) return CP_EINVAL;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return h->fail(CP_ECUDA, "stream: %s", cudaGetErrorString(e));
  int status = 0;
  CUDA_TRY(h, cudaMemcpy(&status, h->status_dev, sizeof(int), cudaMemcpyDeviceToHost));
  if (status != 0) {
    cudaMemsetAsync(h->status_dev, 0, sizeof(int), h->stream);
    return h->fail((cp_status)status, "device reported status %d (%s)", status,
                   status == CP_ENONFINITE ? "non-finite factor in a table rebuild" : "degenerate distribution");
  }
  return CP_OK;
}

cp_status cp_sgd_batch_max(cp_sgd_t h, int32_t mode, int64_t* bmax_host) {
  cp_status st = check_mode(h, mode);
  if (st) return st;
  if (!bmax_host) return h->fail(CP_EINVAL, "NULL output");
  *bmax_host = h->bmax[mode];
  return CP_OK;
}

cp_status cp_sgd_sample(cp_sgd_t h, int32_t mode, uint64_t iter, int32_t* idx_dev, double* w_dev,
                        int64_t* batch_eff_host) {
  cp_status st = check_mode(h, mode);
  if (st) return st;
  if (!idx_dev || !w_dev) return h->fail(CP_EINVAL, "NULL output buffer");
  uint64_t* pin = (uint64_t*)h->pinned;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));  // pinned staging reuse
  pin[0] = iter;
  CUDA_TRY(h, cudaMemcpyAsync(h->iter_tmp, pin, sizeof(uint64_t), cudaMemcpyHostToDevice, h->stream));
  st = launch_sample(h, mode, h->iter_tmp, idx_dev, w_dev, h->beff_api, false);
  if (st) return st;
  if (batch_eff_host) {
    CUDA_TRY(h, cudaMemcpyAsync(pin + 1, h->beff_api, sizeof(int64_t), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    *batch_eff_host = (int64_t)pin[1];
  }
  return CP_OK;
}

// the sampled-ALS rule is implemented by the fused and wide kernels only; the split / legacy update
// kernels would read it as the adaptive rule (and its unallocated accumulator)
static cp_status als_path_ok(cp_sgd_t h, int n) {
  if (h->rule == CP_STEP_ALS && !wide_mode(h, n))
    return h->fail(CP_EINVAL, "rule=als: mode %d is not on the wide path (the fused kernel runs only whole "
                              "constant-step sweeps / single steps)", n);
  return CP_OK;
}

static cp_status step_direct(cp_sgd_t h, int n, double alpha, int next_mode) {
  cp_status sa = als_path_ok(h, n);
  if (sa) return sa;
  const double a = (alpha < 0.0) ? h->alpha : alpha;
  auto* rr = rr_store(h, false);
  static const std::vector<int64_t> none;
  cp_status st = do_step(h, n, next_mode, a, nullptr, rr ? *rr : none);
  if (st) return st;
  h->iter_host++;
  h->last_mode = n;
  return CP_OK;
}

cp_status cp_sgd_step(cp_sgd_t h, int32_t mode, double alpha) {
  cp_status st = check_mode(h, mode);
  if (st) return st;
  if (multi(h) && (h->flags & CP_FLAG_EXTERNAL_COMM))
    return h->fail(CP_ESTATE, "external-comm handles must use cp_sgd_step_phase");
  if (h->fused_cu || h->pw_ok) {
    const double a = (alpha < 0.0) ? h->alpha : alpha;
    st = h->fused_cu ? launch_fused(h, 1, mode, 0, a, nullptr) : launch_pw(h, 1, mode, 0, a, nullptr, nullptr);
    if (st) return st;
    if (h->fused_cu || h->pw_ok) {
      h->iter_host++;
      h->last_mode = mode;
      return CP_OK;
    }  // else: the persistent grid was not co-resident -- the chain
  }
  return step_direct(h, mode, alpha, (mode + 1) % h->N);  // prefetch guess: the cyclic successor
}

cp_status cp_sgd_step_phase(cp_sgd_t h, int32_t mode, int32_t phase, double alpha) {
  cp_status st = check_mode(h, mode);
  if (st) return st;
  const double a = (alpha < 0.0) ? h->alpha : alpha;
  st = als_path_ok(h, mode);
  if (st) return st;
  if (phase == 0) {
    st = phase0(h, mode, a, nullptr);
    if (!st && multi(h) && !(h->flags & CP_FLAG_EXTERNAL_COMM)) st = exchange_after0(h, mode);
    return st;
  }
  if (phase == 1) {
    st = phase1(h, mode, a, nullptr, -1);
    if (!st && sharded(h) && !(h->flags & CP_FLAG_EXTERNAL_COMM)) {
      auto* rr = rr_store(h, false);
      static const std::vector<int64_t> none;
      st = exchange_after1(h, mode, rr ? *rr : none);
    }
    return st;
  }
  if (phase == 2) {
    st = phase2(h, mode, -1);
    if (!st) {
      h->iter_host++;
      h->last_mode = mode;
    }
    return st;
  }
  return h->fail(CP_EINVAL, "phase %d not in {0,1,2}", phase);
}

cp_status cp_sgd_exchange_info(cp_sgd_t h, int32_t mode, void** buf_dev, int64_t* count, int64_t* row_begin,
                               int64_t* row_end) {
  cp_status st = check_mode(h, mode);
  if (st) return st;
  if (replica(h) || (sharded(h) && wide_mode(h, mode) && mode < h->N - 1)) {  // the rank's chunk sum of M, [tiles][R][128]
    if (buf_dev) *buf_dev = h->Mred;
    if (count) *count = ceil_div(h->dims[mode], kGUTI) * h->R * kGUTI;
    if (row_begin) *row_begin = 0;
    if (row_end) *row_end = h->dims[mode];
    return CP_OK;
  }
  if (buf_dev) *buf_dev = (mode == h->N - 1 && sharded(h)) ? nullptr : h->Msum;
  if (count) *count = (mode == h->N - 1 && sharded(h)) ? 0 : (int64_t)h->R * h->In_local[mode];
  if (row_begin) *row_begin = h->row0[mode];
  if (row_end) *row_end = h->row0[mode] + h->In_local[mode];
  return CP_OK;
}

cp_status cp_sgd_exchange_copy(cp_sgd_t h, int32_t mode, void* buf_dev, int32_t to_lib) {
  cp_status st = check_mode(h, mode);
  if (st) return st;
  if (!buf_dev) return h->fail(CP_EINVAL, "NULL buffer");
  const bool red = replica(h) || (sharded(h) && wide_mode(h, mode) && mode < h->N - 1);
  if (sharded(h) && mode == h->N - 1) return h->fail(CP_EINVAL, "the last mode has no M exchange (owned rows)");
  void* lib = red ? h->Mred : h->Msum;
  const size_t bytes = red ? h->esz * (size_t)(ceil_div(h->dims[mode], kGUTI) * h->R * kGUTI)
                           : h->esz * (size_t)h->R * (size_t)h->In_local[mode];
  if (to_lib)
    CUDA_TRY(h, cudaMemcpyAsync(lib, buf_dev, bytes, cudaMemcpyDeviceToDevice, h->stream));
  else
    CUDA_TRY(h, cudaMemcpyAsync(buf_dev, lib, bytes, cudaMemcpyDeviceToDevice, h->stream));
  return CP_OK;
}

cp_status cp_sgd_sweep(cp_sgd_t h, int32_t nsweeps, int32_t order, const double* alpha_per_iter) {
  if (!h) return CP_EINVAL;
  if (nsweeps < 0) return h->fail(CP_EINVAL, "nsweeps < 0");
  if (order != CP_ORDER_CYCLIC && order != CP_ORDER_RANDOM) return h->fail(CP_EINVAL, "bad order");
  if (multi(h) && (h->flags & CP_FLAG_EXTERNAL_COMM))
    return h->fail(CP_ESTATE, "external-comm handles must use cp_sgd_step_phase");
  if (h->fused_cu && !alpha_per_iter) {
    if (nsweeps == 0) return CP_OK;
    const int64_t nst = (int64_t)nsweeps * h->N;
    cp_status st = launch_fused(h, (int)nst, 0, order, h->alpha, nullptr);
    if (st) return st;
    const uint64_t r_last = h->iter_host + nst - 1;
    h->last_mode = order == CP_ORDER_CYCLIC ? h->N - 1 : random_mode(h->seed, r_last, h->N);
    h->iter_host += nst;
    return CP_OK;
  }
  if (h->pw_ok) {  // one cooperative persistent launch for the whole call
    if (nsweeps == 0) return CP_OK;
    const int64_t nst = (int64_t)nsweeps * h->N;
    const double* al = nullptr;
    if (alpha_per_iter) {
      if (h->pw_alphas_cap < nst) {
        cudaFree(h->pw_alphas);
        h->pw_alphas = nullptr;
        h->pw_alphas_cap = 0;
        CUDA_TRY(h, cudaMalloc(&h->pw_alphas, sizeof(double) * nst));
        h->pw_alphas_cap = nst;
      }
      CUDA_TRY(h, cudaStreamSynchronize(h->stream));  // the previous call's schedule is no longer read
      CUDA_TRY(h, cudaMemcpy(h->pw_alphas, alpha_per_iter, sizeof(double) * nst, cudaMemcpyHostToDevice));
      al = h->pw_alphas;
    }
    cp_status st = launch_pw(h, (int)nst, 0, order, h->alpha, nullptr, al);
    if (st) return st;
    if (h->pw_ok) {
      const uint64_t r_last = h->iter_host + nst - 1;
      h->last_mode = order == CP_ORDER_CYCLIC ? h->N - 1 : random_mode(h->seed, r_last, h->N);
      h->iter_host += nst;
      return CP_OK;
    }  // else: not co-resident -- the chain below
    if (h->pw_chg) return CP_OK;  // cp_sgd_steps_host's optimistic call: nothing ran, it takes over and re-runs
  }
  const bool use_graph = order == CP_ORDER_CYCLIC && !alpha_per_iter && !(h->flags & CP_FLAG_NO_GRAPH) && !h->prof;
  if (!use_graph) {
    for (int s = 0; s < nsweeps; ++s)
      for (int j = 0; j < h->N; ++j) {
        const int n = (order == CP_ORDER_CYCLIC) ? j : random_mode(h->seed, h->iter_host, h->N);
        const int nx = (order == CP_ORDER_CYCLIC) ? (j + 1) % h->N : random_mode(h->seed, h->iter_host + 1, h->N);
        const double a = alpha_per_iter ? alpha_per_iter[(int64_t)s * h->N + j] : h->alpha;
        cp_status st = step_direct(h, n, a, nx);
        if (st) return st;
      }
    return CP_OK;
  }
  // graph path: the step size is read from alpha_dev; r lives on the device
  double* pin = h->pinned;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  pin[4] = h->alpha;
  CUDA_TRY(h, cudaMemcpyAsync(h->alpha_dev, pin + 4, sizeof(double), cudaMemcpyHostToDevice, h->stream));
  if (!h->sweep_exec) {
    cudaGraph_t g = nullptr;
    // capture on a private stream (the caller's may be the legacy default stream, which cannot
    // be captured); the graph is launched on the caller's stream
    h->ls = h->cap_stream;
    cudaError_t eb = cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (eb != cudaSuccess) {
      h->ls = h->stream;
      return h->fail(CP_ECUDA, "cudaStreamBeginCapture: %s", cudaGetErrorString(eb));
    }
    auto* rr = rr_store(h, false);
    static const std::vector<int64_t> none;
    cp_status st = CP_OK;
    const uint64_t l0 = h->launches;
    const int saved_pref = h->pref_mode;
    h->pref_mode = 0;  // the graph assumes the batch of mode 0 is prefetched when it starts
    for (int n = 0; n < h->N && !st; ++n)
      st = do_step(h, n, (n + 1) % h->N, h->alpha, h->alpha_dev, rr ? *rr : none);
    h->graph_end_pref = h->pref_mode;
    h->pref_mode = saved_pref;
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    h->ls = h->stream;
    h->sweep_launches = h->launches - l0;
    h->launches = l0;
    if (st) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (e != cudaSuccess) return h->fail(CP_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    e = cudaGraphInstantiate(&h->sweep_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return h->fail(CP_ECUDA, "graph instantiate: %s", cudaGetErrorString(e));
  }
  for (int s = 0; s < nsweeps; ++s) {
    if (h->pref_mode != 0) {
      cp_status st = launch_prefetch(h, 0);
      if (st) return st;
    }
    CUDA_TRY(h, cudaGraphLaunch(h->sweep_exec, h->stream));
    h->pref_mode = h->graph_end_pref;
    h->launches += h->sweep_launches;
    h->iter_host += h->N;
  }
  if (nsweeps > 0) h->last_mode = h->N - 1;
  return CP_OK;
}

cp_status cp_sgd_sweep_multi(cp_sgd_t* hs, int32_t nh, int32_t nsweeps) {
  if (!hs || nh < 1 || !hs[0]) return CP_EINVAL;
  cp_sgd_s* h0 = hs[0];
  if (nsweeps < 0) return h0->fail(CP_EINVAL, "nsweeps < 0");
  for (int i = 0; i < nh; ++i) {
    cp_sgd_s* h = hs[i];
    if (!h) return h0->fail(CP_EINVAL, "NULL handle %d", i);
    if (!h->fused_cu || h->world_size != 1)
      return h0->fail(CP_EINVAL, "handle %d: multi-chain sweeps need the fused single-GPU path", i);
    bool same = h->dtype == h0->dtype && h->N == h0->N && h->R == h0->R && h->fused_cu == h0->fused_cu &&
                h->fused_bpc == h0->fused_bpc && h->fused_rpc == h0->fused_rpc && h->device == h0->device;
    for (int k = 0; same && k < h->N; ++k) same = h->dims[k] == h0->dims[k];
    if (!same) return h0->fail(CP_EINVAL, "handle %d: geometry differs from handle 0", i);
    for (int j = 0; j < i; ++j)
      if (hs[j] == h) return h0->fail(CP_EINVAL, "handle %d repeated", i);
  }
  if (nsweeps == 0) return CP_OK;
  const int64_t nst = (int64_t)nsweeps * h0->N;
  int64_t imax = 0;
  for (int k = 0; k < h0->N; ++k) imax = std::max(imax, h0->dims[k]);
  if (h0->dtype == CP_F64)
    return imax > kFThreads ? launch_fused_multi_t<double, 2>(hs, nh, (int)nst) : launch_fused_multi_t<double, 1>(hs, nh, (int)nst);
  return imax > kFThreads ? launch_fused_multi_t<float, 2>(hs, nh, (int)nst) : launch_fused_multi_t<float, 1>(hs, nh, (int)nst);
}

// the factors' host <-> device copies of cp_sgd_steps_host: ONE transfer when both sides hold the modes back to back
// (a per-transfer cost of several us dominates 400 KB copies), else one per mode
static cp_status copy_factors(cp_sgd_t h, void* const* dst, void* const* src, cudaMemcpyKind kind) {
  bool packed = true;
  size_t tot = 0;
  for (int k = 0; k < h->N; ++k) {
    const size_t b = h->esz * h->dims[k] * h->R;
    if (k > 0 && ((const char*)dst[k - 1] + tot != dst[k] || (const char*)src[k - 1] + tot != src[k])) packed = false;
    tot = b;
  }
  if (packed) {
    size_t all = 0;
    for (int k = 0; k < h->N; ++k) all += h->esz * h->dims[k] * h->R;
    CUDA_TRY(h, cudaMemcpyAsync(dst[0], src[0], all, kind, h->stream));
    return CP_OK;
  }
  for (int k = 0; k < h->N; ++k)
    CUDA_TRY(h, cudaMemcpyAsync(dst[k], src[k], h->esz * h->dims[k] * h->R, kind, h->stream));
  return CP_OK;
}

cp_status cp_sgd_steps_host(cp_sgd_t h, int32_t first_mode, int32_t nsteps, double alpha,
                            void* const* factors_host) {
  cp_status st = check_mode(h, first_mode);
  if (st) return st;
  if (!factors_host) return h->fail(CP_EINVAL, "NULL factors_host");
  const bool fused = h->fused_cu && nsteps > 0;
  bool wide = !fused && h->world_size == 1;  // every mode on the wide path: k_update_wide takes over
  for (int k = 0; k < h->N; ++k) wide = wide && wide_mode(h, k);
  const bool stage = fused || wide;
  if (stage && !h->fstage[0]) {  // the staging of every mode in one block, packed back to back
    size_t tot = 0;
    for (int k = 0; k < h->N; ++k) tot += h->esz * h->dims[k] * h->R;
    CUDA_TRY(h, cudaMalloc(&h->fstage[0], tot));
    for (int k = 1; k < h->N; ++k)
      h->fstage[k] = (char*)h->fstage[k - 1] + h->esz * h->dims[k - 1] * h->R;
  }
  {
    void* dst[kMaxOrder];
    for (int k = 0; k < h->N; ++k) dst[k] = stage ? h->fstage[k] : h->factors[k];
    st = copy_factors(h, dst, factors_host, cudaMemcpyHostToDevice);
    if (st) return st;
  }
  h->pref_mode = -1;
  // the host factors may differ from the device ones: rebuild the tables
  if (fused) {  // one persistent launch: changed factors taken over + their tables rebuilt, then the steps
    st = launch_fused(h, nsteps, first_mode, CP_ORDER_CYCLIC, (alpha < 0.0) ? h->alpha : alpha, nullptr, 1);
    if (st) return st;
    h->iter_host += nsteps;
    h->last_mode = (first_mode + nsteps - 1) % h->N;
  } else if (wide) {  // changed factors (bitwise, per mode) taken over by k_update_wide, tables rebuilt
    if (!h->take_chg) CUDA_TRY(h, cudaMalloc(&h->take_chg, sizeof(int) * kMaxOrder));
    CUDA_TRY(h, cudaMemsetAsync(h->take_chg, 0, sizeof(int) * kMaxOrder, h->stream));
    {  // every mode in one launch
      int64_t nmax = 0;
      for (int k = 0; k < h->N; ++k) nmax = std::max<int64_t>(nmax, h->dims[k] * h->R);
      const dim3 grid((unsigned)std::min<int64_t>(ceil_div(nmax, 256), 148 * 2), (unsigned)h->N);
      if (h->esz == 8) {
        TakeAll<double> a{};
        for (int k = 0; k < h->N; ++k) {
          a.fstage[k] = (const double*)h->fstage[k];
          a.A[k] = (const double*)h->factors[k];
          a.n[k] = h->dims[k] * h->R;
        }
        k_take_compare_all<double><<<grid, 256, 0, h->ls>>>(a, h->take_chg);
      } else {
        TakeAll<float> a{};
        for (int k = 0; k < h->N; ++k) {
          a.fstage[k] = (const float*)h->fstage[k];
          a.A[k] = (const float*)h->factors[k];
          a.n[k] = h->dims[k] * h->R;
        }
        k_take_compare_all<float><<<grid, 256, 0, h->ls>>>(a, h->take_chg);
      }
      h->launches++;
      st = check_launch(h, "k_take_compare_all");
      if (st) return st;
    }
    const bool whole = first_mode == 0 && nsteps % h->N == 0 && alpha < 0.0;
    if (whole && h->pw_ok) {
      // optimistic (the usual case: the host holds what the last call returned): the persistent launch itself checks
      // the flags and does nothing if any is set (status kPWTakeOver) -- no take-over launches, no host round trip
      const uint64_t it0 = h->iter_host;
      const int lm0 = h->last_mode;
      h->pw_chg = h->take_chg;
      st = cp_sgd_sweep(h, nsteps / h->N, CP_ORDER_CYCLIC, nullptr);
      h->pw_chg = nullptr;
      if (st) return st;
      if (h->pw_ok) {  // (a refused cooperative launch ran nothing: the take-over path below, on the chain)
        st = copy_factors(h, factors_host, h->factors, cudaMemcpyDeviceToHost);
        if (st) return st;
        // the status with the factors (pinned, same stream): one host round trip for the whole call
        if (!h->chg_host) CUDA_TRY(h, cudaMallocHost(&h->chg_host, sizeof(int) * kMaxOrder));
        CUDA_TRY(h, cudaMemcpyAsync(h->chg_host, h->status_dev, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CUDA_TRY(h, cudaStreamSynchronize(h->stream));
        const int status = h->chg_host[0];
        if (status == 0) return CP_OK;
        if (status != kPWTakeOver) return cp_sgd_sync(h);  // reports (and clears) the device status
        CUDA_TRY(h, cudaMemsetAsync(h->status_dev, 0, sizeof(int), h->stream));
        h->iter_host = it0;  // nothing ran: take over, then the sweeps
        h->last_mode = lm0;
      }
    }
    // the take-over / table rebuild of every mode, decided on the device: a mode whose flag is clear leaves the
    // kernel at once -- no host round trip between the copies in and the sweep
    for (int k = 0; k < h->N; ++k) {
      st = h->esz == 8 ? launch_uw_t<double>(h, k, 0.0, nullptr, h->take_chg + k)
                       : launch_uw_t<float>(h, k, 0.0, nullptr, h->take_chg + k);
      if (st) return st;
    }
    if (whole) {  // whole cyclic sweeps: the sweep graph
      st = cp_sgd_sweep(h, nsteps / h->N, CP_ORDER_CYCLIC, nullptr);
      if (st) return st;
    } else {
      for (int s = 0; s < nsteps; ++s) {
        st = cp_sgd_step(h, (first_mode + s) % h->N, alpha);
        if (st) return st;
      }
    }
  } else {
    for (int k = 0; k < h->N; ++k) {
      st = launch_table_any(h, k);
      if (st) return st;
    }
    for (int s = 0; s < nsteps; ++s) {
      st = cp_sgd_step(h, (first_mode + s) % h->N, alpha);
      if (st) return st;
    }
  }
  st = copy_factors(h, factors_host, h->factors, cudaMemcpyDeviceToHost);
  if (st) return st;
  return cp_sgd_sync(h);
}

cp_status cp_sgd_p2p_buffer(cp_sgd_t h, void** buf_dev, int64_t* bytes) {
  if (!h || !buf_dev) return CP_EINVAL;
  if (!h->p2p_buf) return h->fail(CP_ESTATE, "not a CP_FLAG_P2P replica handle");
  *buf_dev = h->p2p_buf;
  if (bytes) *bytes = kP2PHead + 2 * (int64_t)h->esz * h->p2p_msz;
  return CP_OK;
}

cp_status cp_sgd_p2p_peers(cp_sgd_t h, void* const* peer_bufs_dev) {
  if (!h || !peer_bufs_dev) return CP_EINVAL;
  if (!h->p2p_buf) return h->fail(CP_ESTATE, "not a CP_FLAG_P2P replica handle");
  for (int g = 0; g < h->world_size; ++g) {
    if (!peer_bufs_dev[g]) return h->fail(CP_EINVAL, "peer buffer %d is NULL", g);
    h->peer[g] = peer_bufs_dev[g];
  }
  if (h->peer[h->world_rank] != h->p2p_buf) return h->fail(CP_EINVAL, "entry world_rank must be this handle's buffer");
  h->peers_set = true;
  return CP_OK;
}

cp_status cp_ipc_get_handle(const void* dev_ptr, void* out64_host) {
  if (!dev_ptr || !out64_host) return CP_EINVAL;
  cudaIpcMemHandle_t hd;
  if (cudaIpcGetMemHandle(&hd, const_cast<void*>(dev_ptr)) != cudaSuccess) {
    cudaGetLastError();
    return CP_ECUDA;
  }
  memcpy(out64_host, &hd, sizeof hd);
  return CP_OK;
}

cp_status cp_sgd_p2p_open(cp_sgd_t h, const void* handles64_host) {
  if (!h || !handles64_host) return CP_EINVAL;
  if (!h->p2p_buf) return h->fail(CP_ESTATE, "not a CP_FLAG_P2P replica handle");
  std::vector<void*> ptrs(h->world_size);
  for (int g = 0; g < h->world_size; ++g) {
    if (g == h->world_rank) {
      ptrs[g] = h->p2p_buf;
      continue;
    }
    cudaIpcMemHandle_t hd;
    memcpy(&hd, (const unsigned char*)handles64_host + 64 * g, sizeof hd);
    void* q = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&q, hd, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return h->fail(CP_ECUDA, "cudaIpcOpenMemHandle(rank %d): %s", g, cudaGetErrorString(e));
    h->peer_opened.push_back(q);
    ptrs[g] = q;
  }
  return cp_sgd_p2p_peers(h, ptrs.data());
}

cp_status cp_nccl_unique_id(void* out128_host) {
  if (!out128_host) return CP_EINVAL;
  std::string e;
  if (!g_nccl.load(e)) return CP_ENCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != 0) return CP_ENCCL;
  memcpy(out128_host, &id, sizeof id < 128 ? sizeof id : 128);
  return CP_OK;
}

cp_status cp_slice_sqnorms(const void* X_dev, int32_t dtype, int64_t nslices, int64_t slice_len, double* out_dev,
                           void* stream) {
  if (!X_dev || !out_dev || nslices < 1 || slice_len < 1 || nslices > 65535 || (dtype != CP_F32 && dtype != CP_F64))
    return CP_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  double* part = nullptr;
  if (cudaMallocAsync((void**)&part, sizeof(double) * (size_t)nslices * kSliceChunks, st) != cudaSuccess)
    return CP_ENOMEM;
  const dim3 grid(kSliceChunks, (unsigned)nslices);
  if (dtype == CP_F64)
    k_slice_sq<double><<<grid, 256, 0, st>>>((const double*)X_dev, slice_len, part);
  else
    k_slice_sq<float><<<grid, 256, 0, st>>>((const float*)X_dev, slice_len, part);
  k_slice_sum<0><<<(unsigned)((nslices + 255) / 256), 256, 0, st>>>(part, nslices, out_dev);
  cudaFreeAsync(part, st);
  return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ECUDA;
}

cp_status cp_fit(cp_sgd_t h, double* fit_host) {
  if (!h || !fit_host) return CP_EINVAL;
  if (sharded(h) && (h->flags & CP_FLAG_EXTERNAL_COMM))
    return h->fail(CP_ESTATE, "cp_fit on an external-comm sharded handle: the rank-local residual is not the fit");
  int64_t nfib = 1;
  for (int k = 1; k < h->N; ++k) nfib *= h->ldims[k];
  // a fixed number of partials on every rank (the kernel zeroes the ones past nfib): the NCCL sum
  // below must see the same count everywhere, whatever each rank's slab length
  const int blocks = h->fit_blocks;
  {
    ProfScope ps(h, kKFit);
    if (h->dtype == CP_F64)
      k_fit<double><<<blocks, 256, 0, h->ls>>>((const double*)h->X, h->N, h->ldims_dev, h->lo_last, h->R,
                                                   (const double* const*)h->fac_dev, nfib, h->fit_partial);
    else
      k_fit<float><<<blocks, 256, 0, h->ls>>>((const float*)h->X, h->N, h->ldims_dev, h->lo_last, h->R,
                                                  (const float* const*)h->fac_dev, nfib, h->fit_partial);
    h->launches++;
  }
  cp_status st = check_launch(h, "k_fit");
  if (st) return st;
  if (sharded(h) && !(h->flags & CP_FLAG_EXTERNAL_COMM)) {
    // sum the per-block partials of all ranks (same layout on every rank)
    st = nccl_check(h, g_nccl.AllReduce(h->fit_partial, h->fit_partial, 2 * (size_t)blocks, kNcclFloat64, kNcclSum,
                                        h->comm, h->stream),
                    "ncclAllReduce(fit)");
    if (st) return st;
  }
  std::vector<double> part(2 * blocks);
  CUDA_TRY(h, cudaMemcpyAsync(part.data(), h->fit_partial, sizeof(double) * 2 * blocks, cudaMemcpyDeviceToHost,
                              h->stream));
  st = cp_sgd_sync(h);
  if (st) return st;
  double res = 0.0, xx = 0.0;
  for (int b = 0; b < blocks; ++b) {
    res += part[2 * b];
    xx += part[2 * b + 1];
  }
  if (!(xx > 0.0)) return h->fail(CP_EDEGENERATE, "||X|| = 0");
  *fit_host = 1.0 - std::sqrt(res) / std::sqrt(xx);
  return CP_OK;
}

cp_status cp_sgd_get_table(cp_sgd_t h, int32_t mode, uint64_t* q_host, uint64_t* T_host, double* p_host) {
  cp_status st = check_mode(h, mode);
  if (st) return st;
  st = cp_sgd_sync(h);
  if (st) return st;
  const int64_t I = h->dims[mode];
  if (q_host) {
    std::vector<uint64_t> c(I);
    CUDA_TRY(h, cudaMemcpy(c.data(), h->cdf[mode], sizeof(uint64_t) * I, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < I; ++i) q_host[i] = c[i] - (i ? c[i - 1] : 0);
  }
  if (T_host) CUDA_TRY(h, cudaMemcpy(T_host, h->Ttot + mode, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (p_host) CUDA_TRY(h, cudaMemcpy(p_host, h->pprob[mode], sizeof(double) * I, cudaMemcpyDeviceToHost));
  return CP_OK;
}

cp_status cp_sgd_get_grad(cp_sgd_t h, void* G_host, int32_t* mode_host, void* Gamma_host) {
  if (!h) return CP_EINVAL;
  cp_status st = cp_sgd_sync(h);
  if (st) return st;
  if (h->last_mode < 0) return h->fail(CP_ESTATE, "no step taken yet");
  if (mode_host) *mode_host = h->last_mode;
  if (G_host)
    CUDA_TRY(h, cudaMemcpy(G_host, h->Gout, h->esz * h->dims[h->last_mode] * h->R, cudaMemcpyDeviceToHost));
  if (Gamma_host) CUDA_TRY(h, cudaMemcpy(Gamma_host, h->Gam_out, h->esz * h->R * h->R, cudaMemcpyDeviceToHost));
  return CP_OK;
}

cp_status cp_sgd_get_accum(cp_sgd_t h, int32_t mode, void* S_host) {
  cp_status st = check_mode(h, mode);
  if (st) return st;
  if (!h->S[mode]) return h->fail(CP_ESTATE, "only the adaptive rule has an accumulator");
  st = cp_sgd_sync(h);
  if (st) return st;
  CUDA_TRY(h, cudaMemcpy(S_host, h->S[mode], h->esz * h->dims[mode] * h->R, cudaMemcpyDeviceToHost));
  return CP_OK;
}

cp_status cp_sgd_get_iter(cp_sgd_t h, uint64_t* r_host) {
  if (!h || !r_host) return CP_EINVAL;
  cp_status st = cp_sgd_sync(h);
  if (st) return st;
  CUDA_TRY(h, cudaMemcpy(r_host, h->iter_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return CP_OK;
}

cp_status cp_sgd_set_iter(cp_sgd_t h, uint64_t r) {
  if (!h) return CP_EINVAL;
  cp_status st = cp_sgd_sync(h);
  if (st) return st;
  CUDA_TRY(h, cudaMemcpy(h->iter_dev, &r, sizeof(uint64_t), cudaMemcpyHostToDevice));
  h->iter_host = r;
  h->pref_mode = -1;
  return CP_OK;
}

cp_status cp_sgd_refresh_tables(cp_sgd_t h) {
  if (!h) return CP_EINVAL;
  h->pref_mode = -1;
  for (int k = 0; k < h->N; ++k) {
    cp_status st = launch_table_any(h, k);
    if (st) return st;
  }
  return cp_sgd_sync(h);
}

// debug: phase timestamps of the last k_update_table (CPSGD_DEBUG_TIMERS set at init)
cp_status cp_sgd_debug_timers(cp_sgd_t h, long long* out16) {
  if (!h || !out16) return CP_EINVAL;
  if (!h->dbg) return h->fail(CP_ESTATE, "CPSGD_DEBUG_TIMERS was not set at init");
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  CUDA_TRY(h, cudaMemcpy(out16, h->dbg, sizeof(long long) * kDbgEntries, cudaMemcpyDeviceToHost));
  return CP_OK;
}

cp_status cp_sgd_get_launches(cp_sgd_t h, uint64_t* n_host) {
  if (!h || !n_host) return CP_EINVAL;
  *n_host = h->launches;
  return CP_OK;
}

cp_status cp_sgd_profile(cp_sgd_t h, int32_t on) {
  if (!h) return CP_EINVAL;
  if (on) {
    CUDA_TRY(h, cudaStreamSynchronize(h->stream));
    h->prof_recs.clear();
    h->ev_next = 0;
  }
  h->prof = on != 0;
  return CP_OK;
}

cp_status cp_sgd_profile_read(cp_sgd_t h, int32_t cap, int32_t* ids, double* total_ms, int64_t* counts,
                              int32_t* n_out) {
  if (!h) return CP_EINVAL;
  CUDA_TRY(h, cudaStreamSynchronize(h->stream));
  double tot[kNumKernelIds] = {};
  int64_t cnt[kNumKernelIds] = {};
  for (auto& r : h->prof_recs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      tot[r.id] += ms;
      cnt[r.id]++;
    }
  }
  int m = 0;
  for (int k = 0; k < kNumKernelIds && m < cap; ++k) {
    if (!cnt[k]) continue;
    ids[m] = k;
    total_ms[m] = tot[k];
    counts[m] = cnt[k];
    ++m;
  }
  if (n_out) *n_out = m;
  cudaGetLastError();
  return CP_OK;
}

cp_status cp_sgd_trace_layout(cp_sgd_t h, int64_t* out7) {
  if (!h || !out7) return CP_EINVAL;
  const TraceLayout L = trace_layout(h);
  out7[0] = L.stride;
  out7[1] = L.o_idx;
  out7[2] = L.o_w;
  out7[3] = L.o_A;
  out7[4] = L.o_S;
  out7[5] = L.o_cdf;
  out7[6] = L.o_meta;
  return CP_OK;
}

cp_status cp_sgd_trace(cp_sgd_t h, void* buf_dev, int64_t cap) {
  if (!h) return CP_EINVAL;
  if (buf_dev && cap < 1) return h->fail(CP_EINVAL, "trace capacity < 1");
  cp_status st = cp_sgd_sync(h);  // earlier launches keep their (old) trace pointers
  if (st) return st;
  h->trace_base = (unsigned char*)buf_dev;
  h->trace_cap = buf_dev ? cap : 0;
  h->trace_count = 0;
  return CP_OK;
}

cp_status cp_sgd_trace_count(cp_sgd_t h, int64_t* n_host) {
  if (!h || !n_host) return CP_EINVAL;
  *n_host = h->trace_count;
  return CP_OK;
}

cp_status cp_sgd_path(cp_sgd_t h, int32_t* path_host) {
  if (!h || !path_host) return CP_EINVAL;
  *path_host = h->fused_cu ? 1 : (h->pw_ok ? 2 : 0);
  return CP_OK;
}

}  // extern "C"
