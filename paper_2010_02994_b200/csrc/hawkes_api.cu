// hawkes_api.cu -- context, C ABI (include/hawkes.h), kernel launch plumbing, exchanges.
//
// One evaluation (ell and d ell/dx) on rank r of W, PAIRS (default):
//   pass 1   sym_kernel<PASS=1> over this rank's chunk pairs (a <= b), each unordered pair
//            once -> per-(slot, event) partials (M', X', G1')     [rate pass, Alg. 2 step 1]
//   exchange W > 1: per-event slot sums, ncclAllReduce                       [S4]
//   fin1     fixed-order slot sum; lambda, rho' = 2^-64 / lambda, Lambda_n (erfc, expm1),
//            ell_n = log lambda_n - Lambda_n                            [Eq. 1, P:L92-101]
//   ell      fixed-order reduction of ell_n over all N events (same on every rank)
//   pass 2   sym_kernel<PASS=2> -> partials G2'                        [gradient pass, step 2]
//   exchange W > 1: per-event slot sums, ncclAllReduce                       [S6]
//   fin2     g_i = rho'_i G1'_i + G2'_i                                 [App. A, P:L385]
// ROWS (ordered pairs, pass_kernel): row tiles dealt to ranks zig-zag, allgather of (rho',
// ell_n) rows between the passes and of gradient rows at the end; bitwise identical for any
// W.  Around the evaluation: the HMC leapfrog / transition, block-MH moves and the on-device
// MH sweep, the BMDS density, CUDA-graph capture and replay, kernel timing and diagnostics.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cstddef>
#include <string>
#include <vector>

#include "../../include/hawkes.h"
#include "hawkes_kernels.cuh"
#include "hawkes_kernels_f32.cuh"
#include "hawkes_kernels_sym.cuh"
#include "hawkes_moves.cuh"
#include "hawkes_bmds.cuh"
#include "hawkes_ops.cuh"
#include "hawkes_mh.cuh"
#include "hawkes_mh_coop.cuh"
#include "hawkes_plan.h"

using namespace hk;

namespace {


thread_local std::string g_create_error;

// ------------------------------------------------------------------ NCCL via dlopen
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool load(std::string& err) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
      return false;
    }
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    allGather = (decltype(allGather))dlsym(h, "ncclAllGather");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    allReduce = (decltype(allReduce))dlsym(h, "ncclAllReduce");
    errStr = (decltype(errStr))dlsym(h, "ncclGetErrorString");
    if (!commInitRank || !allGather || !allReduce || !commDestroy || !errStr) {
      err = "libnccl.so.2 lacks required symbols";
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;

}  // namespace

// ======================================================================= context
struct hawkes_ctx {
  int64_t N = 0;
  int D = 0;
  int npad = 0;
  int ntiles = 0;          // row tiles of RT rows
  int chunk = 0, nchunks = 0, nslots = 0;
  hawkes_opts opts{};
  cudaStream_t stream = nullptr;
  int sms = 0;
  std::string err;
  int sticky = HAWKES_OK;

  // sharding: logical ranks this process runs (1, or emulate_world), their tile lists
  int W = 1;               // world size of the row sharding (real or emulated)
  std::vector<int> my_ranks;
  std::vector<std::vector<int>> tiles_of;   // per rank
  int max_tiles = 0;
  int* d_all_tiles = nullptr;               // [W][max_tiles], -1 padded
  std::vector<int*> d_tiles;                // per rank (points into d_all_tiles)
  std::vector<int2*> d_items1, d_items2;    // per rank
  std::vector<int> n_items;                 // per rank
  ncclComm_t comm = nullptr;
  // HAWKES_ALGO_PAIRS
  bool pairs = false;
  std::vector<int2*> d_sym;                 // per rank: off-diagonal chunk pairs
  std::vector<int> n_sym;
  int* d_own = nullptr;                     // [nchunks][nchunks] owner rank of pair (a <= b)
  int* d_every_tile = nullptr;              // all row tiles 0..ntiles-1
  bool multi = false;                       // W > 1 (real or emulated) or an NCCL communicator:
                                            // the sharded code path with its exchanges
  double* sums1 = nullptr;                  // W > 1: [W or 1][npad][K1] per-event sums
  double* sums2 = nullptr;                  // W > 1: [W or 1][npad][K2]

  // device buffers
  double* rec = nullptr;   // npad x REC
  float* rec32 = nullptr;  // npad x REC32 (fp32 path only)
  int* gid = nullptr;      // npad
  double* part1 = nullptr; // nchunks x npad x K1
  double* part2 = nullptr; // nchunks x npad x K2
  double* G1 = nullptr;    // npad x D
  double* rl = nullptr;    // npad x 2 (rho', ell_n)
  double* rates = nullptr; // npad x 4 (lambda, mu, xi, Lambda)
  double* grad = nullptr;  // npad x D
  double* xstage = nullptr;// N x D staging
  double* sendbuf = nullptr;
  double* recvbuf = nullptr;
  int* counters = nullptr; // 4 per logical rank
  int2* tab = nullptr;     // exp table
  int* bad = nullptr;      // device-side input validation flag
  EvalStatus* st = nullptr;
  EvalStatus* h_st = nullptr;  // pinned
  // leapfrog state
  double *lf_x = nullptr, *lf_p = nullptr, *lf_minv = nullptr, *lf_lo = nullptr, *lf_hi = nullptr;

  // state
  bool have_t = false, have_x = false, have_p = false;
  bool rates_valid = false;   // pass 1 + exchange done for current (x, t, Theta)
  bool grad_valid = false;
  bool rates_exchanged = false;
  double tN = 0.0;
  hawkes_params params{};
  PassConst pc{};
  PassConst32 pc32{};
  FinConst fc{};

  // timing
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_rate, ev_grad;
  std::vector<cudaEvent_t> ev_pool;
  double acc_rate_ms = 0, acc_grad_ms = 0;
  int64_t n_rate = 0, n_grad = 0;
  int64_t launches = 0;

  int grid1 = 0, grid2 = 0;
  int grid_s1 = 0, grid_s2 = 0;
  DevConsts* d_consts = nullptr;
  // CUDA graphs of one evaluation (single process, W = 1, timing off)
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t gexec[3] = {nullptr, nullptr, nullptr};   // rates, rates+grad, grad only
  bool graphs = false;
  bool capturing = false;
  int64_t graph_launches[3] = {0, 0, 0};
  int evals_same_consts = 0;   // evaluations since the last constants change
  // block moves (hawkes_propose_move / hawkes_accept_move)
  int* d_slot_of = nullptr;    // N, -1 or the event's index in the pending proposal
  int* d_move_idx = nullptr;   // MOVE_MAX
  double* d_move_x = nullptr;  // MOVE_MAX x D
  double* d_move_delta = nullptr;  // Npad x 2
  double* d_move_rows = nullptr;   // MOVE_MAX x 2
  double* d_move_part = nullptr;   // ceil(N/256) block sums
  double* d_move_rows_part = nullptr;  // MOVE_MAX x nsplit (<= MOVE_NSPLIT) x 2
  bool lam_valid = false;      // rates[][] hold lambda of the current state (all rows)
  // coarsening regions and the on-device block MH sweep (hawkes_set_regions / hawkes_mh_sweep)
  int reg_kind = 0;
  double* d_reg_c = nullptr;   // N x D region centres
  double* d_reg_s = nullptr;   // N half-widths / radii
  int* d_mh_blocks = nullptr;  // mh_cap event indices of the current sweep
  int* d_mh_stamp = nullptr;   // N: cooperative sweep's (block << 8) | slot stamps
  int* d_mh_acc = nullptr;     // mh_bcap decisions
  double* d_mh_la = nullptr;   // mh_bcap log alphas
  size_t mh_cap = 0, mh_bcap = 0;
  cudaGraphExec_t mh_gexec = nullptr;  // captured block step (k = mh_gk)
  int mh_gk = 0;
  bool coop_ok = false;                // device supports cooperative launches
  int64_t mh_graph_launches = 0;       // kernel launches per replay
  cudaStream_t mh_stream = nullptr;
  cudaEvent_t mh_ev0 = nullptr, mh_ev1 = nullptr;
  // BMDS (hawkes_set_bmds / hawkes_bmds_logdensity / hawkes_set_potential)
  double* d_Y = nullptr;       // N x N, lower triangle mirrored into the upper
  double* d_bgrad = nullptr;   // N x D
  double* d_brow = nullptr;    // N per-row values
  double* d_bpart = nullptr;   // (NB + 1) x N x (D + 1) unordered-pair BMDS slots, NB = ceil(N/32)
  BmdsConst bc{};
  bool have_bmds = false;
  int potential = HAWKES_POTENTIAL_HAWKES;
  int move_k = 0;              // pending proposal size (0: none)
};

namespace {

int set_err(hawkes_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (code == HAWKES_ERR_CUDA || code == HAWKES_ERR_NCCL) c->sticky = code;
  } else {
    g_create_error = buf;
  }
  return code;
}

#define CU(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return set_err(ctx, HAWKES_ERR_CUDA, "%s failed: %s (%s:%d)", #call,              \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                       \
  } while (0)

#define CHECK_LAUNCH()                                                                  \
  do {                                                                                  \
    ++ctx->launches;                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      return set_err(ctx, HAWKES_ERR_CUDA, "kernel launch failed: %s (%s:%d)",          \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                       \
  } while (0)

#define NC(call)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (call);                                                           \
    if (r_ != ncclSuccess)                                                              \
      return set_err(ctx, HAWKES_ERR_NCCL, "%s failed: %s", #call, g_nccl.errStr(r_));  \
  } while (0)

#define ENTER(ctx)                                                                      \
  do {                                                                                  \
    if (!(ctx)) return HAWKES_ERR_ARG;                                                  \
    if ((ctx)->sticky != HAWKES_OK) return (ctx)->sticky;                               \
    cudaError_t e_ = cudaSetDevice((ctx)->opts.device);                                 \
    if (e_ != cudaSuccess) return set_err(ctx, HAWKES_ERR_CUDA, "cudaSetDevice: %s",    \
                                          cudaGetErrorString(e_));                      \
  } while (0)

template <typename T>
int dalloc(hawkes_ctx* ctx, T** p, size_t count) {
  cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(ctx, HAWKES_ERR_OOM, "cudaMalloc of %zu bytes failed: %s", count * sizeof(T),
                   cudaGetErrorString(e));
  }
  return HAWKES_OK;
}

#define TRY(x)                      \
  do {                              \
    int rc_ = (x);                  \
    if (rc_ != HAWKES_OK) return rc_; \
  } while (0)

int K1_of(int D) { return ((D + 3) / 2) * 2; }
int K2_of(int D) { return ((D + 1) / 2) * 2; }
int REC_of(int D) { return ((D + 3) / 2) * 2; }
int Layout32Rec(int D) { return ((2 * D + 3 + 3) / 4) * 4; }

// ---------------------------------------------------------------- dispatch on D
template <template <int> class F, typename... A>
int dispatchD(int D, A&&... a) {
  switch (D) {
    case 1: return F<1>::run(a...);
    case 2: return F<2>::run(a...);
    case 3: return F<3>::run(a...);
    case 4: return F<4>::run(a...);
    case 5: return F<5>::run(a...);
    case 6: return F<6>::run(a...);
    case 7: return F<7>::run(a...);
    case 8: return F<8>::run(a...);
  }
  return HAWKES_ERR_DIM;
}

template <int D, int PASS>
size_t pass_smem() {
  return (size_t)STAGES * TILE_J * Layout<D>::REC * sizeof(double) + STAGES * sizeof(uint64_t) +
         EXP_TABLE * sizeof(int2);
}

template <int D, int PASS, int R, int V>
size_t sym_smem() {
  const int KR = PASS == 1 ? 1 + D : D;
  const int copies = (V & 2) ? TAB_COPIES : 1;
  return (size_t)STAGES * TILE_J * Layout<D>::REC * sizeof(double) + STAGES * sizeof(uint64_t) +
         (size_t)EXP_TABLE * copies * sizeof(int2) + (size_t)4 * 32 * R * KR * sizeof(double) +
         ((V & 4) ? (size_t)4 * 32 * Layout<D>::REC * sizeof(double) : 0);
}

// sym_kernel variants: R rows per lane; V1 / V2 = the pass-1 / pass-2 variant bits
// (hawkes_kernels_sym.cuh).  Measured on B200 (profiles/r01_sym_variants.txt): the
// interleaved exp table pays in pass 1 (-3.4 %) but not in pass 2, where it costs more
// integer instructions than the bank conflicts it removes; the SoA columns pay in both.
template <int D, int R, int V1, int V2>
struct SymOps {
  static int setup(hawkes_ctx* ctx) {
    auto s1 = sym_kernel<D, 1, R, V1>;
    auto s2 = sym_kernel<D, 2, R, V2>;
    CU(cudaFuncSetAttribute(s1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym_smem<D, 1, R, V1>()));
    CU(cudaFuncSetAttribute(s2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym_smem<D, 2, R, V2>()));
    int b1 = 0, b2 = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, s1, THREADS, sym_smem<D, 1, R, V1>()));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, s2, THREADS, sym_smem<D, 2, R, V2>()));
    ctx->grid_s1 = std::max(1, b1) * ctx->sms;
    ctx->grid_s2 = std::max(1, b2) * ctx->sms;
    return HAWKES_OK;
  }
  static int launch(hawkes_ctx* ctx, int pass, const SymArgs& b) {
    const int grid = std::min(pass == 1 ? ctx->grid_s1 : ctx->grid_s2, b.n_items);
    if (pass == 1)
      sym_kernel<D, 1, R, V1><<<grid, THREADS, sym_smem<D, 1, R, V1>(), ctx->stream>>>(b);
    else
      sym_kernel<D, 2, R, V2><<<grid, THREADS, sym_smem<D, 2, R, V2>(), ctx->stream>>>(b);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

// default: pass 1 V = 6 (interleaved exp table copies + SoA columns), pass 2 V = 4 (SoA
// columns): the copies cut pass 1's bank conflicts (2 copies of the 2048-entry table:
// -1.6 %; 16 copies of the -DHK_EXP256 table: -3.4 %) but cost pass 2 an extra LOP3 per exp
// (+2.3 %).  HAWKES_SYM_V = 0 / 2 / 4 / 6 forces one variant for both passes (diagnostics,
// A/B on one box; 2 and 6-for-pass-2 exist for D = 2 only)
static int sym_variant() {
  static int v = [] {
    const char* e = getenv("HAWKES_SYM_V");
    return e ? atoi(e) : -1;
  }();
  return v;
}

template <int D, int V1, int V2>
int sym_call_v(hawkes_ctx* ctx, int pass, const SymArgs* b) {
  return pass ? SymOps<D, 4, V1, V2>::launch(ctx, pass, *b) : SymOps<D, 4, V1, V2>::setup(ctx);
}

template <int D>
int sym_call(hawkes_ctx* ctx, int pass, const SymArgs* b) {
  const int v = sym_variant();
  if (v == 0) return sym_call_v<D, 0, 0>(ctx, pass, b);
  if constexpr (D == 2) {
    if (v == 2) return sym_call_v<D, 2, 2>(ctx, pass, b);
    if (v == 4) return sym_call_v<D, 4, 4>(ctx, pass, b);
    if (v == 6) return sym_call_v<D, 6, 6>(ctx, pass, b);
  }
  return sym_call_v<D, 6, 4>(ctx, pass, b);
}

constexpr int SYM32_R = 4;
template <int D, int PASS>
size_t sym32_smem() {
  const int KR = PASS == 1 ? 1 + D : D;
  return (size_t)STAGES * TILE_J * Layout32<D>::REC * sizeof(float) + STAGES * sizeof(uint64_t) +
         (size_t)4 * 32 * SYM32_R * KR * sizeof(double) +
         (size_t)4 * 32 * Layout32<D>::REC * sizeof(float);   // per-warp SoA column buffers
}

// fp32 sym kernels read columns from per-warp SoA buffers (SOA = true, the default);
// HAWKES_SYM32_SOA=0 selects the AoS reads (diagnostics, D = 2 only)
static bool sym32_soa() {
  static bool v = [] {
    const char* e = getenv("HAWKES_SYM32_SOA");
    return !(e && atoi(e) == 0);
  }();
  return v;
}

template <int D, bool SOA>
int sym32_setup(hawkes_ctx* ctx) {
  auto s1 = sym_kernel_f32<D, 1, SYM32_R, SOA>;
  auto s2 = sym_kernel_f32<D, 2, SYM32_R, SOA>;
  CU(cudaFuncSetAttribute(s1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym32_smem<D, 1>()));
  CU(cudaFuncSetAttribute(s2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym32_smem<D, 2>()));
  int b1 = 0, b2 = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, s1, THREADS, sym32_smem<D, 1>()));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, s2, THREADS, sym32_smem<D, 2>()));
  ctx->grid_s1 = std::max(1, b1) * ctx->sms;
  ctx->grid_s2 = std::max(1, b2) * ctx->sms;
  return HAWKES_OK;
}

template <int D, bool SOA>
int sym32_launch(hawkes_ctx* ctx, int pass, const SymArgs32& b) {
  const int grid = std::min(pass == 1 ? ctx->grid_s1 : ctx->grid_s2, b.n_items);
  if (pass == 1)
    sym_kernel_f32<D, 1, SYM32_R, SOA><<<grid, THREADS, sym32_smem<D, 1>(), ctx->stream>>>(b);
  else
    sym_kernel_f32<D, 2, SYM32_R, SOA><<<grid, THREADS, sym32_smem<D, 2>(), ctx->stream>>>(b);
  CHECK_LAUNCH();
  return HAWKES_OK;
}

template <int D>
size_t pass_smem32() {
  return (size_t)STAGES * TILE_J * Layout32<D>::REC * sizeof(float) + STAGES * sizeof(uint64_t);
}

template <int D>
struct SetupD {
  static int run(hawkes_ctx* ctx) {
    CU(cudaFuncSetAttribute(k_move_delta_rows<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)move_smem_bytes<D>(MOVE_MAX)));
    if (ctx->rec32) {
      auto k1 = pass_kernel_f32<D, 1, R_ROWS>;
      auto k2 = pass_kernel_f32<D, 2, R_ROWS>;
      const size_t sm = pass_smem32<D>();
      CU(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      CU(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      int b1 = 0, b2 = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k1, THREADS, sm));
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k2, THREADS, sm));
      ctx->grid1 = std::max(1, b1) * ctx->sms;
      ctx->grid2 = std::max(1, b2) * ctx->sms;
      if constexpr (D <= SYM_MAX_D) if (ctx->pairs) {
        if constexpr (D == 2)
          if (!sym32_soa()) return sym32_setup<D, false>(ctx);
        return sym32_setup<D, true>(ctx);
      }
      return HAWKES_OK;
    }
    auto k1 = pass_kernel<D, 1, R_ROWS>;
    auto k2 = pass_kernel<D, 2, R_ROWS>;
    const size_t sm = pass_smem<D, 1>();
    CU(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    CU(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int b1 = 0, b2 = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, k1, THREADS, sm));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, k2, THREADS, sm));
    ctx->grid1 = std::max(1, b1) * ctx->sms;
    ctx->grid2 = std::max(1, b2) * ctx->sms;
    if constexpr (D <= SYM_MAX_D) if (ctx->pairs) TRY(sym_call<D>(ctx, 0, nullptr));
    return HAWKES_OK;
  }
};

void record_start(hawkes_ctx* ctx, bool rate) {
  if (!ctx->timing) return;
  cudaEvent_t a, b;
  if (ctx->ev_pool.size() >= 2) {
    a = ctx->ev_pool.back(); ctx->ev_pool.pop_back();
    b = ctx->ev_pool.back(); ctx->ev_pool.pop_back();
  } else {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  cudaEventRecord(a, ctx->stream);
  (rate ? ctx->ev_rate : ctx->ev_grad).push_back({a, b});
}
void record_stop(hawkes_ctx* ctx, bool rate) {
  if (!ctx->timing) return;
  cudaEventRecord((rate ? ctx->ev_rate : ctx->ev_grad).back().second, ctx->stream);
}
void harvest_events(hawkes_ctx* ctx) {
  for (int which = 0; which < 2; ++which) {
    auto& v = which == 0 ? ctx->ev_rate : ctx->ev_grad;
    for (auto& pr : v) {
      float ms = 0.f;
      cudaEventSynchronize(pr.second);
      cudaEventElapsedTime(&ms, pr.first, pr.second);
      if (which == 0) { ctx->acc_rate_ms += ms; ++ctx->n_rate; }
      else { ctx->acc_grad_ms += ms; ++ctx->n_grad; }
      ctx->ev_pool.push_back(pr.first);
      ctx->ev_pool.push_back(pr.second);
    }
    v.clear();
  }
}

template <int D>
struct PassD {
  static int run(hawkes_ctx* ctx, int pass, int rank) {
    if (ctx->rec32) return run32(ctx, pass, rank);
    PassArgs a;
    a.rec = ctx->rec;
    a.gid = ctx->gid;
    a.items = pass == 1 ? ctx->d_items1[rank] : ctx->d_items2[rank];
    a.counter = ctx->counters + 4 * rank + (pass - 1);
    a.part = pass == 1 ? ctx->part1 : ctx->part2;
    a.tab = ctx->tab;
    a.npad = ctx->npad;
    a.N = (int)ctx->N;
    a.n_items = ctx->n_items[rank];
    a.chunk = ctx->chunk;
    a.c = ctx->pc;
    record_start(ctx, pass == 1);
    if (a.n_items > 0) {
      const size_t sm = pass_smem<D, 1>();
      const int grid = std::min(pass == 1 ? ctx->grid1 : ctx->grid2, a.n_items);
      if (pass == 1)
        pass_kernel<D, 1, R_ROWS><<<grid, THREADS, sm, ctx->stream>>>(a);
      else
        pass_kernel<D, 2, R_ROWS><<<grid, THREADS, sm, ctx->stream>>>(a);
      CHECK_LAUNCH();
    }
    if constexpr (D <= SYM_MAX_D) if (ctx->pairs && ctx->n_sym[rank] > 0) {
      SymArgs b;
      b.rec = ctx->rec;
      b.gid = ctx->gid;
      b.items = ctx->d_sym[rank];
      b.counter = ctx->counters + 4 * rank + 2 + (pass - 1);
      b.part = pass == 1 ? ctx->part1 : ctx->part2;
      b.tab = ctx->tab;
      b.npad = ctx->npad;
      b.N = (int)ctx->N;
      b.n_items = ctx->n_sym[rank];
      b.chunk = ctx->chunk;
      b.nchunks = ctx->nchunks;
      b.c = ctx->pc;
      TRY(sym_call<D>(ctx, pass, &b));
    }
    record_stop(ctx, pass == 1);
    return HAWKES_OK;
  }
  static int run32(hawkes_ctx* ctx, int pass, int rank) {
    PassArgs32 a;
    a.rec = ctx->rec32;
    a.gid = ctx->gid;
    a.items = pass == 1 ? ctx->d_items1[rank] : ctx->d_items2[rank];
    a.counter = ctx->counters + 4 * rank + (pass - 1);
    a.part = pass == 1 ? ctx->part1 : ctx->part2;
    a.npad = ctx->npad;
    a.N = (int)ctx->N;
    a.n_items = ctx->n_items[rank];
    a.chunk = ctx->chunk;
    a.c = ctx->pc32;
    record_start(ctx, pass == 1);
    if (a.n_items > 0) {
      const size_t sm = pass_smem32<D>();
      const int grid = std::min(pass == 1 ? ctx->grid1 : ctx->grid2, a.n_items);
      if (pass == 1)
        pass_kernel_f32<D, 1, R_ROWS><<<grid, THREADS, sm, ctx->stream>>>(a);
      else
        pass_kernel_f32<D, 2, R_ROWS><<<grid, THREADS, sm, ctx->stream>>>(a);
      CHECK_LAUNCH();
    }
    if constexpr (D <= SYM_MAX_D) if (ctx->pairs && ctx->n_sym[rank] > 0) {
      SymArgs32 b;
      b.rec = ctx->rec32;
      b.gid = ctx->gid;
      b.items = ctx->d_sym[rank];
      b.counter = ctx->counters + 4 * rank + 2 + (pass - 1);
      b.part = pass == 1 ? ctx->part1 : ctx->part2;
      b.npad = ctx->npad;
      b.N = (int)ctx->N;
      b.n_items = ctx->n_sym[rank];
      b.chunk = ctx->chunk;
      b.nchunks = ctx->nchunks;
      b.c = ctx->pc32;
      bool soa = true;
      if constexpr (D == 2) soa = sym32_soa();
      int rc = HAWKES_OK;
      if (soa)
        rc = sym32_launch<D, true>(ctx, pass, b);
      else if constexpr (D == 2)
        rc = sym32_launch<D, false>(ctx, pass, b);
      if (rc != HAWKES_OK) return rc;
    }
    record_stop(ctx, pass == 1);
    return HAWKES_OK;
  }
};

template <int D>
struct Fin1D {
  // ROWS: this rank's row tiles from the chunk partials.  PAIRS: every row, from the chunk
  // partials (W == 1) or from the exchanged per-event sums (W > 1).
  static int run(hawkes_ctx* ctx, int rank) {
    const bool all = ctx->pairs;
    const int nt = all ? ctx->ntiles : (int)ctx->tiles_of[rank].size();
    if (!nt) return HAWKES_OK;
    const bool sums = all && ctx->multi;
    const bool final_here = all || !ctx->multi;   // else rho' is exchanged first
    k_fin1<D><<<nt, FIN_THREADS, 0, ctx->stream>>>(
        sums ? ctx->sums1 : ctx->part1, ctx->npad, sums ? 1 : ctx->nslots,
        all ? ctx->d_every_tile : ctx->d_tiles[rank], (int)ctx->N, ctx->rec, ctx->G1, ctx->rl,
        ctx->rates, &ctx->d_consts->fc,
        final_here && !ctx->rec32 ? ctx->rec + Layout<D>::RHO : nullptr,
        final_here && ctx->rec32 ? ctx->rec32 + Layout32<D>::RHO : nullptr);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

template <int D>
struct Fin2D {
  static int run(hawkes_ctx* ctx, int rank) {
    const bool all = ctx->pairs;
    const int nt = all ? ctx->ntiles : (int)ctx->tiles_of[rank].size();
    if (!nt) return HAWKES_OK;
    const bool sums = all && ctx->multi;
    k_fin2<D><<<nt, FIN_THREADS, 0, ctx->stream>>>(
        sums ? ctx->sums2 : ctx->part2, ctx->npad, sums ? 1 : ctx->nslots,
        all ? ctx->d_every_tile : ctx->d_tiles[rank], (int)ctx->N, ctx->G1, ctx->rl, ctx->grad);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

template <int D>
struct RhoD {
  static int run(hawkes_ctx* ctx) {
    const int n = (int)ctx->N;
    k_rho_to_rec<D><<<(n + 255) / 256, 256, 0, ctx->stream>>>(ctx->rec, ctx->rec32, ctx->rl, n);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

template <int D>
struct PackXD {
  static int run(hawkes_ctx* ctx, const double* xdev) {
    k_pack_x<D><<<(ctx->npad + 255) / 256, 256, 0, ctx->stream>>>(ctx->rec, xdev, (int)ctx->N,
                                                                  ctx->npad, ctx->bad);
    CHECK_LAUNCH();
    if (ctx->rec32) {
      k_pack_x32<D><<<(ctx->npad + 255) / 256, 256, 0, ctx->stream>>>(ctx->rec32, xdev,
                                                                      (int)ctx->N, ctx->npad);
      CHECK_LAUNCH();
    }
    return HAWKES_OK;
  }
};

template <int D>
struct PackTD {
  static int run(hawkes_ctx* ctx, const double* tdev) {
    k_pack_t<D><<<(ctx->npad + 255) / 256, 256, 0, ctx->stream>>>(ctx->rec, tdev, (int)ctx->N,
                                                                  ctx->npad);
    CHECK_LAUNCH();
    if (ctx->rec32) {
      k_pack_t32<D><<<(ctx->npad + 255) / 256, 256, 0, ctx->stream>>>(ctx->rec32, tdev,
                                                                      (int)ctx->N, ctx->npad);
      CHECK_LAUNCH();
    }
    return HAWKES_OK;
  }
};

template <int D>
struct MoveD {
  static int run(hawkes_ctx* ctx, int k, int decide) {
    MoveArgs<D> a;
    a.rec = ctx->rec;
    a.gid = ctx->gid;
    a.slot_of = ctx->d_slot_of;
    a.idx = ctx->d_move_idx;
    a.new_x = ctx->d_move_x;
    a.k = k;
    a.N = (int)ctx->N;
    a.c = ctx->pc;
    a.tab = ctx->tab;
    // one launch for the rows outside S and the moved rows, one for the terms and their
    // fixed-order sum (decide: the MH sweep's Metropolis decision in the same kernel)
    const int nb = (int)((ctx->N + 255) / 256);
    const int len = move_split_len((int)ctx->N);
    const int nsplit = (int)((ctx->N + len - 1) / len);
    k_move_delta_rows<D><<<(unsigned)(nb + k * nsplit), 256, move_smem_bytes<D>(k), ctx->stream>>>(
        a, ctx->tab, ctx->d_move_delta, ctx->d_move_rows_part, nb, nsplit);
    CHECK_LAUNCH();
    k_move_terms_final<<<nb, 256, 0, ctx->stream>>>(ctx->rates, ctx->d_move_delta, ctx->d_move_rows_part,
                                                    nsplit, ctx->d_slot_of, (int)ctx->N, ctx->fc.tx2,
                                                    ctx->fc.h2, ctx->fc.zero_floor, ctx->d_move_part,
                                                    ctx->d_move_rows, ctx->st, decide, ctx->d_mh_acc,
                                                    ctx->d_mh_la);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

template <int D>
struct CommitD {
  static int run(hawkes_ctx* ctx, int k, int gated) {
    const int n = (int)std::max<int64_t>(ctx->N, k);
    k_move_commit<D><<<(n + 255) / 256, 256, 0, ctx->stream>>>(
        ctx->rates, ctx->d_move_delta, ctx->d_move_rows, ctx->d_slot_of, ctx->d_move_idx,
        ctx->d_move_x, k, (int)ctx->N, ctx->fc.tx2, ctx->fc.h2, ctx->rec, ctx->rec32,
        ctx->xstage, ctx->st, gated);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

template <int D>
struct MhProposeD {
  static int run(hawkes_ctx* ctx, int k) {
    k_mh_propose<D><<<1, 256, 0, ctx->stream>>>(ctx->d_mh_blocks, k, ctx->xstage, ctx->d_reg_c,
                                               ctx->d_reg_s, ctx->reg_kind, ctx->d_move_idx,
                                               ctx->d_move_x, ctx->d_slot_of, ctx->st);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

// the whole sweep as one cooperative launch (hawkes_mh_coop.cuh)
template <int D>
struct MhCoopD {
  static int run(hawkes_ctx* ctx, int n_blocks, int k) {
    const int N = (int)ctx->N;
    const int len = move_split_len(N);
    MhCoopArgs<D> a;
    a.rec = ctx->rec;
    a.rec32 = ctx->rec32;
    a.gid = ctx->gid;
    a.blocks = ctx->d_mh_blocks;
    a.n_blocks = n_blocks;
    a.k = k;
    a.N = N;
    a.nsplit = (N + len - 1) / len;
    a.centre = ctx->d_reg_c;
    a.size = ctx->d_reg_s;
    a.kind = ctx->reg_kind;
    a.xcur = ctx->xstage;
    a.rates = ctx->rates;
    a.delta = ctx->d_move_delta;
    a.rows_part = ctx->d_move_rows_part;
    a.part = ctx->d_move_part;
    a.rows = ctx->d_move_rows;
    a.stamp = ctx->d_mh_stamp;
    a.gtab = ctx->tab;
    a.c = ctx->pc;
    a.tx2 = ctx->fc.tx2;
    a.h2 = ctx->fc.h2;
    a.floor_ = ctx->fc.zero_floor;
    a.st = ctx->st;
    a.acc_out = ctx->d_mh_acc;
    a.la_out = ctx->d_mh_la;
    const size_t smem = mh_coop_smem<D>(k);
    auto kern = k_mh_sweep_coop<D>;
    CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mh_coop_smem<D>(MOVE_MAX)));
    int per_sm = 0;
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    if (per_sm < 1) return set_err(ctx, HAWKES_ERR_CUDA, "cooperative MH sweep does not fit on an SM");
    const int nb = (N + 255) / 256;
    const char* e = getenv("HAWKES_MH_COOP_CTAS");   // diagnostics: CTAs per SM
    const int want = e ? std::max(1, atoi(e)) : per_sm;
    const int grid = std::max(1, std::min(std::min(want, per_sm) * ctx->sms, nb + k * a.nsplit));
    void* args[] = {&a};
    CU(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(256), args, smem, ctx->stream));
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

template <int D>
struct BmdsD {
  // default: the unordered-pair kernel (each pair once); HAWKES_BMDS_SYM=0 selects the
  // per-row kernel (each ordered pair; diagnostics, A/B)
  static int run(hawkes_ctx* ctx, const double* x) {
    const char* e = getenv("HAWKES_BMDS_SYM");
    if (ctx->d_bpart && !(e && atoi(e) == 0)) {
      const int N = (int)ctx->N;
      const long long NB = (N + 31) / 32;
      const size_t smem = bmds_sym_smem<D>();
      auto kern = k_bmds_sym<D>;
      CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * BSYM_WARPS, smem));
      const long long ntasks = NB * (NB + 1) / 2;
      const long long want = (ntasks + BSYM_WARPS - 1) / BSYM_WARPS;
      const int grid = (int)std::max(1LL, std::min<long long>((long long)std::max(1, per_sm) * ctx->sms, want));
      kern<<<grid, 32 * BSYM_WARPS, smem, ctx->stream>>>(x, ctx->d_Y, N, ctx->bc, ctx->tab, ctx->d_bpart, ntasks);
      CHECK_LAUNCH();
      k_bmds_sym_fin<D><<<(N + 255) / 256, 256, 0, ctx->stream>>>(ctx->d_bpart, N, ctx->d_bgrad, ctx->d_brow);
      CHECK_LAUNCH();
    } else {
      k_bmds<D><<<(unsigned)ctx->N, BMDS_THREADS, 0, ctx->stream>>>(x, ctx->d_Y, (int)ctx->N, ctx->bc,
                                                                     ctx->tab, ctx->d_bgrad, ctx->d_brow);
      CHECK_LAUNCH();
    }
    k_sum_partials<<<1, 1024, 0, ctx->stream>>>(ctx->d_brow, (int)ctx->N, &ctx->st->bmds);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
};

template <int D>
struct DriftD {
  static int run(hawkes_ctx* ctx, double eps, bool box, bool minv) {
    const int n = (int)ctx->N;
    k_drift<D><<<(n + 255) / 256, 256, 0, ctx->stream>>>(
        ctx->lf_x, ctx->lf_p, minv ? ctx->lf_minv : nullptr, box ? ctx->lf_lo : nullptr,
        box ? ctx->lf_hi : nullptr, n, eps, ctx->bad);
    CHECK_LAUNCH();
    return dispatchD<PackXD>(D, ctx, (const double*)ctx->lf_x);
  }
};

// Exchange K values per row: own rows of every logical rank -> all rows everywhere.
int exchange_rows(hawkes_ctx* ctx, double* rows, int K) {
  if (!ctx->multi) return HAWKES_OK;
  const long long per_rank = (long long)ctx->max_tiles * RT * K;
  for (int r : ctx->my_ranks) {
    const int nt = (int)ctx->tiles_of[r].size();
    const long long tot = (long long)nt * RT * K;
    if (tot == 0) continue;
    // with a real communicator the rank packs into its send buffer; emulated ranks pack
    // directly into their slot of the gather buffer (the loop-back "allgather")
    double* dst = ctx->comm ? ctx->sendbuf : ctx->recvbuf + r * per_rank;
    k_pack_rows<<<(unsigned)((tot + 255) / 256), 256, 0, ctx->stream>>>(rows, K, ctx->d_tiles[r], nt,
                                                                       (int)ctx->N, dst);
    CHECK_LAUNCH();
  }
  if (ctx->comm) {
    // zero the tail of the send buffer beyond this rank's rows (fixed message size)
    const int r = ctx->my_ranks[0];
    const long long tot = (long long)ctx->tiles_of[r].size() * RT * K;
    if (tot < per_rank)
      CU(cudaMemsetAsync(ctx->sendbuf + tot, 0, (per_rank - tot) * sizeof(double), ctx->stream));
    NC(g_nccl.allGather(ctx->sendbuf, ctx->recvbuf, (size_t)per_rank, ncclDouble, ctx->comm,
                        ctx->stream));
  }
  const long long all = per_rank * ctx->W;
  k_unpack_rows<<<(unsigned)((all + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->recvbuf, K, ctx->d_all_tiles, ctx->max_tiles, ctx->W, (int)ctx->N, rows);
  CHECK_LAUNCH();
  return HAWKES_OK;
}

// rate pass + finalize + exchange + ell reduction (device-side; no host sync)
// PAIRS, W > 1: per-event sums over this process's chunk pairs, then the exchange
// (NCCL allreduce, or the rank-ordered sum of the emulated ranks' buffers)
int reduce_pair_partials(hawkes_ctx* ctx, const double* part, double* sums, int K) {
  const long long n = (long long)ctx->N * K;
  const long long stride = (long long)ctx->npad * K;
  for (int r : ctx->my_ranks) {
    double* out = ctx->comm ? sums : sums + (1 + r) * stride;
    k_slot_sum<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
        part, ctx->npad, ctx->nchunks, ctx->chunk, K, ctx->d_own, r, (int)ctx->N, out);
    CHECK_LAUNCH();
  }
  if (ctx->comm) {
    NC(g_nccl.allReduce(sums, sums, (size_t)n, ncclDouble, ncclSum, ctx->comm, ctx->stream));
  } else {
    k_sum_ranks<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(sums + stride, stride, ctx->W,
                                                                     n, sums);
    CHECK_LAUNCH();
  }
  return HAWKES_OK;
}

int run_rates(hawkes_ctx* ctx);
int run_grad(hawkes_ctx* ctx);

// Graphs bake the kernel constants in (they are kernel parameters, so the FP64 instructions
// read them from the constant bank); set_params / set_times drop the graphs, and a graph is
// captured only at the second evaluation with unchanged constants, so MCMC moves that
// change Theta every step never pay for a capture.
bool use_graph(const hawkes_ctx* ctx) {
  return ctx->graphs && !ctx->timing && !ctx->capturing && ctx->evals_same_consts >= 2;
}

void drop_mh_graph(hawkes_ctx* ctx) {
  if (ctx->mh_gexec) cudaGraphExecDestroy(ctx->mh_gexec);
  ctx->mh_gexec = nullptr;
  ctx->mh_gk = 0;
}

void drop_graphs(hawkes_ctx* ctx) {
  for (auto& ge : ctx->gexec)
    if (ge) {
      cudaGraphExecDestroy(ge);
      ge = nullptr;
    }
  ctx->evals_same_consts = 0;
  drop_mh_graph(ctx);   // its launches carry the folded constants by value
}

// Capture one evaluation sequence (0: rate pass; 1: rate + gradient pass; 2: gradient pass
// with cached rates) on the context's own stream and instantiate it.
int capture(hawkes_ctx* ctx, int which) {
  cudaStream_t user = ctx->stream;
  const bool rv = ctx->rates_valid, gv = ctx->grad_valid;
  const int64_t l0 = ctx->launches;
  ctx->stream = ctx->gstream;
  ctx->capturing = true;
  int rc = HAWKES_OK;
  cudaError_t e = cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal);
  if (e == cudaSuccess) {
    ctx->rates_valid = which == 2;
    ctx->grad_valid = false;
    rc = which == 0 ? run_rates(ctx) : run_grad(ctx);
  }
  cudaGraph_t g = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(ctx->gstream, &g);
  ctx->stream = user;
  ctx->capturing = false;
  ctx->rates_valid = rv;
  ctx->grad_valid = gv;
  if (rc != HAWKES_OK) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess || e2 != cudaSuccess)
    return set_err(ctx, HAWKES_ERR_CUDA, "graph capture failed: %s",
                   cudaGetErrorString(e != cudaSuccess ? e : e2));
  cudaError_t e3 = cudaGraphInstantiate(&ctx->gexec[which], g, 0);
  cudaGraphDestroy(g);
  if (e3 != cudaSuccess)
    return set_err(ctx, HAWKES_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e3));
  ctx->graph_launches[which] = ctx->launches - l0;
  ctx->launches = l0;
  return HAWKES_OK;
}

int replay(hawkes_ctx* ctx, int which) {
  if (!ctx->gexec[which]) TRY(capture(ctx, which));
  CU(cudaEventRecord(ctx->ev_in, ctx->stream));
  CU(cudaStreamWaitEvent(ctx->gstream, ctx->ev_in, 0));
  CU(cudaGraphLaunch(ctx->gexec[which], ctx->gstream));
  CU(cudaEventRecord(ctx->ev_out, ctx->gstream));
  CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_out, 0));
  ctx->launches += ctx->graph_launches[which];
  return HAWKES_OK;
}

int run_rates(hawkes_ctx* ctx) {
  if (ctx->rates_valid) return HAWKES_OK;
  if (!ctx->capturing) ++ctx->evals_same_consts;
  if (use_graph(ctx)) {
    TRY(replay(ctx, 0));
    ctx->rates_valid = true;
    ctx->rates_exchanged = false;
    ctx->grad_valid = false;
    ctx->lam_valid = true;
    return HAWKES_OK;
  }
  CU(cudaMemsetAsync(ctx->counters, 0, sizeof(int) * 4 * ctx->W, ctx->stream));
  if (ctx->pairs) {
    for (int r : ctx->my_ranks) TRY(dispatchD<PassD>(ctx->D, ctx, 1, r));
    if (ctx->multi) TRY(reduce_pair_partials(ctx, ctx->part1, ctx->sums1, K1_of(ctx->D)));
    TRY(dispatchD<Fin1D>(ctx->D, ctx, 0));
  } else {
    for (int r : ctx->my_ranks) {
      TRY(dispatchD<PassD>(ctx->D, ctx, 1, r));
      TRY(dispatchD<Fin1D>(ctx->D, ctx, r));
    }
    TRY(exchange_rows(ctx, ctx->rl, 2));
    if (ctx->multi) TRY(dispatchD<RhoD>(ctx->D, ctx));
  }
  k_ell_reduce<<<1, 1024, 0, ctx->stream>>>(ctx->rl, (int)ctx->N, ctx->st);
  CHECK_LAUNCH();
  ctx->rates_valid = true;
  ctx->rates_exchanged = false;
  ctx->grad_valid = false;
  ctx->lam_valid = true;
  return HAWKES_OK;
}

int run_grad(hawkes_ctx* ctx) {
  if (ctx->grad_valid) return HAWKES_OK;
  if (!ctx->capturing && !ctx->rates_valid) ++ctx->evals_same_consts;
  if (use_graph(ctx)) {
    TRY(replay(ctx, ctx->rates_valid ? 2 : 1));
    if (!ctx->rates_valid) ctx->rates_exchanged = false;
    ctx->rates_valid = ctx->grad_valid = true;
    ctx->lam_valid = true;
    return HAWKES_OK;
  }
  TRY(run_rates(ctx));
  if (ctx->pairs) {
    for (int r : ctx->my_ranks) TRY(dispatchD<PassD>(ctx->D, ctx, 2, r));
    if (ctx->multi) TRY(reduce_pair_partials(ctx, ctx->part2, ctx->sums2, K2_of(ctx->D)));
    TRY(dispatchD<Fin2D>(ctx->D, ctx, 0));
  } else {
    for (int r : ctx->my_ranks) {
      TRY(dispatchD<PassD>(ctx->D, ctx, 2, r));
      TRY(dispatchD<Fin2D>(ctx->D, ctx, r));
    }
    TRY(exchange_rows(ctx, ctx->grad, ctx->D));
  }
  ctx->grad_valid = true;
  return HAWKES_OK;
}

int fetch_status(hawkes_ctx* ctx) {
  CU(cudaMemcpyAsync(ctx->h_st, ctx->st, sizeof(EvalStatus), cudaMemcpyDeviceToHost, ctx->stream));
  int bad = 0;
  CU(cudaMemcpyAsync(&ctx->h_st->nonfinite, ctx->bad, sizeof(int), cudaMemcpyDeviceToHost,
                     ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  bad = ctx->h_st->nonfinite;
  if (bad) {
    CU(cudaMemsetAsync(ctx->bad, 0, sizeof(int), ctx->stream));
    if (bad & 2) {
      ctx->have_bmds = false;
      return set_err(ctx, HAWKES_ERR_NONFINITE,
                     "BMDS dissimilarities must be finite and > 0 below the diagonal");
    }
    ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
    ctx->have_x = false;
    return set_err(ctx, HAWKES_ERR_NONFINITE,
                   "locations contain NaN/Inf or |x| > 1e100 (device-side validation)");
  }
  return HAWKES_OK;
}

// drop a pending block move (restores the event -> proposal-slot map)
int clear_move(hawkes_ctx* ctx) {
  if (ctx->move_k > 0) {
    k_scatter_slots<<<(ctx->move_k + 255) / 256, 256, 0, ctx->stream>>>(ctx->d_slot_of, ctx->d_move_idx,
                                                                        ctx->move_k, 0);
    CHECK_LAUNCH();
    ctx->move_k = 0;
  }
  return HAWKES_OK;
}

int check_ready(hawkes_ctx* ctx) {
  if (!ctx->have_t || !ctx->have_x || !ctx->have_p)
    return set_err(ctx, HAWKES_ERR_STATE, "set_times, set_locations and set_params are all required");
  return HAWKES_OK;
}

void build_plan_pairs(hawkes_ctx* ctx, std::vector<std::vector<int2>>& it1,
                      std::vector<std::vector<int2>>& it2, std::vector<std::vector<int2>>& sym,
                      std::vector<int>& own) {
  const int W = ctx->W, C = ctx->nchunks, N = (int)ctx->N;
  own = pair_owners(N, ctx->chunk, W);
  ctx->tiles_of.assign(W, {});
  ctx->max_tiles = 0;
  it1.assign(W, {});
  it2.assign(W, {});
  sym.assign(W, {});
  for (int r = 0; r < W; ++r) {
    std::vector<std::pair<double, int2>> items;   // (pair count, (a, b)); heaviest first
    for (int a = 0; a < C; ++a)
      for (int b = a; b < C; ++b) {
        if (own[(size_t)a * C + b] != r) continue;
        const double na = (double)std::min<long long>(ctx->chunk, (long long)N - (long long)a * ctx->chunk);
        const double nb = (double)std::min<long long>(ctx->chunk, (long long)N - (long long)b * ctx->chunk);
        items.push_back({a == b ? 0.5 * na * na : na * nb, make_int2(a, b)});
      }
    std::stable_sort(items.begin(), items.end(),
                     [](const std::pair<double, int2>& x, const std::pair<double, int2>& y) {
                       return x.first > y.first;
                     });
    for (auto& e : items) sym[r].push_back(e.second);
  }
}

void build_plan(hawkes_ctx* ctx, std::vector<std::vector<int2>>& it1,
                std::vector<std::vector<int2>>& it2) {
  const int W = ctx->W;
  ctx->tiles_of.assign(W, {});
  for (int k = 0; k < ctx->ntiles; ++k) ctx->tiles_of[owner_of_tile(k, W)].push_back(k);
  ctx->max_tiles = 0;
  for (auto& v : ctx->tiles_of) ctx->max_tiles = std::max<int>(ctx->max_tiles, (int)v.size());
  it1.assign(W, {});
  it2.assign(W, {});
  const int N = (int)ctx->N;
  for (int r = 0; r < W; ++r) {
    std::vector<std::pair<long long, int2>> c1, c2;
    for (int tile : ctx->tiles_of[r]) {
      const int row0 = tile * RT, row1 = std::min(N, row0 + RT);
      for (int ck = 0; ck < ctx->nchunks; ++ck) {
        long long w1 = 0, w2 = 0;
        const int j0 = ck * ctx->chunk, j1 = std::min(N, j0 + ctx->chunk);
        for (int jt = j0; jt < j1; jt += TILE_J) {
          const int je = std::min(j1, jt + TILE_J) - 1;
          const long long n = (long long)(je - jt + 1);
          if (je < row0) { w1 += 33 * n; w2 += 20 * n; }        // earlier: pass1 both exps
          else if (jt > row1 - 1) { w1 += 20 * n; w2 += 32 * n; } // later: pass2 both exps
          else { w1 += 40 * n; w2 += 40 * n; }
        }
        c1.push_back({w1, make_int2(tile, ck)});
        c2.push_back({w2, make_int2(tile, ck)});
      }
    }
    auto cmp = [](const std::pair<long long, int2>& a, const std::pair<long long, int2>& b) {
      return a.first > b.first;
    };
    std::stable_sort(c1.begin(), c1.end(), cmp);
    std::stable_sort(c2.begin(), c2.end(), cmp);
    for (auto& e : c1) it1[r].push_back(e.second);
    for (auto& e : c2) it2[r].push_back(e.second);
  }
}

void drop_graphs(hawkes_ctx* ctx);

int upload_consts(hawkes_ctx* ctx) {
  drop_graphs(ctx);
  DevConsts h;
  h.pc = ctx->pc;
  h.pc32 = ctx->pc32;
  h.fc = ctx->fc;
  CU(cudaMemcpyAsync(ctx->d_consts, &h, sizeof h, cudaMemcpyHostToDevice, ctx->stream));
  return HAWKES_OK;
}

// Kernel constants for Theta; written to ctx only when every check passes.
int compute_constants(hawkes_ctx* ctx, const hawkes_params& p, double tN) {
  const int D = ctx->D;
  const double two_pi = 6.283185307179586476925286766559;
  // background weight mu0/((2pi)^{D/2} tau_x^D * sqrt(2pi) tau_t), times alpha = 1/tau_x^2
  const double lnw_b = log(p.mu0) - 0.5 * (D + 1) * log(two_pi) - D * log(p.tau_x) - log(p.tau_t) -
                       2.0 * log(p.tau_x);
  // self-excitation weight theta omega/((2pi)^{D/2} h^D), times beta = 1/h^2
  const double lnw_s = log(p.theta) + log(p.omega) - 0.5 * D * log(two_pi) - D * log(p.sigma_x) -
                       2.0 * log(p.sigma_x);
  if ((p.mu0 > 0 && !(fabs(lnw_b) < 600.0)) || (p.theta > 0 && !(fabs(lnw_s) < 600.0)))
    return set_err(ctx, HAWKES_ERR_PARAM,
                   "Theta puts the kernel constants outside the fp64 exp range (|log w| >= 600)");
  PassConst pc;
  pc.kx = -0.5 / (p.tau_x * p.tau_x);
  pc.kt = -0.5 / (p.tau_t * p.tau_t);
  pc.ks = -0.5 / (p.sigma_x * p.sigma_x);
  pc.omega = p.omega;
  pc.lnc_b = p.mu0 > 0 ? lnw_b + 64.0 * LN2 : -INFINITY;
  pc.lnc_s = p.theta > 0 ? lnw_s + 64.0 * LN2 : -INFINITY;
  if (!isfinite(pc.kx) || !isfinite(pc.kt) || !isfinite(pc.ks))
    return set_err(ctx, HAWKES_ERR_PARAM, "bandwidths too small for fp64");
  FinConst fc;
  fc.tx2 = p.tau_x * p.tau_x;
  fc.h2 = p.sigma_x * p.sigma_x;
  fc.mu0 = p.mu0;
  fc.tau_t = p.tau_t;
  fc.theta = p.theta;
  fc.omega = p.omega;
  fc.tN = tN;
  fc.scale_log2 = -64.0;
  // every clamped pair term is <= e^-706.9 in the kernels' scaled units
  fc.zero_floor = (double)ctx->N * exp(-700.0) * std::max(fc.tx2, fc.h2);
  if (ctx->opts.precision == HAWKES_FP32) {
    // log2 domain; one power-of-two scale 2^-E puts the largest possible term near 2^20
    const double L2E = 1.4426950408889634074;
    const double l2b = p.mu0 > 0 ? lnw_b * L2E : -INFINITY;
    const double l2s = p.theta > 0 ? lnw_s * L2E : -INFINITY;
    const double E = floor(std::max(l2b, l2s)) - 20.0;
    PassConst32 c32;
    c32.kx = (float)(pc.kx * L2E);
    c32.kt = (float)(pc.kt * L2E);
    c32.ks = (float)(pc.ks * L2E);
    c32.omega = (float)(p.omega * L2E);
    c32.cb = (float)(l2b - E);
    c32.cs = (float)(l2s - E);
    if (!isfinite(c32.kx) || !isfinite(c32.kt) || !isfinite(c32.ks) || !isfinite(c32.omega) ||
        c32.kx == 0.f || c32.kt == 0.f || c32.ks == 0.f)
      return set_err(ctx, HAWKES_ERR_PARAM, "Theta outside the fp32 path's range");
    fc.scale_log2 = E;
    fc.zero_floor = 0.0;   // ex2.approx.ftz flushes to exact zeros
    ctx->pc32 = c32;
  }
  ctx->pc = pc;
  ctx->fc = fc;
  return upload_consts(ctx);
}

int copy_in(hawkes_ctx* ctx, double* dst, const double* src, size_t n, int mem) {
  CU(cudaMemcpyAsync(dst, src, n * sizeof(double),
                     mem == HAWKES_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     ctx->stream));
  return HAWKES_OK;
}
int copy_out(hawkes_ctx* ctx, double* dst, const double* src, size_t n, int mem) {
  CU(cudaMemcpyAsync(dst, src, n * sizeof(double),
                     mem == HAWKES_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     ctx->stream));
  return HAWKES_OK;
}

bool finite_bounded(double v) { return fabs(v) <= 1e100; }

// fexp's table: T[j] = 2^(j/EXP_TABLE) as (low word, high word - (j << EXP_BIAS_SHIFT))
// (the bias lets one integer multiply-add insert the binary exponent; hawkes_kernels.cuh)
void make_exp_table(int2* h) {
  for (int j = 0; j < EXP_TABLE; ++j) {
    const double v = (double)exp2l((long double)j / (long double)EXP_TABLE);
    long long b;
    memcpy(&b, &v, 8);
    h[j] = make_int2((int)(b & 0xffffffffLL), (int)(b >> 32) - (j << EXP_BIAS_SHIFT));
  }
}

}  // namespace

// ========================================================================== ABI
extern "C" {

int hawkes_abi_version(void) { return HAWKES_ABI_VERSION; }

int hawkes_default_opts(hawkes_opts* o) {
  if (!o) return HAWKES_ERR_ARG;
  memset(o, 0, sizeof *o);
  o->world = 1;
  return HAWKES_OK;
}

const char* hawkes_last_error(const hawkes_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

int hawkes_create(int64_t N, int32_t D, const hawkes_opts* opts_in, hawkes_ctx** out) {
  hawkes_ctx* ctx = nullptr;
  if (!out) return set_err(nullptr, HAWKES_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (N < 1 || N > (1LL << 30)) return set_err(nullptr, HAWKES_ERR_ARG, "N must be in [1, 2^30]");
  if (D < 1 || D > HAWKES_MAX_D) return set_err(nullptr, HAWKES_ERR_DIM, "D must be in [1, %d]", HAWKES_MAX_D);
  hawkes_opts o;
  hawkes_default_opts(&o);
  if (opts_in) o = *opts_in;
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world)
    return set_err(nullptr, HAWKES_ERR_ARG, "bad rank/world");
  if (o.precision != HAWKES_FP64 && o.precision != HAWKES_FP32)
    return set_err(nullptr, HAWKES_ERR_ARG, "bad precision");
  if (o.world > 1 && !o.nccl_unique_id)
    return set_err(nullptr, HAWKES_ERR_ARG, "world > 1 needs nccl_unique_id");
  if ((o.world > 1 || o.nccl_unique_id) && o.emulate_world > 1)
    return set_err(nullptr, HAWKES_ERR_ARG, "emulate_world needs world == 1 and no NCCL id");

  ctx = new hawkes_ctx();
  ctx->N = N;
  ctx->D = D;
  ctx->opts = o;
  ctx->stream = (cudaStream_t)o.cuda_stream;
  {
    cudaError_t e = cudaSetDevice(o.device);
    if (e != cudaSuccess) {
      set_err(nullptr, HAWKES_ERR_CUDA, "cudaSetDevice(%d): %s", o.device, cudaGetErrorString(e));
      delete ctx;
      return HAWKES_ERR_CUDA;
    }
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, o.device);
    if (e != cudaSuccess || prop.major != 10) {
      set_err(nullptr, HAWKES_ERR_CUDA, "device %d is not sm_100 (%s)", o.device,
              e == cudaSuccess ? prop.name : cudaGetErrorString(e));
      delete ctx;
      return HAWKES_ERR_CUDA;
    }
    ctx->sms = prop.multiProcessorCount;
    ctx->coop_ok = prop.cooperativeLaunch != 0;
  }
  auto fail = [&](int rc) {
    if (!ctx->err.empty()) g_create_error = ctx->err;
    hawkes_destroy(ctx);
    return rc;
  };
  ctx->ntiles = (int)((N + RT - 1) / RT);
  ctx->npad = ctx->ntiles * RT;
  if (o.algorithm < HAWKES_ALGO_AUTO || o.algorithm > HAWKES_ALGO_PAIRS) {
    delete ctx;
    return set_err(nullptr, HAWKES_ERR_ARG, "bad algorithm");
  }
  if (o.algorithm == HAWKES_ALGO_PAIRS && D > SYM_MAX_D) {
    delete ctx;
    return set_err(nullptr, HAWKES_ERR_ARG, "HAWKES_ALGO_PAIRS supports D <= %d", SYM_MAX_D);
  }
  ctx->pairs = o.algorithm == HAWKES_ALGO_PAIRS || (o.algorithm == HAWKES_ALGO_AUTO && D <= SYM_AUTO_MAX_D);
  ctx->chunk = ctx->pairs ? chunk_pairs_of(N, o.world > 1 ? o.world : std::max(1, o.emulate_world))
                           : chunk_of(N);
  ctx->nchunks = (int)((N + ctx->chunk - 1) / ctx->chunk);
  ctx->nslots = ctx->nchunks + (ctx->pairs ? 1 : 0);   // PAIRS: + diagonal column slot
  ctx->W = o.world > 1 ? o.world : std::max(1, o.emulate_world);
  // an NCCL id with world == 1 builds a one-rank communicator and runs the sharded path
  // (exchanges included) on one GPU: the NCCL plumbing's single-GPU test
  ctx->multi = ctx->W > 1 || o.nccl_unique_id != nullptr;
  if (o.world > 1)
    ctx->my_ranks = {o.rank};
  else
    for (int r = 0; r < ctx->W; ++r) ctx->my_ranks.push_back(r);

  std::vector<std::vector<int2>> it1, it2, sym;
  std::vector<int> own;
  if (ctx->pairs)
    build_plan_pairs(ctx, it1, it2, sym, own);
  else
    build_plan(ctx, it1, it2);

  const int REC = REC_of(D);
  int rc;
  if ((rc = dalloc(ctx, &ctx->rec, (size_t)ctx->npad * REC)) ||
      (rc = dalloc(ctx, &ctx->gid, (size_t)ctx->npad)) ||
      (rc = dalloc(ctx, &ctx->part1, (size_t)ctx->nslots * ctx->npad * K1_of(D))) ||
      (rc = dalloc(ctx, &ctx->part2, (size_t)ctx->nslots * ctx->npad * K2_of(D))) ||
      (rc = dalloc(ctx, &ctx->G1, (size_t)ctx->npad * D)) ||
      (rc = dalloc(ctx, &ctx->rl, (size_t)ctx->npad * 2)) ||
      (rc = dalloc(ctx, &ctx->rates, (size_t)ctx->npad * 4)) ||
      (rc = dalloc(ctx, &ctx->grad, (size_t)ctx->npad * D)) ||
      (rc = dalloc(ctx, &ctx->xstage, (size_t)N * D)) ||
      (rc = dalloc(ctx, &ctx->counters, (size_t)4 * ctx->W)) ||
      (rc = dalloc(ctx, &ctx->tab, EXP_TABLE)) || (rc = dalloc(ctx, &ctx->bad, 1)) ||
      (rc = dalloc(ctx, &ctx->st, 1)) || (rc = dalloc(ctx, &ctx->d_consts, 1)) ||
      (rc = dalloc(ctx, &ctx->d_slot_of, (size_t)N)) || (rc = dalloc(ctx, &ctx->d_move_idx, MOVE_MAX)) ||
      (rc = dalloc(ctx, &ctx->d_move_x, (size_t)MOVE_MAX * D)) ||
      (rc = dalloc(ctx, &ctx->d_move_delta, (size_t)ctx->npad * 2)) ||
      (rc = dalloc(ctx, &ctx->d_move_rows, (size_t)MOVE_MAX * 2)) ||
      (rc = dalloc(ctx, &ctx->d_move_part, (size_t)(N + 255) / 256)) ||
      (rc = dalloc(ctx, &ctx->d_move_rows_part, (size_t)MOVE_MAX * 2 * MOVE_NSPLIT)))
    return fail(rc);
  if (cudaMemset(ctx->d_slot_of, 0xff, (size_t)N * sizeof(int)) != cudaSuccess)
    return fail(set_err(ctx, HAWKES_ERR_CUDA, "cudaMemset failed"));
  if (!ctx->multi && !getenv("HAWKES_NO_GRAPHS")) {
    if (cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming) != cudaSuccess)
      return fail(set_err(ctx, HAWKES_ERR_CUDA, "stream/event creation failed"));
    ctx->graphs = true;
  }
  if (o.precision == HAWKES_FP32) {
    if ((rc = dalloc(ctx, &ctx->rec32, (size_t)ctx->npad * Layout32Rec(D)))) return fail(rc);
    if (cudaMemset(ctx->rec32, 0, (size_t)ctx->npad * Layout32Rec(D) * sizeof(float)) != cudaSuccess)
      return fail(set_err(ctx, HAWKES_ERR_CUDA, "cudaMemset failed"));
  }
  if (ctx->pairs) {
    std::vector<int> every(ctx->ntiles);
    for (int k = 0; k < ctx->ntiles; ++k) every[k] = k;
    if ((rc = dalloc(ctx, &ctx->d_every_tile, every.size())) ||
        (rc = dalloc(ctx, &ctx->d_own, own.size())))
      return fail(rc);
    if (cudaMemcpy(ctx->d_every_tile, every.data(), every.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->d_own, own.data(), own.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_err(ctx, HAWKES_ERR_CUDA, "copy of the pair plan failed"));
    ctx->d_sym.assign(ctx->W, nullptr);
    ctx->n_sym.assign(ctx->W, 0);
    for (int r = 0; r < ctx->W; ++r) {
      ctx->n_sym[r] = (int)sym[r].size();
      if ((rc = dalloc(ctx, &ctx->d_sym[r], sym[r].size()))) return fail(rc);
      if (!sym[r].empty() &&
          cudaMemcpy(ctx->d_sym[r], sym[r].data(), sym[r].size() * sizeof(int2), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(set_err(ctx, HAWKES_ERR_CUDA, "copy of the pair items failed"));
    }
    if (ctx->multi) {
      const size_t copies = o.nccl_unique_id ? 1 : (size_t)ctx->W + 1;
      if ((rc = dalloc(ctx, &ctx->sums1, copies * ctx->npad * K1_of(D))) ||
          (rc = dalloc(ctx, &ctx->sums2, copies * ctx->npad * K2_of(D))))
        return fail(rc);
    }
  } else if (ctx->multi) {
    const size_t per_rank = (size_t)ctx->max_tiles * RT * std::max(4, D);
    if ((rc = dalloc(ctx, &ctx->sendbuf, per_rank)) ||
        (rc = dalloc(ctx, &ctx->recvbuf, per_rank * ctx->W)))
      return fail(rc);
  }
  {
    cudaError_t e = cudaMallocHost((void**)&ctx->h_st, sizeof(EvalStatus));
    if (e != cudaSuccess) return fail(set_err(ctx, HAWKES_ERR_OOM, "cudaMallocHost failed"));
  }
  // tile lists / items
  {
    std::vector<int> all((size_t)ctx->W * std::max(1, ctx->max_tiles), -1);
    if (all.empty()) all.push_back(-1);
    for (int r = 0; r < ctx->W; ++r)
      for (size_t k = 0; k < ctx->tiles_of[r].size(); ++k) all[(size_t)r * ctx->max_tiles + k] = ctx->tiles_of[r][k];
    if ((rc = dalloc(ctx, &ctx->d_all_tiles, all.size()))) return fail(rc);
    if (cudaMemcpy(ctx->d_all_tiles, all.data(), all.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_err(ctx, HAWKES_ERR_CUDA, "copy of tile lists failed"));
    ctx->d_tiles.resize(ctx->W);
    ctx->d_items1.assign(ctx->W, nullptr);
    ctx->d_items2.assign(ctx->W, nullptr);
    ctx->n_items.assign(ctx->W, 0);
    for (int r = 0; r < ctx->W; ++r) {
      ctx->d_tiles[r] = ctx->d_all_tiles + (size_t)r * ctx->max_tiles;
      ctx->n_items[r] = (int)it1[r].size();
      if ((rc = dalloc(ctx, &ctx->d_items1[r], it1[r].size())) ||
          (rc = dalloc(ctx, &ctx->d_items2[r], it2[r].size())))
        return fail(rc);
      if (!it1[r].empty() &&
          (cudaMemcpy(ctx->d_items1[r], it1[r].data(), it1[r].size() * sizeof(int2), cudaMemcpyHostToDevice) != cudaSuccess ||
           cudaMemcpy(ctx->d_items2[r], it2[r].data(), it2[r].size() * sizeof(int2), cudaMemcpyHostToDevice) != cudaSuccess))
        return fail(set_err(ctx, HAWKES_ERR_CUDA, "copy of work items failed"));
    }
  }
  {
    int2 h[EXP_TABLE];
    make_exp_table(h);
    if (cudaMemcpy(ctx->tab, h, sizeof h, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_err(ctx, HAWKES_ERR_CUDA, "copy of exp table failed"));
  }
  if (cudaMemset(ctx->bad, 0, sizeof(int)) != cudaSuccess ||
      cudaMemset(ctx->st, 0, sizeof(EvalStatus)) != cudaSuccess ||
      cudaMemset(ctx->rec, 0, (size_t)ctx->npad * REC * sizeof(double)) != cudaSuccess)
    return fail(set_err(ctx, HAWKES_ERR_CUDA, "cudaMemset failed"));
  if ((rc = dispatchD<SetupD>(D, ctx))) return fail(rc);
  if (o.nccl_unique_id) {
    std::string e;
    if (!g_nccl.load(e)) return fail(set_err(ctx, HAWKES_ERR_NCCL, "%s", e.c_str()));
    ncclUniqueId id;
    memcpy(&id, o.nccl_unique_id, sizeof id);
    ncclResult_t r = g_nccl.commInitRank(&ctx->comm, o.world, id, o.rank);
    if (r != ncclSuccess) {
      ctx->comm = nullptr;
      return fail(set_err(ctx, HAWKES_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.errStr(r)));
    }
  }
  *out = ctx;
  return HAWKES_OK;
}

int hawkes_destroy(hawkes_ctx* ctx) {
  if (!ctx) return HAWKES_OK;
  cudaSetDevice(ctx->opts.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream); else cudaDeviceSynchronize();
  if (ctx->comm && g_nccl.commDestroy) g_nccl.commDestroy(ctx->comm);
  for (auto& ge : ctx->gexec)
    if (ge) cudaGraphExecDestroy(ge);
  if (ctx->mh_gexec) cudaGraphExecDestroy(ctx->mh_gexec);
  if (ctx->mh_ev0) cudaEventDestroy(ctx->mh_ev0);
  if (ctx->mh_ev1) cudaEventDestroy(ctx->mh_ev1);
  if (ctx->mh_stream) {
    cudaStreamSynchronize(ctx->mh_stream);
    cudaStreamDestroy(ctx->mh_stream);
  }
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  if (ctx->gstream) {
    cudaStreamSynchronize(ctx->gstream);
    cudaStreamDestroy(ctx->gstream);
  }
  void* bufs[] = {ctx->d_mh_stamp, ctx->d_reg_c, ctx->d_reg_s, ctx->d_mh_blocks, ctx->d_mh_acc, ctx->d_mh_la, ctx->d_Y, ctx->d_bgrad, ctx->d_brow, ctx->d_bpart, ctx->d_move_rows_part, ctx->d_move_part, ctx->d_slot_of, ctx->d_move_idx, ctx->d_move_x, ctx->d_move_delta, ctx->d_move_rows,
                  ctx->d_consts, ctx->rec, ctx->rec32, ctx->gid, ctx->part1, ctx->part2, ctx->G1, ctx->rl, ctx->rates,
                  ctx->grad, ctx->xstage, ctx->sendbuf, ctx->recvbuf, ctx->counters, ctx->tab,
                  ctx->bad, ctx->st, ctx->d_all_tiles, ctx->lf_x, ctx->lf_p, ctx->lf_minv,
                  ctx->lf_lo, ctx->lf_hi, ctx->d_own, ctx->d_every_tile, ctx->sums1, ctx->sums2};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (auto* p : ctx->d_items1) if (p) cudaFree(p);
  for (auto* p : ctx->d_items2) if (p) cudaFree(p);
  for (auto* p : ctx->d_sym) if (p) cudaFree(p);
  if (ctx->h_st) cudaFreeHost(ctx->h_st);
  for (auto& pr : ctx->ev_rate) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto& pr : ctx->ev_grad) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  delete ctx;
  return HAWKES_OK;
}

int hawkes_set_times(hawkes_ctx* ctx, const double* t, int32_t mem) {
  ENTER(ctx);
  if (!t || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_set_times");
  const int64_t N = ctx->N;
  std::vector<double> h(N);
  if (mem == HAWKES_MEM_DEVICE) {
    CU(cudaMemcpyAsync(h.data(), t, N * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  } else {
    memcpy(h.data(), t, N * sizeof(double));
  }
  for (int64_t i = 0; i < N; ++i) {
    if (!finite_bounded(h[i]) || h[i] < 0.0)
      return set_err(ctx, HAWKES_ERR_NONFINITE, "t[%lld] = %g is not a finite time >= 0", (long long)i, h[i]);
    if (i && h[i] < h[i - 1])
      return set_err(ctx, HAWKES_ERR_UNSORTED, "t is not non-decreasing at %lld", (long long)i);
  }
  // tie-group ids: first index sharing the time (g_j == g_i <=> t_j == t_i)
  std::vector<int> g(ctx->npad);
  for (int64_t i = 0; i < N; ++i) g[i] = (i && h[i] == h[i - 1]) ? g[i - 1] : (int)i;
  for (int64_t i = N; i < ctx->npad; ++i) g[i] = g[N - 1];
  // stage t in the (rho', ell_n) buffer: xstage keeps the current locations
  CU(cudaMemcpyAsync(ctx->rl, h.data(), N * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->gid, g.data(), ctx->npad * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  TRY(dispatchD<PackTD>(ctx->D, ctx, (const double*)ctx->rl));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->tN = h[N - 1];
  ctx->fc.tN = ctx->tN;
  TRY(upload_consts(ctx));
  ctx->have_t = true;
  ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
  TRY(clear_move(ctx));
  return HAWKES_OK;
}

int hawkes_set_locations(hawkes_ctx* ctx, const double* x, int32_t mem) {
  ENTER(ctx);
  if (!x || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_set_locations");
  const size_t n = (size_t)ctx->N * ctx->D;
  if (mem == HAWKES_MEM_HOST) {
    for (size_t k = 0; k < n; ++k)
      if (!finite_bounded(x[k]))
        return set_err(ctx, HAWKES_ERR_NONFINITE, "x[%zu] = %g is not finite (or |x| > 1e100)", k, x[k]);
  }
  TRY(copy_in(ctx, ctx->xstage, x, n, mem));
  TRY(dispatchD<PackXD>(ctx->D, ctx, (const double*)ctx->xstage));
  ctx->have_x = true;
  ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
  TRY(clear_move(ctx));
  return HAWKES_OK;
}

int hawkes_set_params(hawkes_ctx* ctx, const hawkes_params* p) {
  ENTER(ctx);
  if (!p) return set_err(ctx, HAWKES_ERR_ARG, "params is NULL");
  const double v[6] = {p->mu0, p->tau_x, p->tau_t, p->theta, p->omega, p->sigma_x};
  for (int k = 0; k < 6; ++k)
    if (!isfinite(v[k]) || v[k] < 0.0)
      return set_err(ctx, HAWKES_ERR_PARAM, "Theta[%d] = %g is not finite and >= 0", k, v[k]);
  if (!(p->tau_x > 0 && p->tau_t > 0 && p->omega > 0 && p->sigma_x > 0))
    return set_err(ctx, HAWKES_ERR_PARAM, "tau_x, tau_t, omega and sigma_x must be > 0");
  TRY(compute_constants(ctx, *p, ctx->tN));
  ctx->params = *p;
  ctx->have_p = true;
  ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
  TRY(clear_move(ctx));
  return HAWKES_OK;
}

int hawkes_loglik(hawkes_ctx* ctx, double* out) {
  ENTER(ctx);
  if (!out) return set_err(ctx, HAWKES_ERR_ARG, "out_loglik is NULL");
  TRY(check_ready(ctx));
  TRY(run_rates(ctx));
  TRY(fetch_status(ctx));
  *out = ctx->h_st->ell;
  return HAWKES_OK;
}

int hawkes_grad_locations(hawkes_ctx* ctx, double* out_grad, int32_t mem, double* out_ll) {
  ENTER(ctx);
  if (!out_grad || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_grad_locations");
  TRY(check_ready(ctx));
  TRY(run_rates(ctx));
  TRY(run_grad(ctx));
  TRY(copy_out(ctx, out_grad, ctx->grad, (size_t)ctx->N * ctx->D, mem));
  TRY(fetch_status(ctx));
  if (out_ll) *out_ll = ctx->h_st->ell;
  if (!(ctx->h_st->ell > -INFINITY))
    return set_err(ctx, HAWKES_ERR_GRAD_UNDEFINED, "some lambda_n = 0: ell = -inf, gradient undefined");
  return HAWKES_OK;
}

int hawkes_get_rates(hawkes_ctx* ctx, double* lambda, double* mu, double* xi, double* Lambda,
                     int32_t mem) {
  ENTER(ctx);
  if (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE)
    return set_err(ctx, HAWKES_ERR_ARG, "bad mem");
  TRY(check_ready(ctx));
  TRY(run_rates(ctx));
  if (!ctx->rates_exchanged && !ctx->pairs) {
    TRY(exchange_rows(ctx, ctx->rates, 4));
    ctx->rates_exchanged = true;
  }
  const int64_t N = ctx->N;
  std::vector<double> h((size_t)N * 4);
  CU(cudaMemcpyAsync(h.data(), ctx->rates, h.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  TRY(fetch_status(ctx));
  double* outs[4] = {lambda, mu, xi, Lambda};
  for (int k = 0; k < 4; ++k) {
    if (!outs[k]) continue;
    std::vector<double> col(N);
    for (int64_t i = 0; i < N; ++i) col[i] = h[(size_t)i * 4 + k];
    if (mem == HAWKES_MEM_HOST)
      memcpy(outs[k], col.data(), N * sizeof(double));
    else
      CU(cudaMemcpy(outs[k], col.data(), N * sizeof(double), cudaMemcpyHostToDevice));
  }
  return HAWKES_OK;
}

extern "C++" {
// leapfrog buffers + the optional diagonal inverse mass and box, copied in (per mem)
static int lf_prepare(hawkes_ctx* ctx, int32_t mem, const double* inv_mass, const double* box_lo,
                      const double* box_hi) {
  const size_t n = (size_t)ctx->N * ctx->D;
  if (!ctx->lf_x) {
    int rc;
    if ((rc = dalloc(ctx, &ctx->lf_x, n)) || (rc = dalloc(ctx, &ctx->lf_p, n))) return rc;
  }
  if (inv_mass && !ctx->lf_minv) TRY(dalloc(ctx, &ctx->lf_minv, n));
  if (box_lo && !ctx->lf_lo) {
    TRY(dalloc(ctx, &ctx->lf_lo, n));
    TRY(dalloc(ctx, &ctx->lf_hi, n));
  }
  if (inv_mass) TRY(copy_in(ctx, ctx->lf_minv, inv_mass, n, mem));
  if (box_lo) {
    TRY(copy_in(ctx, ctx->lf_lo, box_lo, n, mem));
    TRY(copy_in(ctx, ctx->lf_hi, box_hi, n, mem));
  }
  return HAWKES_OK;
}

// n_steps leapfrog steps from (lf_x, lf_p), whose positions the records already hold.
// on_start runs after the potential's gradient at the start point is available (the HMC
// step snapshots U(x0) there).  Ends with k_kinetic of the final momenta in st->kinetic.
template <class F>
static int lf_core(hawkes_ctx* ctx, double step, int32_t n_steps, bool has_minv, bool has_box,
                   F on_start) {
  const size_t n = (size_t)ctx->N * ctx->D;
  const bool use_h = ctx->potential & HAWKES_POTENTIAL_HAWKES;
  const bool use_b = (ctx->potential & HAWKES_POTENTIAL_BMDS) != 0;
  auto potential_grad = [&]() -> int {
    if (use_h) TRY(run_grad(ctx));
    if (use_b) TRY(dispatchD<BmdsD>(ctx->D, ctx, (const double*)ctx->lf_x));
    return HAWKES_OK;
  };
  const double* g1 = use_h ? ctx->grad : nullptr;
  const double* g2 = use_b ? ctx->d_bgrad : nullptr;
  TRY(potential_grad());
  TRY(on_start());
  const unsigned nb = (unsigned)((n + 255) / 256);
  for (int s = 0; s < n_steps; ++s) {
    k_kick<<<nb, 256, 0, ctx->stream>>>(ctx->lf_p, g1, g2, (long long)n, 0.5 * step);
    CHECK_LAUNCH();
    TRY(dispatchD<DriftD>(ctx->D, ctx, step, has_box, has_minv));
    ctx->rates_valid = ctx->grad_valid = false;
    TRY(potential_grad());
    k_kick<<<nb, 256, 0, ctx->stream>>>(ctx->lf_p, g1, g2, (long long)n, 0.5 * step);
    CHECK_LAUNCH();
  }
  k_kinetic<<<1, 1024, 0, ctx->stream>>>(ctx->lf_p, has_minv ? ctx->lf_minv : nullptr, (long long)n, ctx->st);
  CHECK_LAUNCH();
  return HAWKES_OK;
}
}  // extern "C++"

int hawkes_leapfrog(hawkes_ctx* ctx, double* x, double* p, int32_t mem, double step,
                    int32_t n_steps, const double* inv_mass, const double* box_lo,
                    const double* box_hi, double* out_ll, double* out_kin) {
  ENTER(ctx);
  if (!x || !p || n_steps < 0 || !isfinite(step) ||
      (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE) || ((box_lo == nullptr) != (box_hi == nullptr)))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_leapfrog");
  if ((ctx->potential & HAWKES_POTENTIAL_HAWKES) && (!ctx->have_t || !ctx->have_p))
    return set_err(ctx, HAWKES_ERR_STATE, "set_times and set_params are required");
  const bool use_h = ctx->potential & HAWKES_POTENTIAL_HAWKES;
  const bool use_b = (ctx->potential & HAWKES_POTENTIAL_BMDS) != 0;
  if (use_b && !ctx->have_bmds) return set_err(ctx, HAWKES_ERR_STATE, "BMDS potential without hawkes_set_bmds");
  const size_t n = (size_t)ctx->N * ctx->D;
  if (mem == HAWKES_MEM_HOST) {
    for (size_t k = 0; k < n; ++k)
      if (!finite_bounded(x[k]) || !finite_bounded(p[k]))
        return set_err(ctx, HAWKES_ERR_NONFINITE, "x or p not finite at %zu", k);
  }
  TRY(lf_prepare(ctx, mem, inv_mass, box_lo, box_hi));
  TRY(copy_in(ctx, ctx->lf_x, x, n, mem));
  TRY(copy_in(ctx, ctx->lf_p, p, n, mem));
  CU(cudaMemsetAsync(&ctx->st->undefined, 0, sizeof(int), ctx->stream));
  TRY(clear_move(ctx));
  TRY(dispatchD<PackXD>(ctx->D, ctx, (const double*)ctx->lf_x));
  ctx->have_x = true;
  ctx->rates_valid = ctx->grad_valid = false;
  TRY(lf_core(ctx, step, n_steps, inv_mass != nullptr, box_lo != nullptr, [] { return HAWKES_OK; }));
  CU(cudaMemcpyAsync(ctx->xstage, ctx->lf_x, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  TRY(copy_out(ctx, x, ctx->lf_x, n, mem));
  TRY(copy_out(ctx, p, ctx->lf_p, n, mem));
  TRY(fetch_status(ctx));
  if (out_ll) *out_ll = (use_h ? ctx->h_st->ell : 0.0) + (use_b ? ctx->h_st->bmds : 0.0);
  if (out_kin) *out_kin = ctx->h_st->kinetic;
  if (ctx->h_st->undefined)
    return set_err(ctx, HAWKES_ERR_GRAD_UNDEFINED, "ell = -inf during the trajectory");
  return HAWKES_OK;
}

int hawkes_hmc_step(hawkes_ctx* ctx, uint64_t seed, uint64_t iteration, double step, int32_t n_steps,
                    const double* inv_mass, const double* box_lo, const double* box_hi, int32_t mem,
                    double* x_out, int32_t* out_accepted, double* out_log_alpha) {
  ENTER(ctx);
  if (n_steps < 0 || !isfinite(step) || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE) ||
      ((box_lo == nullptr) != (box_hi == nullptr)))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_hmc_step");
  const bool use_h = ctx->potential & HAWKES_POTENTIAL_HAWKES;
  const bool use_b = (ctx->potential & HAWKES_POTENTIAL_BMDS) != 0;
  if (!ctx->have_x) return set_err(ctx, HAWKES_ERR_STATE, "hawkes_set_locations is required");
  if (use_h && (!ctx->have_t || !ctx->have_p))
    return set_err(ctx, HAWKES_ERR_STATE, "set_times and set_params are required");
  if (use_b && !ctx->have_bmds) return set_err(ctx, HAWKES_ERR_STATE, "BMDS potential without hawkes_set_bmds");
  if (inv_mass && mem == HAWKES_MEM_HOST) {
    const size_t n = (size_t)ctx->N * ctx->D;
    for (size_t k = 0; k < n; ++k)
      if (!(inv_mass[k] > 0.0) || !(inv_mass[k] < INFINITY))
        return set_err(ctx, HAWKES_ERR_ARG, "inv_mass_diag must be finite and > 0");
  }
  TRY(fetch_status(ctx));   // surface a pending device-side validation failure of x0
  const size_t n = (size_t)ctx->N * ctx->D;
  TRY(lf_prepare(ctx, mem, inv_mass, box_lo, box_hi));
  TRY(clear_move(ctx));
  const uint2 key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
  // x0 = the context's state (records already hold it, so a cached gradient is reused)
  CU(cudaMemcpyAsync(ctx->lf_x, ctx->xstage, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  CU(cudaMemsetAsync(&ctx->st->undefined, 0, sizeof(int), ctx->stream));
  const unsigned nq = (unsigned)((n + 1) / 2);
  k_hmc_momenta<<<(nq + 255) / 256, 256, 0, ctx->stream>>>(ctx->lf_p, inv_mass ? ctx->lf_minv : nullptr,
                                                           (long long)n, key, iteration, 0);
  CHECK_LAUNCH();
  k_kinetic<<<1, 1024, 0, ctx->stream>>>(ctx->lf_p, inv_mass ? ctx->lf_minv : nullptr, (long long)n, ctx->st);
  CHECK_LAUNCH();
  TRY(lf_core(ctx, step, n_steps, inv_mass != nullptr, box_lo != nullptr, [&]() -> int {
    k_hmc_begin<<<1, 1, 0, ctx->stream>>>(ctx->st, use_h, use_b);
    CHECK_LAUNCH();
    return HAWKES_OK;
  }));
  k_hmc_decide<<<1, 1, 0, ctx->stream>>>(ctx->st, ctx->bad, use_h, use_b, key, iteration);
  CHECK_LAUNCH();
  k_hmc_select<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->xstage, ctx->lf_x, (long long)n,
                                                                      ctx->st);
  CHECK_LAUNCH();
  TRY(fetch_status(ctx));
  const bool acc = ctx->h_st->accepted != 0;
  if (ctx->h_st->undef0) {
    ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
    return set_err(ctx, HAWKES_ERR_GRAD_UNDEFINED, "ell = -inf at the chain's current state");
  }
  if (!acc) {   // back to x0: the records and cached rates were those of the trajectory
    TRY(dispatchD<PackXD>(ctx->D, ctx, (const double*)ctx->xstage));
    ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
  }
  if (x_out) {
    TRY(copy_out(ctx, x_out, ctx->xstage, n, mem));
    CU(cudaStreamSynchronize(ctx->stream));
  }
  if (out_accepted) *out_accepted = acc ? 1 : 0;
  if (out_log_alpha) *out_log_alpha = ctx->h_st->log_alpha;
  return HAWKES_OK;
}

int hawkes_diag_normals(uint64_t seed, uint64_t iteration, double* out_dev, int64_t n) {
  if (!out_dev || n < 0) return HAWKES_ERR_ARG;
  if (n == 0) return HAWKES_OK;
  const long long nq = (n + 1) / 2;
  k_hmc_momenta<<<(unsigned)((nq + 255) / 256), 256>>>(out_dev, nullptr, (long long)n,
                                                        make_uint2((unsigned)seed, (unsigned)(seed >> 32)),
                                                        iteration, 1);
  if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return HAWKES_ERR_CUDA;
  return HAWKES_OK;
}

int hawkes_propose_move(hawkes_ctx* ctx, int32_t k, const int32_t* idx, const double* new_x,
                        int32_t mem, double* out_delta) {
  ENTER(ctx);
  if (!idx || !new_x || !out_delta || k < 1 || k > MOVE_MAX ||
      (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_propose_move (1 <= k <= %d)", MOVE_MAX);
  TRY(check_ready(ctx));
  const int D = ctx->D;
  std::vector<int> hidx(idx, idx + k);
  {
    std::vector<int> sorted = hidx;
    std::sort(sorted.begin(), sorted.end());
    for (int q = 0; q < k; ++q)
      if (sorted[q] < 0 || sorted[q] >= ctx->N || (q && sorted[q] == sorted[q - 1]))
        return set_err(ctx, HAWKES_ERR_ARG, "move indices must be distinct and in [0, N)");
  }
  std::vector<double> hx((size_t)k * D);
  if (mem == HAWKES_MEM_DEVICE) {
    CU(cudaMemcpyAsync(hx.data(), new_x, hx.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  } else {
    memcpy(hx.data(), new_x, hx.size() * sizeof(double));
  }
  for (double v : hx)
    if (!finite_bounded(v)) return set_err(ctx, HAWKES_ERR_NONFINITE, "proposed location not finite");
  TRY(clear_move(ctx));
  if (!ctx->lam_valid) {
    ctx->rates_valid = false;
    TRY(run_rates(ctx));
    if (!ctx->pairs && !ctx->rates_exchanged) {
      TRY(exchange_rows(ctx, ctx->rates, 4));
      ctx->rates_exchanged = true;
    }
  }
  CU(cudaMemcpyAsync(ctx->d_move_idx, hidx.data(), k * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->d_move_x, hx.data(), hx.size() * sizeof(double), cudaMemcpyHostToDevice,
                     ctx->stream));
  k_scatter_slots<<<(k + 255) / 256, 256, 0, ctx->stream>>>(ctx->d_slot_of, ctx->d_move_idx, k, 1);
  CHECK_LAUNCH();
  ctx->move_k = k;
  TRY(dispatchD<MoveD>(D, ctx, k, 0));
  TRY(fetch_status(ctx));
  *out_delta = ctx->h_st->dell;
  return HAWKES_OK;
}

int hawkes_accept_move(hawkes_ctx* ctx) {
  ENTER(ctx);
  if (ctx->move_k <= 0) return set_err(ctx, HAWKES_ERR_STATE, "no pending move");
  TRY(dispatchD<CommitD>(ctx->D, ctx, ctx->move_k, 0));
  TRY(clear_move(ctx));
  ctx->rates_valid = ctx->grad_valid = false;   // rho', G1 and ell_n of the old state
  ctx->rates_exchanged = true;                  // every rank updated every row
  ctx->lam_valid = true;
  CU(cudaStreamSynchronize(ctx->stream));
  return HAWKES_OK;
}

int hawkes_get_locations(hawkes_ctx* ctx, double* out_x, int32_t mem) {
  ENTER(ctx);
  if (!out_x || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_get_locations");
  if (!ctx->have_x) return set_err(ctx, HAWKES_ERR_STATE, "no locations");
  TRY(copy_out(ctx, out_x, ctx->xstage, (size_t)ctx->N * ctx->D, mem));
  CU(cudaStreamSynchronize(ctx->stream));
  return HAWKES_OK;
}

int hawkes_set_regions(hawkes_ctx* ctx, int32_t kind, const double* centre, const double* size,
                       int32_t mem) {
  ENTER(ctx);
  if (!centre || !size || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE) ||
      (kind != HAWKES_REGION_SQUARE && kind != HAWKES_REGION_DISC))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_set_regions");
  if (kind == HAWKES_REGION_DISC && ctx->D != 2)
    return set_err(ctx, HAWKES_ERR_DIM, "disc regions (Eq. locsPrior2) need D = 2");
  const size_t N = (size_t)ctx->N, D = (size_t)ctx->D;
  std::vector<double> hc(N * D), hs(N);
  if (mem == HAWKES_MEM_DEVICE) {
    CU(cudaMemcpyAsync(hc.data(), centre, hc.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hs.data(), size, hs.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  } else {
    memcpy(hc.data(), centre, hc.size() * sizeof(double));
    memcpy(hs.data(), size, hs.size() * sizeof(double));
  }
  for (size_t i = 0; i < N; ++i)
    if (!(hs[i] > 0.0) || !finite_bounded(hs[i]))
      return set_err(ctx, HAWKES_ERR_NONFINITE, "region size %zu must be finite and > 0", i);
  for (double v : hc)
    if (!finite_bounded(v)) return set_err(ctx, HAWKES_ERR_NONFINITE, "region centre not finite");
  if (!ctx->d_reg_c) {
    TRY(dalloc(ctx, &ctx->d_reg_c, N * D));
    TRY(dalloc(ctx, &ctx->d_reg_s, N));
  }
  CU(cudaMemcpyAsync(ctx->d_reg_c, hc.data(), hc.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->d_reg_s, hs.data(), hs.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  ctx->reg_kind = kind;
  drop_mh_graph(ctx);
  return HAWKES_OK;
}

int hawkes_mh_sweep(hawkes_ctx* ctx, int32_t n_blocks, int32_t k, const int32_t* blocks, double scale,
                    uint64_t seed, uint64_t iteration, int32_t* out_accepted, double* out_log_alpha,
                    int32_t* out_n_accepted) {
  ENTER(ctx);
  if (n_blocks < 0 || n_blocks >= (1 << 23) || k < 1 || k > MOVE_MAX || (n_blocks > 0 && !blocks) ||
      !(scale > 0.0) || !isfinite(scale))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_mh_sweep (1 <= k <= %d, scale > 0)",
                   MOVE_MAX);
  TRY(check_ready(ctx));
  if (!ctx->reg_kind) return set_err(ctx, HAWKES_ERR_STATE, "hawkes_set_regions is required");
  {
    std::vector<int> sorted(k);
    for (int32_t b = 0; b < n_blocks; ++b) {
      std::copy(blocks + (size_t)b * k, blocks + (size_t)(b + 1) * k, sorted.begin());
      std::sort(sorted.begin(), sorted.end());
      for (int q = 0; q < k; ++q)
        if (sorted[q] < 0 || sorted[q] >= ctx->N || (q && sorted[q] == sorted[q - 1]))
          return set_err(ctx, HAWKES_ERR_ARG, "block %d: indices must be distinct and in [0, N)", b);
    }
  }
  if (out_n_accepted) *out_n_accepted = 0;
  if (n_blocks == 0) return HAWKES_OK;
  TRY(fetch_status(ctx));   // surface a pending device-side validation failure first
  TRY(clear_move(ctx));
  const size_t total = (size_t)n_blocks * k;
  if (total > ctx->mh_cap) {
    if (ctx->d_mh_blocks) cudaFree(ctx->d_mh_blocks);
    ctx->d_mh_blocks = nullptr;
    drop_mh_graph(ctx);
    TRY(dalloc(ctx, &ctx->d_mh_blocks, total));
    ctx->mh_cap = total;
  }
  if ((size_t)n_blocks > ctx->mh_bcap) {
    if (ctx->d_mh_acc) cudaFree(ctx->d_mh_acc);
    if (ctx->d_mh_la) cudaFree(ctx->d_mh_la);
    ctx->d_mh_acc = nullptr;
    ctx->d_mh_la = nullptr;
    drop_mh_graph(ctx);
    TRY(dalloc(ctx, &ctx->d_mh_acc, (size_t)n_blocks));
    TRY(dalloc(ctx, &ctx->d_mh_la, (size_t)n_blocks));
    ctx->mh_bcap = n_blocks;
  }
  CU(cudaMemcpyAsync(ctx->d_mh_blocks, blocks, total * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  if (!ctx->lam_valid) {
    ctx->rates_valid = false;
    TRY(run_rates(ctx));
    if (!ctx->pairs && !ctx->rates_exchanged) {
      TRY(exchange_rows(ctx, ctx->rates, 4));
      ctx->rates_exchanged = true;
    }
  }
  // the sweep's parameters live on the device (EvalStatus mh_*), staged through the pinned
  // status block: one block step (propose, Delta ell, terms + decision, gated commit) then
  // serves every block, as plain launches or as one captured graph replayed per block
  CU(cudaStreamSynchronize(ctx->stream));   // h_st is free to stage
  ctx->h_st->mh_it = iteration;
  ctx->h_st->mh_scale = scale;
  ctx->h_st->mh_key_lo = (unsigned)seed;
  ctx->h_st->mh_key_hi = (unsigned)(seed >> 32);
  ctx->h_st->mh_block = 0;
  ctx->h_st->mh_cur = 0;
  ctx->h_st->mh_prevk = 0;
  const size_t off = offsetof(EvalStatus, mh_it), len = offsetof(EvalStatus, mh_ticket) - off;
  CU(cudaMemcpyAsync(reinterpret_cast<char*>(ctx->st) + off, reinterpret_cast<char*>(ctx->h_st) + off, len,
                     cudaMemcpyHostToDevice, ctx->stream));
  auto block_step = [&]() -> int {
    TRY(dispatchD<MhProposeD>(ctx->D, ctx, (int)k));
    TRY(dispatchD<MoveD>(ctx->D, ctx, (int)k, 1));
    TRY(dispatchD<CommitD>(ctx->D, ctx, (int)k, 1));
    return HAWKES_OK;
  };
  // the cooperative persistent kernel for small blocks (k <= 8: launch latency dominates;
  // profiles/r01_mh_sweep.jsonl), the launch-based block step for larger ones (its kernels
  // run at higher occupancy: 37 vs 72 registers), replayed as a CUDA graph for >= 8 blocks
  // unless HAWKES_NO_GRAPHS.  HAWKES_MH_COOP=0 / 1 forces either (diagnostics, tests).
  const char* coop_env = getenv("HAWKES_MH_COOP");
  const bool coop = ctx->coop_ok && (coop_env ? atoi(coop_env) != 0 : k <= 8);
  const bool graph = !coop && n_blocks >= 8 && !getenv("HAWKES_NO_GRAPHS");
  if (coop) {
    if (!ctx->d_mh_stamp) TRY(dalloc(ctx, &ctx->d_mh_stamp, (size_t)ctx->N));
    CU(cudaMemsetAsync(ctx->d_mh_stamp, 0xff, (size_t)ctx->N * sizeof(int), ctx->stream));
    TRY(dispatchD<MhCoopD>(ctx->D, ctx, (int)n_blocks, (int)k));
  } else if (graph) {
    if (!ctx->mh_stream) {
      CU(cudaStreamCreateWithFlags(&ctx->mh_stream, cudaStreamNonBlocking));
      CU(cudaEventCreateWithFlags(&ctx->mh_ev0, cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&ctx->mh_ev1, cudaEventDisableTiming));
    }
    CU(cudaEventRecord(ctx->mh_ev0, ctx->stream));
    CU(cudaStreamWaitEvent(ctx->mh_stream, ctx->mh_ev0, 0));
    if (!ctx->mh_gexec || ctx->mh_gk != k) {
      drop_mh_graph(ctx);
      cudaStream_t user = ctx->stream;
      const int64_t l0 = ctx->launches;
      ctx->stream = ctx->mh_stream;
      int rc = HAWKES_OK;
      cudaError_t e = cudaStreamBeginCapture(ctx->mh_stream, cudaStreamCaptureModeThreadLocal);
      if (e == cudaSuccess) rc = block_step();
      cudaGraph_t g = nullptr;
      cudaError_t e2 = cudaStreamEndCapture(ctx->mh_stream, &g);
      ctx->stream = user;
      ctx->mh_graph_launches = ctx->launches - l0;
      ctx->launches = l0;
      if (rc != HAWKES_OK) {
        if (g) cudaGraphDestroy(g);
        return rc;
      }
      if (e != cudaSuccess || e2 != cudaSuccess)
        return set_err(ctx, HAWKES_ERR_CUDA, "MH graph capture failed: %s",
                       cudaGetErrorString(e != cudaSuccess ? e : e2));
      cudaError_t e3 = cudaGraphInstantiate(&ctx->mh_gexec, g, 0);
      cudaGraphDestroy(g);
      if (e3 != cudaSuccess) {
        ctx->mh_gexec = nullptr;
        return set_err(ctx, HAWKES_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e3));
      }
      ctx->mh_gk = k;
    }
    for (int32_t b = 0; b < n_blocks; ++b) CU(cudaGraphLaunch(ctx->mh_gexec, ctx->mh_stream));
    ctx->launches += n_blocks * ctx->mh_graph_launches;
    CU(cudaEventRecord(ctx->mh_ev1, ctx->mh_stream));
    CU(cudaStreamWaitEvent(ctx->stream, ctx->mh_ev1, 0));
  } else {
    for (int32_t b = 0; b < n_blocks; ++b) TRY(block_step());
  }
  if (!coop) {   // clear the last block's proposal slots
    k_scatter_slots<<<(k + 255) / 256, 256, 0, ctx->stream>>>(ctx->d_slot_of, ctx->d_move_idx, k, 0);
    CHECK_LAUNCH();
    CU(cudaMemsetAsync(&ctx->st->mh_prevk, 0, sizeof(int), ctx->stream));
  }
  std::vector<int> acc(n_blocks);
  CU(cudaMemcpyAsync(acc.data(), ctx->d_mh_acc, n_blocks * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  if (out_log_alpha)
    CU(cudaMemcpyAsync(out_log_alpha, ctx->d_mh_la, n_blocks * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
  CU(cudaStreamSynchronize(ctx->stream));
  int n_acc = 0;
  for (int32_t b = 0; b < n_blocks; ++b) {
    n_acc += acc[b];
    if (out_accepted) out_accepted[b] = acc[b];
  }
  if (out_n_accepted) *out_n_accepted = n_acc;
  if (n_acc > 0) {
    ctx->rates_valid = ctx->grad_valid = false;   // rho', G1 and ell_n of the old state
    ctx->rates_exchanged = true;                  // every rank updated every row
  }
  ctx->lam_valid = true;
  return HAWKES_OK;
}

int hawkes_set_bmds(hawkes_ctx* ctx, const double* Y, int32_t mem, double sigma) {
  ENTER(ctx);
  if (!Y || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_set_bmds");
  if (!(sigma > 0.0) || !isfinite(sigma) || !isfinite(1.0 / (sigma * sigma)))
    return set_err(ctx, HAWKES_ERR_PARAM, "sigma must be finite and > 0");
  const long long N = ctx->N;
  if (mem == HAWKES_MEM_HOST)
    for (long long nn = 1; nn < N; ++nn)
      for (long long m = 0; m < nn; ++m) {
        const double y = Y[nn * N + m];
        if (!(y > 0.0) || !finite_bounded(y))
          return set_err(ctx, HAWKES_ERR_NONFINITE, "Y[%lld, %lld] = %g: need finite y > 0 below the diagonal", nn, m, y);
      }
  if (!ctx->d_Y) {
    TRY(dalloc(ctx, &ctx->d_Y, (size_t)(N * N)));
    TRY(dalloc(ctx, &ctx->d_bgrad, (size_t)N * ctx->D));
    TRY(dalloc(ctx, &ctx->d_brow, (size_t)N));
    TRY(dalloc(ctx, &ctx->d_bpart, (size_t)((N + 31) / 32 + 1) * N * (ctx->D + 1)));
  }
  TRY(copy_in(ctx, ctx->d_Y, Y, (size_t)(N * N), mem));
  k_bmds_mirror<<<(unsigned)((N * N + 255) / 256), 256, 0, ctx->stream>>>(ctx->d_Y, (int)N, ctx->bad);
  CHECK_LAUNCH();
  ctx->bc.inv_s = 1.0 / sigma;
  ctx->bc.inv_s2 = 1.0 / (sigma * sigma);
  ctx->bc.half_log = 0.5 * log(2.0 * 3.14159265358979323846 * sigma * sigma);
  ctx->bc.mhalf_inv_s2 = -0.5 / (sigma * sigma);
  ctx->bc.lphi_c = -log(sigma) - 0.5 * log(2.0 * 3.14159265358979323846);
  ctx->have_bmds = true;
  return HAWKES_OK;
}

int hawkes_bmds_logdensity(hawkes_ctx* ctx, double* out_grad, int32_t mem, double* out_logp) {
  ENTER(ctx);
  if (!out_logp || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_bmds_logdensity");
  if (!ctx->have_bmds || !ctx->have_x)
    return set_err(ctx, HAWKES_ERR_STATE, "hawkes_set_bmds and hawkes_set_locations are required");
  TRY(dispatchD<BmdsD>(ctx->D, ctx, (const double*)ctx->xstage));
  if (out_grad) TRY(copy_out(ctx, out_grad, ctx->d_bgrad, (size_t)ctx->N * ctx->D, mem));
  TRY(fetch_status(ctx));
  *out_logp = ctx->h_st->bmds;
  return HAWKES_OK;
}

int hawkes_set_potential(hawkes_ctx* ctx, int32_t flags) {
  ENTER(ctx);
  if (flags <= 0 || flags > (HAWKES_POTENTIAL_HAWKES | HAWKES_POTENTIAL_BMDS))
    return set_err(ctx, HAWKES_ERR_ARG, "bad potential flags");
  ctx->potential = flags;
  return HAWKES_OK;
}

int hawkes_enable_timing(hawkes_ctx* ctx, int32_t enable) {
  ENTER(ctx);
  harvest_events(ctx);
  ctx->timing = enable != 0;
  ctx->acc_rate_ms = ctx->acc_grad_ms = 0;
  ctx->n_rate = ctx->n_grad = 0;
  ctx->launches = 0;
  return HAWKES_OK;
}

int hawkes_get_kernel_times(hawkes_ctx* ctx, double* rate_ms, int64_t* rate_n, double* grad_ms,
                            int64_t* grad_n, int64_t* total) {
  ENTER(ctx);
  harvest_events(ctx);
  if (rate_ms) *rate_ms = ctx->acc_rate_ms;
  if (rate_n) *rate_n = ctx->n_rate;
  if (grad_ms) *grad_ms = ctx->acc_grad_ms;
  if (grad_n) *grad_n = ctx->n_grad;
  if (total) *total = ctx->launches;
  return HAWKES_OK;
}

int hawkes_plan(int64_t N, int32_t world, int32_t rank, int32_t* tiles_out, int32_t* n_tiles,
                int32_t* rows_per_tile, int32_t* chunk) {
  if (N < 1 || N > (1LL << 30) || world < 1 || rank < 0 || rank >= world || !n_tiles)
    return set_err(nullptr, HAWKES_ERR_ARG, "bad arguments to hawkes_plan");
  const int nt = (int)((N + RT - 1) / RT);
  int cnt = 0;
  for (int k = 0; k < nt; ++k)
    if (owner_of_tile(k, world) == rank) {
      if (tiles_out) tiles_out[cnt] = k;
      ++cnt;
    }
  *n_tiles = cnt;
  if (rows_per_tile) *rows_per_tile = RT;
  if (chunk) *chunk = chunk_of(N);
  return HAWKES_OK;
}

int hawkes_plan_pairs(int64_t N, int32_t world, int32_t rank, int32_t* items_out,
                      int32_t* n_items, int32_t* chunk) {
  if (N < 1 || N > (1LL << 30) || world < 1 || rank < 0 || rank >= world || !n_items)
    return set_err(nullptr, HAWKES_ERR_ARG, "bad arguments to hawkes_plan_pairs");
  const int ck = chunk_pairs_of(N, world);
  const int C = (int)((N + ck - 1) / ck);
  const std::vector<int> own = pair_owners(N, ck, world);
  int cnt = 0;
  for (int a = 0; a < C; ++a)
    for (int b = a; b < C; ++b)
      if (own[(size_t)a * C + b] == rank) {
        if (items_out) {
          items_out[2 * cnt] = a;
          items_out[2 * cnt + 1] = b;
        }
        ++cnt;
      }
  *n_items = cnt;
  if (chunk) *chunk = ck;
  return HAWKES_OK;
}

int hawkes_nccl_unique_id(void* out) {
  if (!out) return set_err(nullptr, HAWKES_ERR_ARG, "out is NULL");
  std::string e;
  if (!g_nccl.load(e)) return set_err(nullptr, HAWKES_ERR_NCCL, "%s", e.c_str());
  auto get = (ncclResult_t(*)(ncclUniqueId*))dlsym(g_nccl.h, "ncclGetUniqueId");
  if (!get) return set_err(nullptr, HAWKES_ERR_NCCL, "ncclGetUniqueId missing");
  ncclUniqueId id;
  ncclResult_t r = get(&id);
  if (r != ncclSuccess) return set_err(nullptr, HAWKES_ERR_NCCL, "ncclGetUniqueId: %s", g_nccl.errStr(r));
  memcpy(out, &id, sizeof id);
  return HAWKES_OK;
}

// ------------------------------------------------------------------ diagnostics
// Not part of the numerical contract; used by tests and bench.py.
int hawkes_diag_exp(const double* a_dev, double* out_dev, int64_t n) {
  hawkes_ctx* ctx = nullptr;
  int2* tab = nullptr;
  int2 h[EXP_TABLE];
  make_exp_table(h);
  CU(cudaMalloc(&tab, sizeof h));
  CU(cudaMemcpy(tab, h, sizeof h, cudaMemcpyHostToDevice));
  k_diag_exp<<<(unsigned)((n + 255) / 256), 256>>>(a_dev, out_dev, n, tab);
  CU(cudaGetLastError());
  CU(cudaDeviceSynchronize());
  CU(cudaFree(tab));
  return HAWKES_OK;
}

// Operand-pattern probe: thread-iterations per second of k_diag_mode (x8 = ops for modes 0-3,5).
int hawkes_diag_fp64_mode(int32_t mode, int32_t warps_per_sm, double* iters_per_s) {
  hawkes_ctx* ctx = nullptr;
  int dev = 0, sms = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  int2* tab = nullptr;
  int2 h[EXP_TABLE];
  make_exp_table(h);
  CU(cudaMalloc(&out, 8));
  CU(cudaMalloc(&tab, sizeof h));
  CU(cudaMemcpy(tab, h, sizeof h, cudaMemcpyHostToDevice));
  const int threads = 128, blocks = sms * std::max(1, warps_per_sm / 4);
  const int iters = mode == 4 ? 1 << 11 : 1 << 14;
  k_diag_mode<<<blocks, threads>>>(out, 16, mode, tab);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_diag_mode<<<blocks, threads>>>(out, iters, mode, tab);
  cudaEventRecord(b);
  CU(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  cudaFree(tab);
  *iters_per_s = (double)blocks * threads * iters * 8.0 / (ms * 1e-3);
  return HAWKES_OK;
}

// FP64-pipe probe: returns achieved DFMA lane-ops per second over the whole device.
int hawkes_diag_fp64_peak(double* ops_per_s) {
  hawkes_ctx* ctx = nullptr;
  int dev = 0, sms = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* out = nullptr;
  CU(cudaMalloc(&out, 8));
  const int iters = 1 << 16, threads = 512, blocks = sms * 4;
  k_diag_dfma<<<blocks, threads>>>(out, 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_diag_dfma<<<blocks, threads>>>(out, iters);
  cudaEventRecord(b);
  CU(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  *ops_per_s = (double)blocks * threads * iters * 8.0 / (ms * 1e-3);
  return HAWKES_OK;
}

}  // extern "C"
