// hawkes_context.cuh -- part of hawkes_api.cu (one translation unit; included once, in
// order): includes, NCCL via dlopen, the context struct, error and allocation helpers,
// dispatch on D.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges cost nothing without a tool attached
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

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
  // optional (NCCL >= 2.4): polled while a host thread waits on a stream with collectives,
  // so a failed peer returns HAWKES_ERR_NCCL instead of hanging every rank
  ncclResult_t (*asyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*commAbort)(ncclComm_t) = nullptr;
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
    asyncError = (decltype(asyncError))dlsym(h, "ncclCommGetAsyncError");
    commAbort = (decltype(commAbort))dlsym(h, "ncclCommAbort");
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
  std::vector<PairItem*> d_sym;             // per rank: chunk pairs (a <= b) and slot blocks
  std::vector<int> n_sym;
  std::vector<long long*> d_coff;           // per rank: [nchunks] slot-block event offsets
  std::vector<int*> d_cn;                   // per rank: [nchunks] slot blocks per chunk
  long long slot_events = 0;                // events of all slot blocks this process holds
  std::vector<int> piece_k;                 // per rank: 1, or the plan's pieces per item
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
  double* lrho = nullptr;  // npad: -ln lambda_n (PAIRS fp64 gradient pass; hawkes_kernels_sym.cuh)
  // walk order of the PAIRS fp64 kernels (hawkes_plan.h): time (records as they are) or
  // spatial (a Morton permutation; rec_p gathered per evaluation, with 128-event tile boxes)
  int order_req = 0;          // HAWKES_ORDER_AUTO / _TIME / _SPACE (hawkes_set_ordering)
  bool order_decided = false; // decided at the first evaluation after set_times / set_ordering
  bool spatial = false;       // the walk is spatial
  double order_cost[2] = {0.0, 0.0};   // walk_cost estimates (time, space) of the decision
  bool ties = false;          // the catalog has equal times
  std::vector<double> h_t;    // host copy of the times (order decision, tie groups)
  int* d_perm = nullptr;      // npad: walk position -> event
  int* d_gid_p = nullptr;     // npad: tie-group ids in walk order
  double* rec_p = nullptr;    // npad x REC: records in walk order
  float* rec32_p = nullptr;   // npad x REC32: fp32 records in walk order (fp32 contexts)
  double* d_boxes = nullptr;  // npad/128 x (2D + 2): tile boxes in walk order
  double* rates = nullptr; // npad x 4 (lambda, mu, xi, Lambda)
  double* grad = nullptr;  // npad x D
  double* xstage = nullptr;// N x D staging
  double* sendbuf = nullptr;
  double* recvbuf = nullptr;
  int* counters = nullptr; // 4 per logical rank, + 1: k_fin1p's block ticket (PAIRS ell)
  double* ell_part = nullptr; // PAIRS: k_fin1p's per-CTA ell sums (ceil(N / 16))
  int2* tab = nullptr;     // exp table
  int* bad = nullptr;      // device-side input validation flag: &st->nonfinite
  EvalStatus* st = nullptr;
  EvalStatus* h_st = nullptr;  // pinned
  // small-call path (hawkes_loglik / hawkes_grad_locations / hawkes_get_rates): k_fin1p's last
  // CTA copies the status into the mapped, pinned h_mirror (device view d_mirror), so those
  // calls need no device-to-host status copy after the evaluation
  EvalStatus* h_mirror = nullptr;
  EvalStatus* d_mirror = nullptr;
  bool mirror_fresh = false;   // a k_fin1p was enqueued since the last fetch_status
  bool counters_armed = false; // PAIRS item counters are zero (re-armed by the finalizes)
  // leapfrog state
  double *lf_x = nullptr, *lf_p = nullptr, *lf_minv = nullptr, *lf_lo = nullptr, *lf_hi = nullptr;
  double *lf_x0 = nullptr, *lf_p0 = nullptr;   // start of the trajectory (fp64 re-run)

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
  FinConst fc64{};            // fc of the fp64 kernels (== fc on an fp64 context)
  // fp32 range guard (R23): an fp32 context whose evaluation tripped the guard
  // evaluates with the fp64 kernels (records and constants of both precisions are kept)
  // until set_times / set_params; retry = the current call must be redone in fp64
  bool fb64 = false;
  bool retry = false;

  // timing
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_rate, ev_grad;
  std::vector<cudaEvent_t> ev_pool;
  double acc_rate_ms = 0, acc_grad_ms = 0;
  int64_t n_rate = 0, n_grad = 0;
  int64_t launches = 0;

  int grid1 = 0, grid2 = 0;
  int grid_s1 = 0, grid_s2 = 0;
  int grid32_1 = 0, grid32_2 = 0, grid32_s1 = 0, grid32_s2 = 0;   // fp32 kernels
  int grid_g1 = 0, grid_g2 = 0;   // spatial-walk (GEN) sym kernels
  int grid32_g1 = 0, grid32_g2 = 0;
  DevConsts* d_consts = nullptr;
  // CUDA graphs of one evaluation (single process, W = 1, timing off)
  cudaStream_t gstream = nullptr;
  // rates, rates+grad, grad only, and (3) hawkes_grad_at: pack + rates + grad, whose pack and
  // gradient-finalize nodes take the caller's x / gradient pointers per launch
  cudaGraphExec_t gexec[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaGraph_t g_at = nullptr;                 // kept: its nodes address the exec's params
  cudaGraphNode_t at_pack = nullptr, at_pack32 = nullptr, at_fin2 = nullptr;
  const double* at_x = nullptr;   // the pointers the exec's nodes hold (no update when unchanged)
  double* at_out = nullptr;
  bool graphs = false;
  bool capturing = false;
  int64_t graph_launches[4] = {0, 0, 0, 0};
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

// NVTX range over one ABI call (visible in an nsys / ncu timeline as "hawkes_<call>")
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define NVTX_CALL() NvtxRange nvtx_range_(__func__)

#define ENTER(ctx)                                                                      \
  NVTX_CALL();                                                                          \
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

// Host wait on the context stream.  With an NCCL communicator the wait polls
// ncclCommGetAsyncError (and an optional HAWKES_NCCL_TIMEOUT_S deadline, default 900 s): a
// peer that failed aborts the communicator and returns HAWKES_ERR_NCCL (sticky) instead of
// leaving every rank blocked in cudaStreamSynchronize.
int wait_stream(hawkes_ctx* ctx) {
  if (!ctx->comm) {
    CU(cudaStreamSynchronize(ctx->stream));
    return HAWKES_OK;
  }
  static const double limit_s = [] {
    const char* e = getenv("HAWKES_NCCL_TIMEOUT_S");
    return e ? atof(e) : 900.0;
  }();
  timespec t0;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(ctx->stream);
    if (q == cudaSuccess) return HAWKES_OK;
    if (q != cudaErrorNotReady)
      return set_err(ctx, HAWKES_ERR_CUDA, "stream wait failed: %s", cudaGetErrorString(q));
    ncclResult_t ar = ncclSuccess;
    bool failed = false;
    if (g_nccl.asyncError && g_nccl.asyncError(ctx->comm, &ar) == ncclSuccess && ar != ncclSuccess &&
        ar != ncclInProgress)
      failed = true;
    timespec t1;
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double el = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    if (failed || (limit_s > 0 && el > limit_s)) {
      if (g_nccl.commAbort) g_nccl.commAbort(ctx->comm);
      ctx->comm = nullptr;
      if (failed) return set_err(ctx, HAWKES_ERR_NCCL, "NCCL asynchronous error: %s", g_nccl.errStr(ar));
      return set_err(ctx, HAWKES_ERR_NCCL, "NCCL collective did not complete in %.0f s", limit_s);
    }
    if (spin > 64) {   // short waits spin; long ones (a whole evaluation) sleep 20 us per poll
      timespec d{0, 20000};
      nanosleep(&d, nullptr);
    }
  }
}

// the fp32 pass kernels run unless the range guard sent this context to fp64
inline bool use32(const hawkes_ctx* ctx) { return ctx->rec32 != nullptr && !ctx->fb64; }
inline const FinConst& fcur(const hawkes_ctx* ctx) { return use32(ctx) ? ctx->fc : ctx->fc64; }

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

}  // namespace
