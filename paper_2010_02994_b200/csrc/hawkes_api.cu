// hawkes_api.cu -- context, C ABI (include/hawkes.h), kernel launch plumbing, exchanges.
//
// One evaluation (ell and d ell/dx) on rank r of W, PAIRS (default):
//   pass 1   sym_kernel<PASS=1> over this rank's chunk pairs (a <= b), each unordered pair
//            once -> per-(slot, event) rate partials (M', X')  [rate pass, Alg. 2 step 1]
//   exchange W > 1: per-event slot sums, ncclAllGather, rank-ordered sum     [S4]
//   fin1     fixed-order slot sum; lambda, rho' = 2^-64 / lambda, Lambda_n (erfc, expm1),
//            ell_n = log lambda_n - Lambda_n; fixed-order ell reduction over all N events
//            (k_fin1p's last CTA)                                       [Eq. 1, P:L92-101]
//   pass 2   sym_kernel<PASS=2>: the pair coefficient c = rho'_i mu' + rho'_j (mu' + xi')
//            and both events' gradient partials c dx, -c dx            [gradient pass, step 2]
//   exchange W > 1: per-event slot sums, ncclAllGather, rank-ordered sum     [S6]
//   fin2     g_i = fixed-order sum of the slots                         [App. A, P:L385]
// ROWS (ordered pairs, pass_kernel): row tiles dealt to ranks zig-zag, allgather of (rho',
// ell_n) rows between the passes and of gradient rows at the end; bitwise identical for any
// W.  Around the evaluation: the HMC leapfrog / transition, block-MH moves and the on-device
// MH sweep, the BMDS density, CUDA-graph capture and replay, kernel timing and diagnostics.

#include "hawkes_context.cuh"
#include "hawkes_launch.cuh"
#include "hawkes_engine.cuh"

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

  std::vector<std::vector<int2>> it1, it2;
  std::vector<std::vector<PairItem>> sym;
  std::vector<std::vector<long long>> coff;
  std::vector<std::vector<int>> cn;
  std::vector<int> own;
  if (ctx->pairs) {
    const int rc0 = dispatchD<SymSetupD>(D, ctx);
    if (rc0 != HAWKES_OK) return fail(rc0);
    build_plan_pairs(ctx, it1, it2, sym, own, coff, cn);
  } else {
    build_plan(ctx, it1, it2);
  }
  // partial slots: PAIRS item-indexed and compact per rank (slot_events x K), ROWS
  // [nchunks][npad][K]
  const size_t slots1 = ctx->pairs ? (size_t)ctx->slot_events * K1P : (size_t)ctx->nslots * ctx->npad * K1_of(D);
  const size_t slots2 = ctx->pairs ? (size_t)ctx->slot_events * K2_of(D) : (size_t)ctx->nslots * ctx->npad * K2_of(D);

  const int REC = REC_of(D);
  int rc;
  if ((rc = dalloc(ctx, &ctx->rec, (size_t)ctx->npad * REC)) ||
      (rc = dalloc(ctx, &ctx->gid, (size_t)ctx->npad)) ||
      // PAIRS' rate partials are (M', X') only (K1P = 2): half the memory at D = 2 that the
      // ROWS layout (M', X', G1') takes -- 211 MB instead of 422 MB at N = 100k, W = 1
      (rc = dalloc(ctx, &ctx->part1, slots1)) || (rc = dalloc(ctx, &ctx->part2, slots2)) ||
      (rc = dalloc(ctx, &ctx->G1, (size_t)ctx->npad * D)) ||
      (rc = dalloc(ctx, &ctx->rl, (size_t)ctx->npad * 2)) ||
      (rc = dalloc(ctx, &ctx->lrho, (size_t)ctx->npad)) ||
      (rc = dalloc(ctx, &ctx->rates, (size_t)ctx->npad * 4)) ||
      (rc = dalloc(ctx, &ctx->grad, (size_t)ctx->npad * D)) ||
      (rc = dalloc(ctx, &ctx->xstage, (size_t)N * D)) ||
      (rc = dalloc(ctx, &ctx->counters, (size_t)4 * ctx->W + 1)) ||
      (rc = dalloc(ctx, &ctx->ell_part, (size_t)(N + 15) / 16)) ||
      (rc = dalloc(ctx, &ctx->tab, EXP_TABLE)) ||
      (rc = dalloc(ctx, &ctx->st, 1)) || (rc = dalloc(ctx, &ctx->d_consts, 1)) ||
      (rc = dalloc(ctx, &ctx->d_slot_of, (size_t)N)) || (rc = dalloc(ctx, &ctx->d_move_idx, MOVE_MAX)) ||
      (rc = dalloc(ctx, &ctx->d_move_x, (size_t)MOVE_MAX * D)) ||
      (rc = dalloc(ctx, &ctx->d_move_delta, (size_t)ctx->npad * 2)) ||
      (rc = dalloc(ctx, &ctx->d_move_rows, (size_t)MOVE_MAX * 2)) ||
      (rc = dalloc(ctx, &ctx->d_move_part, (size_t)(N + 255) / 256)) ||
      (rc = dalloc(ctx, &ctx->d_move_rows_part, (size_t)MOVE_MAX * 2 * MOVE_NSPLIT)))
    return fail(rc);
  if (cudaMemset(ctx->d_slot_of, 0xff, (size_t)N * sizeof(int)) != cudaSuccess ||
      cudaMemset(ctx->lrho, 0, (size_t)ctx->npad * sizeof(double)) != cudaSuccess)
    return fail(set_err(ctx, HAWKES_ERR_CUDA, "cudaMemset failed"));
  if (!ctx->multi && !getenv("HAWKES_NO_GRAPHS")) {
    if (cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking) != cudaSuccess)
      return fail(set_err(ctx, HAWKES_ERR_CUDA, "stream creation failed"));
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
    ctx->d_coff.assign(ctx->W, nullptr);
    ctx->d_cn.assign(ctx->W, nullptr);
    ctx->n_sym.assign(ctx->W, 0);
    for (int r = 0; r < ctx->W; ++r) {
      ctx->n_sym[r] = (int)sym[r].size();
      if ((rc = dalloc(ctx, &ctx->d_sym[r], sym[r].size())) ||
          (rc = dalloc(ctx, &ctx->d_coff[r], coff[r].size())) || (rc = dalloc(ctx, &ctx->d_cn[r], cn[r].size())))
        return fail(rc);
      if ((!sym[r].empty() &&
           cudaMemcpy(ctx->d_sym[r], sym[r].data(), sym[r].size() * sizeof(PairItem), cudaMemcpyHostToDevice) != cudaSuccess) ||
          cudaMemcpy(ctx->d_coff[r], coff[r].data(), coff[r].size() * sizeof(long long), cudaMemcpyHostToDevice) != cudaSuccess ||
          cudaMemcpy(ctx->d_cn[r], cn[r].data(), cn[r].size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
        return fail(set_err(ctx, HAWKES_ERR_CUDA, "copy of the pair items failed"));
    }
    if (ctx->multi) {
      const size_t copies = (size_t)ctx->W + 1;   // row 0: the sum; rows 1..W: per-rank sums
      if ((rc = dalloc(ctx, &ctx->sums1, copies * ctx->npad * K1P)) ||
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
    e = cudaHostAlloc((void**)&ctx->h_mirror, sizeof(EvalStatus), cudaHostAllocMapped);
    if (e != cudaSuccess) return fail(set_err(ctx, HAWKES_ERR_OOM, "cudaHostAlloc failed"));
    memset((void*)ctx->h_mirror, 0, sizeof(EvalStatus));
    if (cudaHostGetDevicePointer((void**)&ctx->d_mirror, ctx->h_mirror, 0) != cudaSuccess)
      return fail(set_err(ctx, HAWKES_ERR_CUDA, "cudaHostGetDevicePointer failed"));
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
  ctx->bad = &ctx->st->nonfinite;
  if (cudaMemset(ctx->st, 0, sizeof(EvalStatus)) != cudaSuccess ||
      cudaMemset(ctx->counters, 0, sizeof(int) * (4 * ctx->W + 1)) != cudaSuccess ||
      cudaMemset(ctx->rec, 0, (size_t)ctx->npad * REC * sizeof(double)) != cudaSuccess)
    return fail(set_err(ctx, HAWKES_ERR_CUDA, "cudaMemset failed"));
  ctx->counters_armed = true;
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
  if (ctx->g_at) cudaGraphDestroy(ctx->g_at);
  if (ctx->mh_gexec) cudaGraphExecDestroy(ctx->mh_gexec);
  if (ctx->mh_ev0) cudaEventDestroy(ctx->mh_ev0);
  if (ctx->mh_ev1) cudaEventDestroy(ctx->mh_ev1);
  if (ctx->mh_stream) {
    cudaStreamSynchronize(ctx->mh_stream);
    cudaStreamDestroy(ctx->mh_stream);
  }
  if (ctx->gstream) {
    cudaStreamSynchronize(ctx->gstream);
    cudaStreamDestroy(ctx->gstream);
  }
  void* bufs[] = {ctx->d_mh_stamp, ctx->d_reg_c, ctx->d_reg_s, ctx->d_mh_blocks, ctx->d_mh_acc, ctx->d_mh_la, ctx->d_Y, ctx->d_bgrad, ctx->d_brow, ctx->d_bpart, ctx->d_move_rows_part, ctx->d_move_part, ctx->d_slot_of, ctx->d_move_idx, ctx->d_move_x, ctx->d_move_delta, ctx->d_move_rows,
                  ctx->d_consts, ctx->rec, ctx->rec32, ctx->gid, ctx->part1, ctx->part2, ctx->G1, ctx->rl, ctx->lrho, ctx->d_perm, ctx->d_gid_p, ctx->rec_p, ctx->rec32_p, ctx->d_boxes, ctx->rates,
                  ctx->grad, ctx->xstage, ctx->sendbuf, ctx->recvbuf, ctx->counters, ctx->ell_part, ctx->tab,
                  ctx->st, ctx->d_all_tiles, ctx->lf_x, ctx->lf_p, ctx->lf_minv,
                  ctx->lf_lo, ctx->lf_hi, ctx->lf_x0, ctx->lf_p0, ctx->d_own, ctx->d_every_tile, ctx->sums1, ctx->sums2};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (auto* p : ctx->d_items1) if (p) cudaFree(p);
  for (auto* p : ctx->d_items2) if (p) cudaFree(p);
  for (auto* p : ctx->d_sym) if (p) cudaFree(p);
  for (auto* p : ctx->d_coff) if (p) cudaFree(p);
  for (auto* p : ctx->d_cn) if (p) cudaFree(p);
  if (ctx->h_st) cudaFreeHost(ctx->h_st);
  if (ctx->h_mirror) cudaFreeHost(ctx->h_mirror);
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
    TRY(wait_stream(ctx));
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
  TRY(wait_stream(ctx));
  ctx->tN = h[N - 1];
  ctx->fc.tN = ctx->tN;
  TRY(upload_consts(ctx));
  ctx->have_t = true;
  ctx->fb64 = false;   // a new catalog: the fp32 range guard decides again
  ctx->h_t.swap(h);
  ctx->ties = false;
  for (int64_t i = 1; i < N; ++i) ctx->ties |= ctx->h_t[i] == ctx->h_t[i - 1];
  ctx->order_decided = false;   // and the walk order
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
  if (mem == HAWKES_MEM_DEVICE) {   // pack straight from the caller's array (stream-ordered)
    TRY(dispatchD<PackXD>(ctx->D, ctx, x, ctx->xstage));
  } else {
    TRY(copy_in(ctx, ctx->xstage, x, n, mem));
    TRY(dispatchD<PackXD>(ctx->D, ctx, (const double*)ctx->xstage));
  }
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
  if (ctx->fb64) drop_graphs(ctx);
  ctx->fb64 = false;   // new constants: the fp32 range guard decides again
  ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
  TRY(clear_move(ctx));
  return HAWKES_OK;
}

int hawkes_loglik(hawkes_ctx* ctx, double* out) {
  ENTER(ctx);
  if (!out) return set_err(ctx, HAWKES_ERR_ARG, "out_loglik is NULL");
  TRY(check_ready(ctx));
  ctx->mirror_fresh = false;
  TRY(checked_rates(ctx, true));
  *out = ctx->h_st->ell;
  return HAWKES_OK;
}

int hawkes_grad_locations(hawkes_ctx* ctx, double* out_grad, int32_t mem, double* out_ll) {
  ENTER(ctx);
  if (!out_grad || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_grad_locations");
  TRY(check_ready(ctx));
  ctx->mirror_fresh = false;
  do {   // twice only if the fp32 range guard sent the context to fp64
    TRY(run_grad(ctx));   // (with the rate pass first when it is due)
    TRY(copy_out(ctx, out_grad, ctx->grad, (size_t)ctx->N * ctx->D, mem));
    TRY(fetch_status(ctx, true));
  } while (take_retry(ctx));
  if (out_ll) *out_ll = ctx->h_st->ell;
  if (!(ctx->h_st->ell > -INFINITY))
    return set_err(ctx, HAWKES_ERR_GRAD_UNDEFINED, "some lambda_n = 0: ell = -inf, gradient undefined");
  return HAWKES_OK;
}

int hawkes_grad_at(hawkes_ctx* ctx, const double* x, double* out_grad, double* out_ll) {
  ENTER(ctx);
  if (!x || !out_grad) return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_grad_at");
  if (!ctx->have_t || !ctx->have_p)
    return set_err(ctx, HAWKES_ERR_STATE, "set_times and set_params are required");
  TRY(clear_move(ctx));
  ctx->mirror_fresh = false;
  bool done = false;
  // the captured path counts the evaluation as run_grad would (use_graph: same constants for
  // >= 2 evaluations); the plain path below counts it itself
  ++ctx->evals_same_consts;
  TRY(grad_at_graph(ctx, x, out_grad, &done));
  if (done) {
    ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = true;
    ctx->rates_exchanged = false;
  } else {
    --ctx->evals_same_consts;
    TRY(dispatchD<PackXD>(ctx->D, ctx, x, ctx->xstage));
    ctx->have_x = true;
    ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
    TRY(run_grad(ctx));
    TRY(copy_out(ctx, out_grad, ctx->grad, (size_t)ctx->N * ctx->D, HAWKES_MEM_DEVICE));
  }
  TRY(fetch_status(ctx, true));
  while (take_retry(ctx)) {   // the fp32 range guard sent the context to fp64
    TRY(run_grad(ctx));
    TRY(copy_out(ctx, out_grad, ctx->grad, (size_t)ctx->N * ctx->D, HAWKES_MEM_DEVICE));
    TRY(fetch_status(ctx, true));
  }
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
  ctx->mirror_fresh = false;
  TRY(checked_rates(ctx, true));
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

int hawkes_set_ordering(hawkes_ctx* ctx, int32_t mode) {
  ENTER(ctx);
  if (mode != HAWKES_ORDER_AUTO && mode != HAWKES_ORDER_TIME && mode != HAWKES_ORDER_SPACE)
    return set_err(ctx, HAWKES_ERR_ARG, "bad ordering mode %d", mode);
  ctx->order_req = mode;
  ctx->order_decided = false;
  drop_graphs(ctx);
  ctx->rates_valid = ctx->grad_valid = false;
  return HAWKES_OK;
}

int hawkes_ordering_in_use(const hawkes_ctx* ctx, int32_t* out, double* out_cost) {
  if (!ctx || !out) return HAWKES_ERR_ARG;
  *out = ctx->spatial ? HAWKES_ORDER_SPACE : HAWKES_ORDER_TIME;
  if (out_cost) {
    out_cost[0] = ctx->order_cost[0];
    out_cost[1] = ctx->order_cost[1];
  }
  return HAWKES_OK;
}

int hawkes_precision_in_use(const hawkes_ctx* ctx, int32_t* out) {
  if (!ctx || !out) return HAWKES_ERR_ARG;
  *out = use32(ctx) ? HAWKES_FP32 : HAWKES_FP64;
  return HAWKES_OK;
}

#include "hawkes_samplers.cuh"

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

int hawkes_plan_items(int64_t N, int32_t world, int32_t rank, int32_t resident, int64_t* items_out,
                      int32_t* n_items, int32_t* pieces, int64_t* slot_events) {
  if (N < 1 || N > (1LL << 30) || world < 1 || rank < 0 || rank >= world || resident < 0 || !n_items)
    return set_err(nullptr, HAWKES_ERR_ARG, "bad arguments to hawkes_plan_items");
  const int ck = chunk_pairs_of(N, world);
  const PairsLayout L = pairs_layout(N, ck, world, {rank}, resident);
  const auto& it = L.items[rank];
  *n_items = (int32_t)it.size();
  if (pieces) *pieces = L.pieces[rank];
  if (slot_events) *slot_events = L.slot_events;
  if (items_out)
    for (size_t q = 0; q < it.size(); ++q) {
      int64_t* o = items_out + 6 * q;
      o[0] = it[q].a;
      o[1] = it[q].b;
      o[2] = it[q].ro;
      o[3] = it[q].co;
      o[4] = it[q].s0;
      o[5] = it[q].s1;
    }
  return HAWKES_OK;
}

int hawkes_plan_walk(const double* x, const double* t, int64_t N, int32_t D, const hawkes_params* p,
                     int32_t* perm_out, double* cost_out) {
  if (!x || !t || !p || N < 1 || N > (1LL << 30) || D < 1 || D > HAWKES_MAX_D)
    return set_err(nullptr, HAWKES_ERR_ARG, "bad arguments to hawkes_plan_walk");
  const std::vector<int> perm = morton_order(x, (int)N, D);
  if (perm_out) memcpy(perm_out, perm.data(), N * sizeof(int32_t));
  if (cost_out) {
    const PassConst pc = make_pass_const(*p, D, nullptr, nullptr);
    cost_out[0] = walk_cost(x, t, nullptr, (int)N, D, pc, false);
    cost_out[1] = walk_cost(x, t, perm.data(), (int)N, D, pc, true);
  }
  return HAWKES_OK;
}

int hawkes_plan_slots(int64_t N, int32_t world, int32_t rank, int64_t* slot_events, int64_t* max_events) {
  if (N < 1 || N > (1LL << 30) || world < 1 || rank < 0 || rank >= world || !slot_events)
    return set_err(nullptr, HAWKES_ERR_ARG, "bad arguments to hawkes_plan_slots");
  const int ck = chunk_pairs_of(N, world);
  const PairsLayout L = pairs_layout(N, ck, world, {rank});
  *slot_events = L.slot_events;
  if (max_events) {   // every rank's, for the balance
    long long mx = 0;
    for (int r = 0; r < world; ++r) {
      long long s = 0;
      for (int c : L.cn[r]) s += (long long)c * ck;
      mx = std::max(mx, s);
    }
    *max_events = mx;
  }
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
  const int iters = (mode == 4 || mode == 15) ? 1 << 11 : 1 << 14;
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
