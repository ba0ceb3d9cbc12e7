// hawkes_engine.cuh -- part of hawkes_api.cu (one translation unit): the exchanges
// (NCCL or emulated ranks), CUDA-graph capture and replay, the rate and gradient
// evaluations, status handling, the work plans, the folded constants and the exp table.
#pragma once
namespace {

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

// PAIRS, W > 1 (S4 / S6): each logical rank sums its own chunk pairs' slots per event in a
// fixed order (k_slot_sum) into row 1 + r of sums[W + 1][npad][K]; the W rows are then
// gathered (ncclAllGather in place, or already in place for emulated ranks) and added in
// rank order into row 0 (k_sum_ranks).  The result is bitwise reproducible run to run at a
// fixed W on every rank: unlike an ncclAllReduce, it does not depend on NCCL's algorithm
// or protocol choice (ring / tree / NVLS), and every rank adds the same W values in the
// same order.
int reduce_pair_partials(hawkes_ctx* ctx, const double* part, double* sums, int K) {
  const long long n = (long long)ctx->N * K;
  const long long stride = (long long)ctx->npad * K;
  for (int r : ctx->my_ranks) {
    k_slot_sum<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
        part, SlotView{ctx->d_coff[r], ctx->d_cn[r], ctx->chunk}, K, (int)ctx->N, sums + (1 + r) * stride);
    CHECK_LAUNCH();
  }
  if (ctx->comm) {
    const int r = ctx->my_ranks[0];
    NC(g_nccl.allGather(sums + (1 + r) * stride, sums + stride, (size_t)stride, ncclDouble, ctx->comm,
                        ctx->stream));
  }
  k_sum_ranks<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(sums + stride, stride, ctx->W, n,
                                                                   sums);
  CHECK_LAUNCH();
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
  if (ctx->g_at) cudaGraphDestroy(ctx->g_at);
  ctx->g_at = nullptr;
  ctx->at_pack = ctx->at_pack32 = ctx->at_fin2 = nullptr;
  ctx->at_x = nullptr;
  ctx->at_out = nullptr;
  ctx->evals_same_consts = 0;
  drop_mh_graph(ctx);   // its launches carry the folded constants by value
}

// Capture one evaluation sequence (0: rate pass; 1: rate + gradient pass; 2: gradient pass
// with cached rates; 3: location packing + rate + gradient pass, hawkes_grad_at) on the
// context's own stream and instantiate it.
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
    // (3: packed from xstage in place; each launch points the pack nodes at the caller's x)
    if (which == 3) rc = dispatchD<PackXD>(ctx->D, ctx, (const double*)ctx->xstage, ctx->xstage);
    if (rc == HAWKES_OK) rc = which == 0 ? run_rates(ctx) : run_grad(ctx);
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
  if (which == 3 && e3 == cudaSuccess) {
    ctx->g_at = g;
    TRY(dispatchD<AtNodesD>(ctx->D, ctx));
    if (!ctx->at_pack || !ctx->at_fin2 || (ctx->rec32 && !ctx->at_pack32))
      return set_err(ctx, HAWKES_ERR_CUDA, "grad_at graph: packing / finalize nodes not found");
  } else {
    cudaGraphDestroy(g);
  }
  if (e3 != cudaSuccess)
    return set_err(ctx, HAWKES_ERR_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(e3));
  ctx->graph_launches[which] = ctx->launches - l0;
  ctx->launches = l0;
  return HAWKES_OK;
}

// Point one kernel node of the grad_at exec at a new value of argument `arg` (a pointer): the
// other arguments keep the values captured in g_at.
int set_node_ptr(hawkes_ctx* ctx, cudaGraphNode_t nd, int arg, int nargs, const void* const* val) {
  cudaKernelNodeParams kp;
  CU(cudaGraphKernelNodeGetParams(nd, &kp));
  void* args[16];
  if (nargs > 16) return set_err(ctx, HAWKES_ERR_CUDA, "set_node_ptr: too many arguments");
  for (int k = 0; k < nargs; ++k) args[k] = kp.kernelParams[k];
  args[arg] = const_cast<void*>(static_cast<const void*>(val));
  kp.kernelParams = args;
  kp.extra = nullptr;
  CU(cudaGraphExecKernelNodeSetParams(ctx->gexec[3], nd, &kp));
  return HAWKES_OK;
}

int replay(hawkes_ctx* ctx, int which) {
  if (!ctx->gexec[which]) TRY(capture(ctx, which));
  // captured on the private stream (capture cannot run on the legacy default stream), launched
  // into the caller's stream: stream order alone sequences it
  CU(cudaGraphLaunch(ctx->gexec[which], ctx->stream));
  ctx->launches += ctx->graph_launches[which];
  return HAWKES_OK;
}

// The PAIRS fp64 walk order (hawkes_plan.h, include/hawkes.h hawkes_ordering), decided at the
// first evaluation after set_times / set_ordering from that evaluation's locations and Theta.
int decide_order(hawkes_ctx* ctx) {
  ctx->order_decided = true;
  ctx->order_cost[0] = ctx->order_cost[1] = 0.0;
  const int N = (int)ctx->N, D = ctx->D;
  const bool eligible = ctx->pairs && D <= SPACE_MAX_D && N >= 2 * TILE_J &&
                        ctx->order_req != HAWKES_ORDER_TIME;
  bool want = false;
  std::vector<int> perm;
  if (eligible) {
    std::vector<double> hx((size_t)N * D);
    CU(cudaMemcpyAsync(hx.data(), ctx->xstage, hx.size() * sizeof(double), cudaMemcpyDeviceToHost,
                       ctx->stream));
    TRY(wait_stream(ctx));
    perm = morton_order(hx.data(), N, D);
    if (ctx->order_req == HAWKES_ORDER_SPACE) {
      want = true;
    } else {
      ctx->order_cost[0] = walk_cost(hx.data(), ctx->h_t.data(), nullptr, N, D, ctx->pc, false);
      ctx->order_cost[1] = walk_cost(hx.data(), ctx->h_t.data(), perm.data(), N, D, ctx->pc, true);
      want = ctx->order_cost[1] < 0.9 * ctx->order_cost[0];
    }
  }
  if (want != ctx->spatial) drop_graphs(ctx);
  ctx->spatial = want;
  if (!want) return HAWKES_OK;
  const int REC = REC_of(D);
  if (!ctx->d_perm) {
    int rc;
    if ((rc = dalloc(ctx, &ctx->d_perm, (size_t)ctx->npad)) ||
        (rc = dalloc(ctx, &ctx->d_gid_p, (size_t)ctx->npad)) ||
        (rc = dalloc(ctx, &ctx->rec_p, (size_t)ctx->npad * REC)) ||
        (rc = dalloc(ctx, &ctx->d_boxes, (size_t)(ctx->npad / TILE_J) * (2 * D + 2))))
      return rc;
    CU(cudaMemsetAsync(ctx->rec_p, 0, (size_t)ctx->npad * REC * sizeof(double), ctx->stream));
    if (ctx->rec32) {
      TRY(dalloc(ctx, &ctx->rec32_p, (size_t)ctx->npad * Layout32Rec(D)));
      CU(cudaMemsetAsync(ctx->rec32_p, 0, (size_t)ctx->npad * Layout32Rec(D) * sizeof(float), ctx->stream));
    }
  }
  // tie-group ids (first event with the same time) in walk order
  std::vector<int> g(N), gp(ctx->npad);
  for (int i = 0; i < N; ++i) g[i] = (i && ctx->h_t[i] == ctx->h_t[i - 1]) ? g[i - 1] : i;
  std::vector<int> hp(ctx->npad);
  for (int p = 0; p < ctx->npad; ++p) {
    hp[p] = perm[std::min(p, N - 1)];
    gp[p] = g[hp[p]];
  }
  CU(cudaMemcpyAsync(ctx->d_perm, hp.data(), hp.size() * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  CU(cudaMemcpyAsync(ctx->d_gid_p, gp.data(), gp.size() * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  TRY(wait_stream(ctx));   // the host vectors go out of scope
  return HAWKES_OK;
}

int run_rates(hawkes_ctx* ctx) {
  if (ctx->rates_valid) return HAWKES_OK;
  if (!ctx->order_decided && !ctx->capturing) TRY(decide_order(ctx));
  if (!ctx->capturing) ++ctx->evals_same_consts;
  if (use_graph(ctx)) {
    TRY(replay(ctx, 0));
    if (ctx->pairs) ctx->mirror_fresh = true;
    ctx->rates_valid = true;
    ctx->rates_exchanged = false;
    ctx->grad_valid = false;
    ctx->lam_valid = true;
    return HAWKES_OK;
  }
  // PAIRS: the finalizes re-arm the item counters they follow (k_fin1p / k_fin2p), so the
  // captured evaluation starts with the pass kernel instead of a memset node
  if (!ctx->pairs || !ctx->counters_armed)
    CU(cudaMemsetAsync(ctx->counters, 0, sizeof(int) * (4 * ctx->W + 1), ctx->stream));
  if (ctx->pairs) {
    if (ctx->spatial) TRY(dispatchD<WalkD>(ctx->D, ctx));
    for (int r : ctx->my_ranks) TRY(dispatchD<PassD>(ctx->D, ctx, 1, r));
    if (ctx->multi) TRY(reduce_pair_partials(ctx, ctx->part1, ctx->sums1, K1P));
    TRY(dispatchD<Fin1D>(ctx->D, ctx, 0));
  } else {
    for (int r : ctx->my_ranks) {
      TRY(dispatchD<PassD>(ctx->D, ctx, 1, r));
      TRY(dispatchD<Fin1D>(ctx->D, ctx, r));
    }
    TRY(exchange_rows(ctx, ctx->rl, 2));
    if (ctx->multi) TRY(dispatchD<RhoD>(ctx->D, ctx));
  }
  if (!ctx->pairs) {   // PAIRS: k_fin1p's last CTA reduces ell
    k_ell_reduce<<<1, 1024, 0, ctx->stream>>>(ctx->rl, (int)ctx->N, ctx->st);
    CHECK_LAUNCH();
  }
  ctx->rates_valid = true;
  ctx->rates_exchanged = false;
  ctx->grad_valid = false;
  ctx->lam_valid = true;
  return HAWKES_OK;
}

int run_grad(hawkes_ctx* ctx) {
  if (ctx->grad_valid) return HAWKES_OK;
  if (!ctx->order_decided && !ctx->capturing) TRY(decide_order(ctx));
  if (!ctx->capturing && !ctx->rates_valid) ++ctx->evals_same_consts;
  if (use_graph(ctx)) {
    if (!ctx->rates_valid && ctx->pairs) ctx->mirror_fresh = true;
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

// hawkes_grad_at: one launch of the captured pack + rate + gradient evaluation (gexec[3]) at
// the caller's device locations x, the gradient finalize also writing the caller's out_grad.
// Takes the graph path when the plain one would (use_graph: W = 1, same constants for >= 2
// evaluations, timing off); returns false (nothing enqueued) otherwise.
int grad_at_graph(hawkes_ctx* ctx, const double* x, double* out_grad, bool* done) {
  *done = false;
  if (ctx->multi || !ctx->pairs || !ctx->order_decided || !ctx->have_x || !use_graph(ctx))
    return HAWKES_OK;
  if (!ctx->gexec[3]) {
    TRY(capture(ctx, 3));
    ctx->at_x = nullptr;
    ctx->at_out = nullptr;
  }
  // k_pack_x(rec, x, N, npad, bad, xcopy); k_pack_x32(rec32, x, N, npad);
  // k_fin2p(part, sv, N, grad, perm, counters, W, grad2) -- only when the caller's pointers
  // changed since the last launch (an MCMC loop usually reuses its buffers)
  if (x != ctx->at_x) {
    TRY(set_node_ptr(ctx, ctx->at_pack, 1, 6, (const void* const*)&x));
    if (ctx->at_pack32) TRY(set_node_ptr(ctx, ctx->at_pack32, 1, 4, (const void* const*)&x));
    ctx->at_x = x;
  }
  if (out_grad != ctx->at_out) {
    TRY(set_node_ptr(ctx, ctx->at_fin2, 7, 8, (const void* const*)&out_grad));
    ctx->at_out = out_grad;
  }
  CU(cudaGraphLaunch(ctx->gexec[3], ctx->stream));
  ctx->launches += ctx->graph_launches[3];
  ctx->mirror_fresh = true;
  *done = true;
  return HAWKES_OK;
}

// mirror_ok: the caller enqueued nothing but evaluations since the last fetch, so when one of
// them ran k_fin1p (which writes the status into h_st) no copy is needed
int fetch_status(hawkes_ctx* ctx, bool mirror_ok = false) {
  // (ctx->bad is st->nonfinite: one copy brings the flags and the results)
  const bool mirror = mirror_ok && ctx->mirror_fresh;
  if (!mirror)
    CU(cudaMemcpyAsync(ctx->h_st, ctx->st, sizeof(EvalStatus), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->mirror_fresh = false;
  int bad = 0;
  TRY(wait_stream(ctx));
  if (mirror) memcpy((void*)ctx->h_st, (const void*)ctx->h_mirror, sizeof(EvalStatus));
  bad = ctx->h_st->nonfinite;
  if (ctx->h_st->range32) {
    CU(cudaMemsetAsync(&ctx->st->range32, 0, sizeof(int), ctx->stream));
    ctx->h_st->range32 = 0;
    if (use32(ctx)) {   // the fp32 result is not trusted: this call is redone in fp64
      ctx->fb64 = true;
      ctx->retry = true;
      drop_graphs(ctx);
      ctx->rates_valid = ctx->grad_valid = ctx->lam_valid = false;
    }
  }
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

// true once if the last fetch_status asked for the call to be redone (fp32 range guard)
bool take_retry(hawkes_ctx* ctx) {
  const bool r = ctx->retry;
  ctx->retry = false;
  return r;
}

// rates for the current state, checked against the fp32 range guard (one host sync)
int checked_rates(hawkes_ctx* ctx, bool mirror_ok = false) {
  for (;;) {
    TRY(run_rates(ctx));
    TRY(fetch_status(ctx, mirror_ok));
    if (!take_retry(ctx)) return HAWKES_OK;
  }
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

// PAIRS plan (hawkes_plan.h pairs_layout): each rank's chunk pairs (heaviest first) and its
// compact slot layout; ROWS' tile lists stay empty.
void build_plan_pairs(hawkes_ctx* ctx, std::vector<std::vector<int2>>& it1,
                      std::vector<std::vector<int2>>& it2, std::vector<std::vector<PairItem>>& sym,
                      std::vector<int>& own, std::vector<std::vector<long long>>& coff,
                      std::vector<std::vector<int>>& cn) {
  const int W = ctx->W;
  own = pair_owners(ctx->N, ctx->chunk, W);
  ctx->tiles_of.assign(W, {});
  ctx->max_tiles = 0;
  it1.assign(W, {});
  it2.assign(W, {});
  PairsLayout lay = pairs_layout(ctx->N, ctx->chunk, W, ctx->my_ranks, ctx->grid_s2);
  sym.swap(lay.items);
  coff.swap(lay.coff);
  cn.swap(lay.cn);
  ctx->slot_events = lay.slot_events;
  ctx->piece_k = lay.pieces;
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
  h.fc64 = ctx->fc64;
  CU(cudaMemcpyAsync(ctx->d_consts, &h, sizeof h, cudaMemcpyHostToDevice, ctx->stream));
  return HAWKES_OK;
}

// The fp64 pass kernels' folded constants for Theta (lnw_b / lnw_s: the log kernel weights
// times alpha / beta, returned for the range checks)
PassConst make_pass_const(const hawkes_params& p, int D, double* lnw_b_out, double* lnw_s_out) {
  const double two_pi = 6.283185307179586476925286766559;
  // background weight mu0/((2pi)^{D/2} tau_x^D * sqrt(2pi) tau_t), times alpha = 1/tau_x^2
  const double lnw_b = log(p.mu0) - 0.5 * (D + 1) * log(two_pi) - D * log(p.tau_x) - log(p.tau_t) -
                       2.0 * log(p.tau_x);
  // self-excitation weight theta omega/((2pi)^{D/2} h^D), times beta = 1/h^2
  const double lnw_s = log(p.theta) + log(p.omega) - 0.5 * D * log(two_pi) - D * log(p.sigma_x) -
                       2.0 * log(p.sigma_x);
  PassConst pc;
  pc.kx = -0.5 / (p.tau_x * p.tau_x);
  pc.kt = -0.5 / (p.tau_t * p.tau_t);
  pc.ks = -0.5 / (p.sigma_x * p.sigma_x);
  pc.omega = p.omega;
  pc.st = sqrt(-pc.kt);
  pc.oms = -p.omega / pc.st;
  pc.lnc_b = p.mu0 > 0 ? lnw_b + 64.0 * LN2 : -INFINITY;
  pc.lnc_s = p.theta > 0 ? lnw_s + 64.0 * LN2 : -INFINITY;
  pc.lnc_sr = p.theta > 0 ? lnw_s : -INFINITY;
  if (lnw_b_out) *lnw_b_out = lnw_b;
  if (lnw_s_out) *lnw_s_out = lnw_s;
  return pc;
}

// Kernel constants for Theta; written to ctx only when every check passes.
int compute_constants(hawkes_ctx* ctx, const hawkes_params& p, double tN) {
  const int D = ctx->D;
  double lnw_b = 0.0, lnw_s = 0.0;
  const PassConst pc = make_pass_const(p, D, &lnw_b, &lnw_s);
  if ((p.mu0 > 0 && !(fabs(lnw_b) < 600.0)) || (p.theta > 0 && !(fabs(lnw_s) < 600.0)))
    return set_err(ctx, HAWKES_ERR_PARAM,
                   "Theta puts the kernel constants outside the fp64 exp range (|log w| >= 600)");
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
  fc.range_floor = 0.0;
  ctx->fc64 = fc;
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
    c32.st = (float)sqrt(-pc.kt * L2E);
    c32.oms = (float)(-p.omega * L2E / sqrt(-pc.kt * L2E));
    if (!isfinite(c32.kx) || !isfinite(c32.kt) || !isfinite(c32.ks) || !isfinite(c32.omega) ||
        c32.kx == 0.f || c32.kt == 0.f || c32.ks == 0.f)
      return set_err(ctx, HAWKES_ERR_PARAM, "Theta outside the fp32 path's range");
    fc.scale_log2 = E;
    fc.zero_floor = 0.0;   // ex2.approx.ftz flushes to exact zeros
    // every flushed term is < 2^-126 in these scaled units and an event has at most N - 1
    // of them: below 2^24 N 2^-126 max(tau_x^2, h^2) the flushed mass could exceed 2^-24
    // of Lambda' (R23), and the evaluation is redone in fp64
    fc.range_floor = (double)ctx->N * ldexp(1.0, -102) * std::max(fc.tx2, fc.h2);
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
