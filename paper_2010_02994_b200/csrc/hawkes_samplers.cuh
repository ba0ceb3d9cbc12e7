// hawkes_samplers.cuh -- part of hawkes_api.cu (one translation unit, included inside its
// extern "C" block): the HMC leapfrog and transition, block-MH moves and the on-device MH
// sweep, the BMDS density and the HMC potential selection.
#pragma once
extern "C++" {
// leapfrog buffers + the optional diagonal inverse mass and box, copied in (per mem)
static int lf_prepare(hawkes_ctx* ctx, int32_t mem, const double* inv_mass, const double* box_lo,
                      const double* box_hi) {
  const size_t n = (size_t)ctx->N * ctx->D;
  if (!ctx->lf_x) {
    int rc;
    if ((rc = dalloc(ctx, &ctx->lf_x, n)) || (rc = dalloc(ctx, &ctx->lf_p, n)) ||
        (rc = dalloc(ctx, &ctx->lf_x0, n)) || (rc = dalloc(ctx, &ctx->lf_p0, n)))
      return rc;
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
  TRY(copy_in(ctx, ctx->lf_x0, x, n, mem));
  TRY(copy_in(ctx, ctx->lf_p0, p, n, mem));
  TRY(clear_move(ctx));
  do {   // twice only if the fp32 range guard sent the context to fp64 during the trajectory
    CU(cudaMemcpyAsync(ctx->lf_x, ctx->lf_x0, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaMemcpyAsync(ctx->lf_p, ctx->lf_p0, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    CU(cudaMemsetAsync(&ctx->st->undefined, 0, sizeof(int), ctx->stream));
    TRY(dispatchD<PackXD>(ctx->D, ctx, (const double*)ctx->lf_x));
    ctx->have_x = true;
    ctx->rates_valid = ctx->grad_valid = false;
    TRY(lf_core(ctx, step, n_steps, inv_mass != nullptr, box_lo != nullptr, [] { return HAWKES_OK; }));
    CU(cudaMemcpyAsync(ctx->xstage, ctx->lf_x, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    TRY(copy_out(ctx, x, ctx->lf_x, n, mem));
    TRY(copy_out(ctx, p, ctx->lf_p, n, mem));
    TRY(fetch_status(ctx));
  } while (take_retry(ctx));
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
  take_retry(ctx);          // (a guard trip seen here only invalidates the cached rates)
  const size_t n = (size_t)ctx->N * ctx->D;
  TRY(lf_prepare(ctx, mem, inv_mass, box_lo, box_hi));
  TRY(clear_move(ctx));
  const uint2 key = make_uint2((unsigned)seed, (unsigned)(seed >> 32));
  // the chain's state, kept for an fp64 re-run of the transition (fp32 range guard)
  CU(cudaMemcpyAsync(ctx->lf_x0, ctx->xstage, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  for (;;) {
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
    if (!take_retry(ctx)) break;
    // the fp32 range guard tripped in the trajectory: the same transition (same momenta and
    // uniform) again with the fp64 kernels, from the saved state
    CU(cudaMemcpyAsync(ctx->xstage, ctx->lf_x0, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    TRY(dispatchD<PackXD>(ctx->D, ctx, (const double*)ctx->xstage));
  }
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
    TRY(wait_stream(ctx));
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
    TRY(wait_stream(ctx));
  } else {
    memcpy(hx.data(), new_x, hx.size() * sizeof(double));
  }
  for (double v : hx)
    if (!finite_bounded(v)) return set_err(ctx, HAWKES_ERR_NONFINITE, "proposed location not finite");
  TRY(clear_move(ctx));
  if (!ctx->lam_valid) {
    ctx->rates_valid = false;
    // fp32: one host sync to check the range guard before the moves use these rates
    TRY(use32(ctx) ? checked_rates(ctx) : run_rates(ctx));
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
  TRY(wait_stream(ctx));
  return HAWKES_OK;
}

int hawkes_get_locations(hawkes_ctx* ctx, double* out_x, int32_t mem) {
  ENTER(ctx);
  if (!out_x || (mem != HAWKES_MEM_HOST && mem != HAWKES_MEM_DEVICE))
    return set_err(ctx, HAWKES_ERR_ARG, "bad arguments to hawkes_get_locations");
  if (!ctx->have_x) return set_err(ctx, HAWKES_ERR_STATE, "no locations");
  TRY(copy_out(ctx, out_x, ctx->xstage, (size_t)ctx->N * ctx->D, mem));
  TRY(wait_stream(ctx));
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
    TRY(wait_stream(ctx));
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
  TRY(wait_stream(ctx));
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
    // fp32: one host sync to check the range guard before the moves use these rates
    TRY(use32(ctx) ? checked_rates(ctx) : run_rates(ctx));
    if (!ctx->pairs && !ctx->rates_exchanged) {
      TRY(exchange_rows(ctx, ctx->rates, 4));
      ctx->rates_exchanged = true;
    }
  }
  // the sweep's parameters live on the device (EvalStatus mh_*), staged through the pinned
  // status block: one block step (propose, Delta ell, terms + decision, gated commit) then
  // serves every block, as plain launches or as one captured graph replayed per block
  TRY(wait_stream(ctx));   // h_st is free to stage
  ctx->h_st->mh_it = iteration;
  ctx->h_st->mh_scale = scale;
  ctx->h_st->mh_key_lo = (unsigned)seed;
  ctx->h_st->mh_key_hi = (unsigned)(seed >> 32);
  ctx->h_st->mh_block = 0;
  ctx->h_st->mh_cur = 0;
  ctx->h_st->mh_prevk = 0;
  const size_t off = offsetof(EvalStatus, mh_it), len = offsetof(EvalStatus, mh_prevk) + sizeof(int) - off;
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
  TRY(wait_stream(ctx));
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
