// hawkes_launch.cuh -- part of hawkes_api.cu (one translation unit): shared-memory sizes,
// kernel variant selection, per-D launch structs (setup, passes, finalizes, packing, moves,
// MH sweep, BMDS, leapfrog) and the kernel timing hooks.
#pragma once
namespace {

// Launch with programmatic stream serialization (hawkes_kernels.cuh pdl_trigger / pdl_wait):
// the kernel's launch and prologue overlap the previous kernel's tail; under stream capture the
// edge becomes a programmatic graph edge.  Only kernels that pdl_wait before touching earlier
// kernels' output go through here.  HAWKES_PDL=0 launches them plainly (A/B).
static bool pdl_enabled() {
  static bool v = [] {
    const char* e = getenv("HAWKES_PDL");
    return !(e && atoi(e) == 0);
  }();
  return v;
}
template <typename... P, typename... A>
cudaError_t launch_pdl(void (*k)(P...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

template <int D, int PASS>
size_t pass_smem() {
  return (size_t)STAGES * TILE_J * Layout<D>::REC * sizeof(double) + STAGES * sizeof(uint64_t) +
         EXP_TABLE * sizeof(int2);
}

// diagnostics: HAWKES_SYM_CPS1 / HAWKES_SYM_CPS2 cap the sym kernels' CTAs per SM (A/B of
// the grid at small N, where the items come in few rounds)
static int sym_cps(int pass) {
  static int v[2] = {[] { const char* e = getenv("HAWKES_SYM_CPS1"); return e ? atoi(e) : 0; }(),
                     [] { const char* e = getenv("HAWKES_SYM_CPS2"); return e ? atoi(e) : 0; }()};
  return v[pass - 1];
}
static int sym_grid(const hawkes_ctx* ctx, int pass, int resident, int n_items) {
  int g = std::min(resident, n_items);
  if (sym_cps(pass) > 0) g = std::min(g, sym_cps(pass) * ctx->sms);
  return std::max(1, g);
}

template <int D, int PASS, int R, int V>
size_t sym_smem() {
  static_assert(32 * R == TILE_J, "one row tile = one column tile");
  return SymCfg<D, PASS, V>::Smem::bytes();
}

// sym_kernel variants: R rows per lane; V1 / V2 = the pass-1 / pass-2 variant bits
// (hawkes_kernels_sym.cuh).  Measured on B200 (profiles/r01_sym_variants.txt): the
// interleaved exp table pays in pass 1 (-3.4 %) but not in pass 2, where it costs more
// integer instructions than the bank conflicts it removes; the SoA columns pay in both.
template <int D, int R, int V1, int V2>
struct SymOps {
  // PIECE: the instantiation for plans of pieces (hawkes_plan.h choose_pieces; SymArgs.piece)
  template <bool PIECE>
  static int attrs(hawkes_ctx* ctx, int* b1, int* b2) {
    auto s1 = sym_kernel<D, 1, R, V1, false, PIECE>;
    auto s2 = sym_kernel<D, 2, R, V2, false, PIECE>;
    CU(cudaFuncSetAttribute(s1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym_smem<D, 1, R, V1>()));
    CU(cudaFuncSetAttribute(s2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym_smem<D, 2, R, V2>()));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(b1, s1, THREADS, sym_smem<D, 1, R, V1>()));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(b2, s2, THREADS, sym_smem<D, 2, R, V2>()));
    return HAWKES_OK;
  }
  static int setup(hawkes_ctx* ctx) {
    int b1 = 0, b2 = 0, p1 = 0, p2 = 0;
    TRY(attrs<false>(ctx, &b1, &b2));
    TRY(attrs<true>(ctx, &p1, &p2));
    ctx->grid_s1 = std::max(1, std::min(b1, p1)) * ctx->sms;
    ctx->grid_s2 = std::max(1, std::min(b2, p2)) * ctx->sms;
    return HAWKES_OK;
  }
  template <bool PIECE>
  static int go(hawkes_ctx* ctx, int pass, const SymArgs& b) {
    const int grid = sym_grid(ctx, pass, pass == 1 ? ctx->grid_s1 : ctx->grid_s2, b.n_items);
    if (pass == 1)
      CU(launch_pdl(sym_kernel<D, 1, R, V1, false, PIECE>, grid, THREADS, sym_smem<D, 1, R, V1>(), ctx->stream, b));
    else
      CU(launch_pdl(sym_kernel<D, 2, R, V2, false, PIECE>, grid, THREADS, sym_smem<D, 2, R, V2>(), ctx->stream, b));
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
  static int launch(hawkes_ctx* ctx, int pass, const SymArgs& b) {
    return b.piece ? go<true>(ctx, pass, b) : go<false>(ctx, pass, b);
  }
};

// the spatial-walk (GEN) kernels: V = 4, D <= SPACE_MAX_D
template <int D>
struct SymGen {
  static size_t smem(int pass) {
    return pass == 1 ? SymCfg<D, 1, 4, true>::Smem::bytes() : SymCfg<D, 2, 4, true>::Smem::bytes();
  }
  template <bool PIECE>
  static int attrs(hawkes_ctx* ctx, int* b1, int* b2) {
    auto g1 = sym_kernel<D, 1, 4, 4, true, PIECE>;
    auto g2 = sym_kernel<D, 2, 4, 4, true, PIECE>;
    CU(cudaFuncSetAttribute(g1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(1)));
    CU(cudaFuncSetAttribute(g2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(2)));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(b1, g1, THREADS, smem(1)));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(b2, g2, THREADS, smem(2)));
    return HAWKES_OK;
  }
  static int setup(hawkes_ctx* ctx) {
    int b1 = 0, b2 = 0, p1 = 0, p2 = 0;
    TRY(attrs<false>(ctx, &b1, &b2));
    TRY(attrs<true>(ctx, &p1, &p2));
    ctx->grid_g1 = std::max(1, std::min(b1, p1)) * ctx->sms;
    ctx->grid_g2 = std::max(1, std::min(b2, p2)) * ctx->sms;
    return HAWKES_OK;
  }
  template <bool PIECE>
  static int go(hawkes_ctx* ctx, int pass, const SymArgs& b) {
    const int grid = sym_grid(ctx, pass, pass == 1 ? ctx->grid_g1 : ctx->grid_g2, b.n_items);
    if (pass == 1)
      CU(launch_pdl(sym_kernel<D, 1, 4, 4, true, PIECE>, grid, THREADS, smem(1), ctx->stream, b));
    else
      CU(launch_pdl(sym_kernel<D, 2, 4, 4, true, PIECE>, grid, THREADS, smem(2), ctx->stream, b));
    CHECK_LAUNCH();
    return HAWKES_OK;
  }
  static int launch(hawkes_ctx* ctx, int pass, const SymArgs& b) {
    return b.piece ? go<true>(ctx, pass, b) : go<false>(ctx, pass, b);
  }
};

// default: V = 4 (SoA columns) in both passes.  The interleaved exp-table copies (V bit 2)
// cut pass 1's bank conflicts while pass 1 also accumulated the row-local gradient (-1.6 %
// with 2 copies of the 2048-entry table, -3.4 % with 16 copies of the -DHK_EXP256 table);
// since pass 1 computes the rates alone (142 registers), the copies' index arithmetic costs
// more than the conflicts (+3.3 %), as it always did in pass 2 (profiles/r01_sym_variants.txt).
// HAWKES_SYM_V = 0 / 2 / 4 / 6 forces one variant for both passes (diagnostics, A/B on one
// box; 2 and 6 exist for D = 2 only)
static int sym_variant() {
  static int v = [] {
    const char* e = getenv("HAWKES_SYM_V");
    return e ? atoi(e) : -1;
  }();
  return v;
}

template <int D, int V1, int V2>
int sym_call_v(hawkes_ctx* ctx, int pass, const SymArgs* b) {
  if (pass) return SymOps<D, 4, V1, V2>::launch(ctx, pass, *b);
  TRY((SymOps<D, 4, V1, V2>::setup(ctx)));
  return HAWKES_OK;
}

template <int D>
int sym_call(hawkes_ctx* ctx, int pass, const SymArgs* b) {
  if constexpr (D <= SPACE_MAX_D) {
    if (pass == 0) TRY(SymGen<D>::setup(ctx));
    else if (ctx->spatial) return SymGen<D>::launch(ctx, pass, *b);
  }
  const int v = sym_variant();
  if (v == 0) return sym_call_v<D, 0, 0>(ctx, pass, b);
  if constexpr (D == 2) {
    if (v == 2) return sym_call_v<D, 2, 2>(ctx, pass, b);
    if (v == 4) return sym_call_v<D, 4, 4>(ctx, pass, b);
    if (v == 6) return sym_call_v<D, 6, 6>(ctx, pass, b);
  }
  return sym_call_v<D, 4, 4>(ctx, pass, b);
}

constexpr int SYM32_R = 4;
template <int D, int PASS, bool GEN = false>
size_t sym32_smem() {
  const int KR = PASS == 1 ? (GEN ? 2 : 1) : D;
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

template <int D, bool SOA, bool GEN, bool PIECE>
int sym32_attrs(hawkes_ctx* ctx, int* b1, int* b2) {
  auto s1 = sym_kernel_f32<D, 1, SYM32_R, SOA, GEN, PIECE>;
  auto s2 = sym_kernel_f32<D, 2, SYM32_R, SOA, GEN, PIECE>;
  CU(cudaFuncSetAttribute(s1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym32_smem<D, 1, GEN>()));
  CU(cudaFuncSetAttribute(s2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sym32_smem<D, 2, GEN>()));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(b1, s1, THREADS, sym32_smem<D, 1, GEN>()));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(b2, s2, THREADS, sym32_smem<D, 2, GEN>()));
  return HAWKES_OK;
}

template <int D, bool SOA, bool GEN = false>
int sym32_setup(hawkes_ctx* ctx) {
  int b1 = 0, b2 = 0, p1 = 0, p2 = 0;
  int rc = sym32_attrs<D, SOA, GEN, false>(ctx, &b1, &b2);
  if (rc == HAWKES_OK) rc = sym32_attrs<D, SOA, GEN, true>(ctx, &p1, &p2);
  if (rc != HAWKES_OK) return rc;
  (GEN ? ctx->grid32_g1 : ctx->grid32_s1) = std::max(1, std::min(b1, p1)) * ctx->sms;
  (GEN ? ctx->grid32_g2 : ctx->grid32_s2) = std::max(1, std::min(b2, p2)) * ctx->sms;
  return HAWKES_OK;
}

template <int D, bool SOA, bool GEN, bool PIECE>
int sym32_go(hawkes_ctx* ctx, int pass, const SymArgs32& b) {
  const int grid = std::min(GEN ? (pass == 1 ? ctx->grid32_g1 : ctx->grid32_g2)
                                : (pass == 1 ? ctx->grid32_s1 : ctx->grid32_s2),
                            b.n_items);
  if (pass == 1)
    CU(launch_pdl(sym_kernel_f32<D, 1, SYM32_R, SOA, GEN, PIECE>, grid, THREADS, sym32_smem<D, 1, GEN>(), ctx->stream, b));
  else
    CU(launch_pdl(sym_kernel_f32<D, 2, SYM32_R, SOA, GEN, PIECE>, grid, THREADS, sym32_smem<D, 2, GEN>(), ctx->stream, b));
  CHECK_LAUNCH();
  return HAWKES_OK;
}

template <int D, bool SOA, bool GEN = false>
int sym32_launch(hawkes_ctx* ctx, int pass, const SymArgs32& b) {
  return b.piece ? sym32_go<D, SOA, GEN, true>(ctx, pass, b) : sym32_go<D, SOA, GEN, false>(ctx, pass, b);
}

template <int D>
size_t pass_smem32() {
  return (size_t)STAGES * TILE_J * Layout32<D>::REC * sizeof(float) + STAGES * sizeof(uint64_t);
}

// the pass kernels' resident grids alone (create, before the plan: pieces need grid_s2)
template <int D>
struct SymSetupD {
  static int run(hawkes_ctx* ctx) {
    if constexpr (D <= SYM_MAX_D) return sym_call<D>(ctx, 0, nullptr);
    return HAWKES_OK;
  }
};

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
      ctx->grid32_1 = std::max(1, b1) * ctx->sms;
      ctx->grid32_2 = std::max(1, b2) * ctx->sms;
      if constexpr (D <= SYM_MAX_D) if (ctx->pairs) {
        bool soa = true;
        if constexpr (D == 2) soa = sym32_soa();
        int rc = HAWKES_OK;
        if (soa) rc = sym32_setup<D, true>(ctx);
        else if constexpr (D == 2) rc = sym32_setup<D, false>(ctx);
        if (rc != HAWKES_OK) return rc;
        if constexpr (D <= SPACE_MAX_D) {   // the spatial walk's fp32 kernels
          rc = sym32_setup<D, true, true>(ctx);
          if (rc != HAWKES_OK) return rc;
        }
      }
      // and the fp64 kernels below: the fp32 range guard can send this context to them
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
    if (use32(ctx)) return run32(ctx, pass, rank);
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
      b.rec = ctx->spatial ? ctx->rec_p : ctx->rec;
      b.lrho = ctx->lrho;
      b.gid = ctx->spatial ? ctx->d_gid_p : ctx->gid;
      b.boxes = ctx->d_boxes;
      b.ties = ctx->ties ? 1 : 0;
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
      b.piece = ctx->piece_k[rank] > 1 ? 1 : 0;
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
      const int grid = std::min(pass == 1 ? ctx->grid32_1 : ctx->grid32_2, a.n_items);
      if (pass == 1)
        pass_kernel_f32<D, 1, R_ROWS><<<grid, THREADS, sm, ctx->stream>>>(a);
      else
        pass_kernel_f32<D, 2, R_ROWS><<<grid, THREADS, sm, ctx->stream>>>(a);
      CHECK_LAUNCH();
    }
    if constexpr (D <= SYM_MAX_D) if (ctx->pairs && ctx->n_sym[rank] > 0) {
      SymArgs32 b;
      b.rec = ctx->spatial ? ctx->rec32_p : ctx->rec32;
      b.boxes = ctx->d_boxes;
      b.ties = ctx->ties ? 1 : 0;
      b.gid = ctx->spatial ? ctx->d_gid_p : ctx->gid;
      b.items = ctx->d_sym[rank];
      b.counter = ctx->counters + 4 * rank + 2 + (pass - 1);
      b.part = pass == 1 ? ctx->part1 : ctx->part2;
      b.npad = ctx->npad;
      b.N = (int)ctx->N;
      b.n_items = ctx->n_sym[rank];
      b.chunk = ctx->chunk;
      b.nchunks = ctx->nchunks;
      b.c = ctx->pc32;
      b.piece = ctx->piece_k[rank] > 1 ? 1 : 0;
      bool soa = true;
      if constexpr (D == 2) soa = sym32_soa();
      int rc = HAWKES_OK;
      if (ctx->spatial) {
        if constexpr (D <= SPACE_MAX_D) rc = sym32_launch<D, true, true>(ctx, pass, b);
      } else if (soa)
        rc = sym32_launch<D, true>(ctx, pass, b);
      else if constexpr (D == 2)
        rc = sym32_launch<D, false>(ctx, pass, b);
      if (rc != HAWKES_OK) return rc;
    }
    record_stop(ctx, pass == 1);
    return HAWKES_OK;
  }
};

// k_fin1p lets the gradient pass launch at its start when that pass's grid is the full
// resident grid on every rank of this process (its items fill all SM slots)
static bool early_pass2(const hawkes_ctx* ctx) {
  const int resident = use32(ctx) ? (ctx->spatial ? ctx->grid32_g2 : ctx->grid32_s2)
                                  : (ctx->spatial ? ctx->grid_g2 : ctx->grid_s2);
  for (int r : ctx->my_ranks)
    if (ctx->n_sym[r] < resident) return false;
  return resident > 0;
}

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
    // rho' into both records (an fp32 context can switch to the fp64 kernels)
    double* rr = final_here ? ctx->rec + Layout<D>::RHO : nullptr;
    float* rr32 = final_here && ctx->rec32 ? ctx->rec32 + Layout32<D>::RHO : nullptr;
    const FinConst* fcp = use32(ctx) ? &ctx->d_consts->fc : &ctx->d_consts->fc64;
    if (all) {   // PAIRS: (M', X') partials, gradient from pass 2 alone
      static_assert(K1P == 2, "k_fin1p pairs (M', X') lanes");
      const long long n = 2 * ctx->N;
      CU(launch_pdl(k_fin1p<D>, (unsigned)((n + 31) / 32), FINP_THREADS, 0, ctx->stream,
          (const double*)(sums ? ctx->sums1 : ctx->part1),
          sums ? SlotView{nullptr, nullptr, ctx->chunk} : SlotView{ctx->d_coff[0], ctx->d_cn[0], ctx->chunk},
          (int)ctx->N, ctx->rec,
          ctx->rl, ctx->rates, fcp, rr, rr32, ctx->ell_part,
          ctx->counters + 4 * ctx->W, ctx->st, (final_here && SYM_FOLD) ? ctx->lrho : nullptr,
          ctx->spatial ? WalkMap{ctx->d_perm, ctx->rec_p + Layout<D>::RHO,
                                 ctx->rec32_p ? ctx->rec32_p + Layout32<D>::RHO : nullptr}
                       : WalkMap{nullptr, nullptr, nullptr},
          ctx->d_mirror, ctx->counters, ctx->W, early_pass2(ctx) ? 1 : 0));
      ctx->mirror_fresh = true;
    } else {     // ROWS: (M', X', G1') partials of this rank's row tiles
      k_fin1<D, Layout<D>::K1, true><<<nt, FIN_THREADS, 0, ctx->stream>>>(
          ctx->part1, ctx->npad, ctx->nslots, ctx->d_tiles[rank], (int)ctx->N, ctx->rec, ctx->G1,
          ctx->rl, ctx->rates, fcp, rr, rr32, &ctx->st->range32);
    }
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
    if (all) {
      const long long n = ctx->N * D;
      CU(launch_pdl(k_fin2p<D>, (unsigned)((n + 31) / 32), FINP_THREADS, 0, ctx->stream,
          (const double*)(sums ? ctx->sums2 : ctx->part2),
          sums ? SlotView{nullptr, nullptr, ctx->chunk} : SlotView{ctx->d_coff[0], ctx->d_cn[0], ctx->chunk},
          (int)ctx->N, ctx->grad,
          (const int*)(ctx->spatial ? ctx->d_perm : nullptr), ctx->counters, ctx->W, (double*)nullptr));
    } else {
      k_fin2<D, true><<<nt, FIN_THREADS, 0, ctx->stream>>>(ctx->part2, ctx->npad, ctx->nslots,
                                                           ctx->d_tiles[rank], (int)ctx->N, ctx->G1,
                                                           ctx->rl, ctx->grad);
    }
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
  static int run(hawkes_ctx* ctx, const double* xdev, double* xcopy = nullptr) {
    k_pack_x<D><<<(ctx->npad + 255) / 256, 256, 0, ctx->stream>>>(ctx->rec, xdev, (int)ctx->N,
                                                                  ctx->npad, ctx->bad, xcopy);
    CHECK_LAUNCH();
    if (ctx->rec32) {
      k_pack_x32<D><<<(ctx->npad + 255) / 256, 256, 0, ctx->stream>>>(ctx->rec32, xdev,
                                                                      (int)ctx->N, ctx->npad);
      CHECK_LAUNCH();
    }
    return HAWKES_OK;
  }
};

// hawkes_grad_at's graph (hawkes_engine.cuh capture, which = 3): its location-packing and
// gradient-finalize kernel nodes, found by kernel function
template <int D>
struct AtNodesD {
  static int run(hawkes_ctx* ctx) {
    size_t n = 0;
    CU(cudaGraphGetNodes(ctx->g_at, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    CU(cudaGraphGetNodes(ctx->g_at, nodes.data(), &n));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType ty;
      CU(cudaGraphNodeGetType(nd, &ty));
      if (ty != cudaGraphNodeTypeKernel) continue;
      cudaKernelNodeParams kp;
      CU(cudaGraphKernelNodeGetParams(nd, &kp));
      if (kp.func == (void*)k_pack_x<D>) ctx->at_pack = nd;
      else if (kp.func == (void*)k_pack_x32<D>) ctx->at_pack32 = nd;
      else if (kp.func == (void*)k_fin2p<D>) ctx->at_fin2 = nd;
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
    a.rates = ctx->rates;
    a.tx2 = ctx->fc.tx2;
    a.h2 = ctx->fc.h2;
    a.floor_ = fcur(ctx).zero_floor;
    a.part = ctx->d_move_part;
    // one launch for the rows outside S (with their Delta-ell terms) and the moved rows, one
    // CTA for the moved events' terms and the fixed-order sum (decide: the MH sweep's
    // Metropolis decision in the same kernel)
    const int nb = (int)((ctx->N + 255) / 256);
    const int len = move_split_len((int)ctx->N);
    const int nsplit = (int)((ctx->N + len - 1) / len);
    k_move_delta_rows<D><<<(unsigned)(nb + k * nsplit), 256, move_smem_bytes<D>(k), ctx->stream>>>(
        a, ctx->tab, ctx->d_move_delta, ctx->d_move_rows_part, nb, nsplit);
    CHECK_LAUNCH();
    k_move_terms_final<<<1, MOVE_FINAL_THREADS, 0, ctx->stream>>>(ctx->rates, ctx->d_move_rows_part, nsplit,
                                                   ctx->d_move_idx, k, ctx->d_move_part, nb,
                                                   ctx->fc.tx2, ctx->fc.h2, fcur(ctx).zero_floor,
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
    a.stamp = ctx->d_mh_stamp;
    a.gtab = ctx->tab;
    a.c = ctx->pc;
    a.tx2 = ctx->fc.tx2;
    a.h2 = ctx->fc.h2;
    a.floor_ = fcur(ctx).zero_floor;
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
      k_bmds_sym_fin<D><<<(unsigned)(((long long)N * (D + 1) + 255) / 256), 256, 0, ctx->stream>>>(ctx->d_bpart, N, ctx->d_bgrad, ctx->d_brow);
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

// spatial walk: gather the records in walk order and the tile boxes (every evaluation)
template <int D>
struct WalkD {
  static int run(hawkes_ctx* ctx) {
    k_walk_records<D><<<(unsigned)(ctx->npad / 128), 128, 0, ctx->stream>>>(
        ctx->rec, ctx->d_perm, (int)ctx->N, ctx->npad, ctx->rec_p, ctx->d_boxes);
    CHECK_LAUNCH();
    if (ctx->rec32_p) {
      k_walk_records32<D><<<(unsigned)(ctx->npad / 128), 128, 0, ctx->stream>>>(
          ctx->rec32, ctx->d_perm, (int)ctx->N, ctx->npad, ctx->rec32_p);
      CHECK_LAUNCH();
    }
    return HAWKES_OK;
  }
};

}  // namespace
