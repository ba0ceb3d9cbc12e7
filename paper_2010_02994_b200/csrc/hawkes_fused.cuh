// hawkes_fused.cuh -- one cooperative launch for a whole ell + gradient evaluation at small N
// (PAIRS, fp64, one process).  SURVEY.md §8(a) S2-S5 in four grid-synchronised phases:
//   pass 1 (sym_items<PASS=1>) | fin1 (fin1p_block: slot sums, lambda, rho', Lambda_n, ell_n,
//   fixed-order ell) | pass 2 (sym_items<PASS=2>) | fin2 (fin2p_block: gradient slot sums)
// with exactly the arithmetic and summation order of the four separate launches (bitwise the
// same results), but one launch, one exp-table load per CTA and no launch gaps.  At the
// paper's catalog sizes (N ~ 3-5k) the passes are ~2 items per CTA and the
// launches, finalize kernels and tails were a third of an evaluation.
#pragma once
#include <cooperative_groups.h>

#include "hawkes_kernels_sym.cuh"
#include "hawkes_ops.cuh"

namespace hk {

struct FusedArgs {
  SymArgs s1, s2;                 // the two passes' item walks (counters zeroed before launch)
  int nslots;                     // C + 1 partial slots per event
  const FinConst* fcp;
  double* rl;                     // (rho', ell_n)
  double* rates;                  // (lambda, mu, xi, Lambda)
  double* rec_rho;                // rho' into the records (read by pass 2)
  float* rec32_rho;               // and the fp32 records' (an fp32 context in its fp64 fallback)
  double* ell_part;
  int* ticket;
  EvalStatus* st;
  double* lrho;                   // -DHK_SYM_FOLD only
  double* grad;
};

// generic-proxy stores (rho' in the records) -> later bulk-copy (async-proxy) reads
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int D, int V>
__global__ void __launch_bounds__(THREADS, D <= 4 ? 3 : 2) sym_eval_fused(FusedArgs f) {
  namespace cg = cooperative_groups;
  using C2 = SymCfg<D, 2, V>;
  static_assert(SymCfg<D, 1, V>::TS == C2::TS && SymCfg<D, 1, V>::SOAW <= C2::SOAW &&
                    SymCfg<D, 1, V>::KR <= C2::KR,
                "pass 2's shared-memory layout holds pass 1's");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const typename C2::Smem sm(smem_raw);
  __shared__ int s_item;
  cg::grid_group grid = cg::this_grid();
  sym_prologue<C2::TS>(f.s1.tab, sm.tab, sm.bars);
  uint32_t parity = 0;
  const int N = f.s1.N;

  sym_items<D, 1, 4, V>(f.s1, sm, &s_item, parity);                     // S2 rate pass
  grid.sync();
  const int nb1 = (int)((2LL * N + 31) / 32);                            // S3 finalize
  for (int b = blockIdx.x; b < nb1; b += gridDim.x)
    fin1p_block<D>(b, nb1, f.s1.part, f.s1.npad, f.nslots, N, f.s1.rec, f.rl, f.rates, f.fcp,
                   f.rec_rho, f.rec32_rho, f.ell_part, f.ticket, f.st, f.lrho);
  fence_proxy_async_global();
  grid.sync();
  fence_proxy_async_global();
  sym_items<D, 2, 4, V>(f.s2, sm, &s_item, parity);                     // S5 gradient pass
  grid.sync();
  const int nb2 = (int)(((long long)N * D + 31) / 32);
  for (int b = blockIdx.x; b < nb2; b += gridDim.x)
    fin2p_block<D>(b, f.s2.part, f.s2.npad, f.nslots, N, f.grad);
}

}  // namespace hk
