// hawkes_ops.cuh -- the O(N) device kernels around the two O(N^2) passes: staging of the
// event records, the finalize steps (chunk-slot reductions, lambda, rho', Lambda_n, ell_n),
// exchange packing, block-move bookkeeping, leapfrog updates, deterministic reductions and
// the FP64 / exp diagnostics.  Included by hawkes_api.cu only (one translation unit).
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "hawkes_kernels.cuh"
#include "hawkes_kernels_f32.cuh"
#include "hawkes_moves.cuh"

namespace hk {

constexpr int R_ROWS = 2;                    // rows per thread
constexpr int SYM_MAX_D = 8;                 // unordered-pair kernels are built for every D
constexpr int SYM_AUTO_MAX_D = 8;            // ... and chosen by HAWKES_ALGO_AUTO up to this D
constexpr int SPACE_MAX_D = 4;               // spatial walk order (GEN kernels) built for D <= 4
                                             // (2x ROWS at N = 4733, >= ROWS at 20k for D <= 7;
                                             // profiles/r01_ab_algo.jsonl)
constexpr int RT = THREADS * R_ROWS;         // rows per row tile
constexpr int FIN_THREADS = RT;              // finalize: one thread per row of a tile
constexpr double LN2 = 0.693147180559945309417232121458;

// --------------------------------------------------------------------- O(N) kernels
// xcopy (optional): also keep the locations in the context's N x D copy (device input to
// set_locations: one pass over the user's array instead of a copy and a pass)
template <int D>
__global__ void k_pack_x(double* __restrict__ rec, const double* __restrict__ x, int N, int npad,
                         int* __restrict__ bad, double* __restrict__ xcopy) {
  using L = Layout<D>;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npad) return;
  const int src = min(i, N - 1);   // padding rows replicate the last event (never stored)
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double v = x[(long long)src * D + d];
    if (!(fabs(v) <= 1e100)) atomicOr(bad, 1);
    rec[(long long)i * L::REC + d] = v;
    if (xcopy && i < N) xcopy[(long long)i * D + d] = v;
  }
}

template <int D>
__global__ void k_pack_t(double* __restrict__ rec, const double* __restrict__ t, int N, int npad) {
  using L = Layout<D>;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npad) return;
  rec[(long long)i * L::REC + L::T] = t[min(i, N - 1)];
  rec[(long long)i * L::REC + L::RHO] = 0.0;
#pragma unroll
  for (int k = D + 2; k < L::REC; ++k) rec[(long long)i * L::REC + k] = 0.0;
}

// fp32 records: hi/lo float splits (v = hi + lo to ~48 bits)
template <int D>
__global__ void k_pack_x32(float* __restrict__ rec, const double* __restrict__ x, int N, int npad) {
  using L = Layout32<D>;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npad) return;
  const int src = min(i, N - 1);
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double v = x[(long long)src * D + d];
    const float hi = (float)v;
    rec[(long long)i * L::REC + L::XH + d] = hi;
    rec[(long long)i * L::REC + L::XL + d] = (float)(v - (double)hi);
  }
}

template <int D>
__global__ void k_pack_t32(float* __restrict__ rec, const double* __restrict__ t, int N, int npad) {
  using L = Layout32<D>;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npad) return;
  const double v = t[min(i, N - 1)];
  const float hi = (float)v;
  rec[(long long)i * L::REC + L::TH] = hi;
  rec[(long long)i * L::REC + L::TL] = (float)(v - (double)hi);
  for (int k = L::RHO; k < L::REC; ++k) rec[(long long)i * L::REC + k] = 0.f;
}

// The slot blocks of event i's chunk c in a rank's compact slot array (PairItem): cn[c] blocks
// of `chunk` events from event offset coff[c], in ascending slot id.  coff == nullptr: one
// event-major slot (the exchanged per-event sums of W > 1).
struct SlotView {
  const long long* coff;
  const int* cn;
  int chunk;
};

// PAIRS with W > 1: per event, the fixed-order sum of the slots this rank computed.
__global__ void k_slot_sum(const double* __restrict__ part, SlotView sv, int K, int N,
                           double* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)N * K) return;
  const int i = (int)(idx / K), k = (int)(idx % K);
  const int c = i / sv.chunk;
  const double* p = part + (sv.coff[c] + (i - c * sv.chunk)) * K + k;
  const long long stride = (long long)sv.chunk * K;
  double v = 0.0;
  for (int s = 0; s < sv.cn[c]; ++s) v += p[s * stride];
  out[idx] = v;
}

// emulated ranks: the "allreduce" of their per-event sums, in rank order
__global__ void k_sum_ranks(const double* __restrict__ in, long long stride, int W, long long n,
                            double* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  double v = in[idx];
  for (int r = 1; r < W; ++r) v += in[r * stride + idx];
  out[idx] = v;
}

struct FinConst {
  double tx2, h2;         // tau_x^2, h^2
  double mu0, tau_t, theta, omega, tN;
  double scale_log2;      // pair sums carry 2^-scale_log2: -64 (fp64 path) or E (fp32 path)
  double zero_floor;      // Lambda' at or below this is lambda = 0 (fexp clamps at e^-707)
  // fp32 range guard (reading R23): a Lambda' below this may have lost more than
  // 2^-24 of its value to terms that ex2.approx.ftz flushed to 0 (each < 2^-126 in the
  // kernels' scaled units, at most N of them per event); the evaluation is then redone by the
  // fp64 kernels.  0 on the fp64 path.
  double range_floor;
};

// kernel constants live in device memory so captured CUDA graphs survive set_params
struct DevConsts {
  PassConst pc;
  PassConst32 pc32;
  FinConst fc;     // constants of the context's precision
  FinConst fc64;   // the fp64 kernels' (an fp32 context after its range guard tripped)
};

// device-side evaluation status (ell, flags, HMC / MH state), one per context
struct EvalStatus {
  double ell;
  int nonfinite;   // device-side input validation failed
  int undefined;   // some evaluation produced ell = -inf inside a leapfrog trajectory
  double kinetic;
  double dell;     // Delta ell of the pending block move
  double bmds;     // BMDS log density of the last BMDS evaluation
  // HMC transition (hawkes_hmc_step)
  double lp0;      // log density at the chain's current state
  double kin0;     // 1/2 sum Minv p0^2
  double log_alpha;
  int accepted;
  int undef0;      // ell(x0) = -inf: the chain's state has zero density
  double mh_hastings;   // block MH: sum of the proposal's log Hastings terms
  // block MH sweep parameters, device-resident so one captured block step serves every block
  unsigned long long mh_it;
  double mh_scale;
  unsigned mh_key_lo, mh_key_hi;
  int mh_block;         // next block of the sweep
  int mh_cur;           // block being processed
  int mh_prevk;         // proposal slots of the previous block still set (cleared by propose)
  int range32;          // fp32 range guard tripped (FinConst::range_floor) in some evaluation
};

// Where the pair kernels walked the events in spatial order (hawkes_plan.h), the per-event
// partial slots are indexed by walk position p and perm[p] is the event; nullptr: identity.
struct WalkMap {
  const int* perm;       // p -> event
  double* recp_rho;      // rho' of the walk-order records (pass 2 reads them), or nullptr
  float* recp32_rho;     // and of the fp32 walk-order records, or nullptr
};

// lambda, rho' and ell_n of the event at walk position p from its summed pass-1 partials
// (M', X'), then the stores (event i = perm[p]): rl[i] = (rho'_i, ell_i); rates[i] = (lambda,
// mu, xi, Lambda); rho' into the records; returns ell_i
template <int D>
__device__ __forceinline__ double fin1_event(int p, double M, double X, const double* __restrict__ rec,
                                           double* __restrict__ rl, double* __restrict__ rates,
                                           const FinConst& f, double* __restrict__ rec_rho,
                                           float* __restrict__ rec32_rho, int* __restrict__ range_flag,
                                           double* __restrict__ lrho, WalkMap wm = WalkMap{nullptr, nullptr, nullptr}) {
  using L = Layout<D>;
  const int i = wm.perm ? wm.perm[p] : p;
  HK_CHECK(i >= 0 && p >= 0);
  // Lambda' = 2^64 lambda = M' tau_x^2 + X' h^2 (undo the alpha / beta folded into the exps)
  const double mu_s = M * f.tx2, xi_s = X * f.h2;
  if (mu_s + xi_s < f.range_floor) *range_flag = 1;   // fp32 only (range_floor = 0 in fp64)
  const double Lp = (mu_s + xi_s > f.zero_floor) ? mu_s + xi_s : 0.0;
  const double rho = (Lp > 0.0) ? 1.0 / Lp : 0.0;
  const double sc = exp2(f.scale_log2);   // exact power of two
  // Lambda_n: mu0 (Phi(a) - Phi(b)) - theta (e^{-omega (t_N - t_n)} - 1),
  // a = (t_N - t_n)/tau_t >= 0, b = -t_n/tau_t <= 0, Phi(a) - Phi(b) = 1 - Q(a) - Q(-b),
  // Q(z) = erfc(z/sqrt2)/2 (reading R10: same value without cancellation)
  const double tn = rec[(long long)i * L::REC + L::T];
  const double qa = 0.5 * erfc((f.tN - tn) / f.tau_t * 0.70710678118654752440);
  const double qb = 0.5 * erfc(tn / f.tau_t * 0.70710678118654752440);
  const double Lam = f.mu0 * ((1.0 - qa) - qb) - f.theta * expm1(-f.omega * (f.tN - tn));
  const double ell = (Lp > 0.0) ? (log(Lp) + f.scale_log2 * LN2) - Lam : -INFINITY;
  rl[2 * (long long)i] = rho;
  rl[2 * (long long)i + 1] = ell;
  // -ln lambda_i for the unordered-pair gradient pass (folded into its self-excitation
  // exponent; -inf where rho' = 0).  lambda = Lambda' 2^scale is exact unless it underflows
  if (lrho) {
    const double lam = Lp * sc;
    lrho[p] = !(Lp > 0.0) ? -INFINITY
              : (lam >= 2.2250738585072014e-308 ? -log(lam) : -(log(Lp) + f.scale_log2 * LN2));
  }
  // every row is final on this process (W = 1 or PAIRS): write rho' into the records here
  if (rec_rho) rec_rho[(long long)i * L::REC] = rho;
  if (wm.recp_rho) wm.recp_rho[(long long)p * L::REC] = rho;
  if (wm.recp32_rho) wm.recp32_rho[(long long)p * Layout32<D>::REC] = (float)rho;
  if (rec32_rho) rec32_rho[(long long)i * Layout32<D>::REC] = (float)rho;
  rates[4 * (long long)i] = Lp * sc;
  rates[4 * (long long)i + 1] = mu_s * sc;
  rates[4 * (long long)i + 2] = xi_s * sc;
  rates[4 * (long long)i + 3] = Lam;
  return ell;
}

// Fixed-order chunk reduction of pass-1 partials for the rows of one row tile, then
// fin1_event.  K: partial stride (Layout<D>::K1 = (M', X', G1') for ROWS; 2 = (M', X') for
// PAIRS, whose gradient comes out of pass 2 alone); HAS_G1: also sum and store the row-local G1'.
template <int D, int K, bool HAS_G1>
__global__ void k_fin1(const double* __restrict__ part, long long npad, int nchunks,
                       const int* __restrict__ tiles, int N, const double* __restrict__ rec,
                       double* __restrict__ G1, double* __restrict__ rl,
                       double* __restrict__ rates, const FinConst* __restrict__ fcp,
                       double* __restrict__ rec_rho, float* __restrict__ rec32_rho,
                       int* __restrict__ range_flag) {
  const int i = tiles[blockIdx.x] * RT + threadIdx.x;
  if (i >= N) return;
  double M = 0.0, X = 0.0, G[D];
#pragma unroll
  for (int d = 0; d < D; ++d) G[d] = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const double* p = part + ((long long)c * npad + i) * K;
    M += p[0];
    X += p[1];
    if (HAS_G1) {
#pragma unroll
      for (int d = 0; d < D; ++d) G[d] += p[2 + d];
    }
  }
  if (HAS_G1) {
#pragma unroll
    for (int d = 0; d < D; ++d) G1[(long long)i * D + d] = G[d];
  }
  fin1_event<D>(i, M, X, rec, rl, rates, *fcp, rec_rho, rec32_rho, range_flag, nullptr);
}

// PAIRS finalizes (every event final on this process): one warp-lane per (event, component)
// so a warp's loads of one slot are contiguous, and the slots split over the CTA's
// FINP_SPLIT warps (warp w sums its contiguous slot range in index order; warp 0 adds the
// FINP_SPLIT range sums in warp order): a fixed summation order, so results are bitwise
// reproducible.  At N = 5000 (41 slots) one thread per (event, component) walking all slots
// took 8.2 / 8.8 us on 78 / 79 CTAs (latency-bound); the split runs 4x the loads in flight.
constexpr int FINP_SPLIT = 4;
constexpr int FINP_THREADS = 32 * FINP_SPLIT;

__device__ __forceinline__ double finp_slot_sum(const double* __restrict__ p, long long stride,
                                                int nslots, bool live) {
  const int per = (nslots + FINP_SPLIT - 1) / FINP_SPLIT;
  const int w = threadIdx.x >> 5;
  const int c0 = w * per, c1 = min(nslots, c0 + per);
  double acc = 0.0;
  if (live) {
    // loads in batches of 16 ahead of their adds (one L2 round trip per batch instead of one
    // per 4 slots), the adds in slot order: the same sum, bit for bit
    constexpr int B = 16;
    int c = c0;
    for (; c + B <= c1; c += B) {
      double v[B];
#pragma unroll
      for (int u = 0; u < B; ++u) v[u] = __ldcg(p + (c + u) * stride);   // L2: written by other CTAs
#pragma unroll
      for (int u = 0; u < B; ++u) acc += v[u];
    }
    if (c < c1) {
      double v[B];
#pragma unroll
      for (int u = 0; u < B; ++u) v[u] = c + u < c1 ? __ldcg(p + (c + u) * stride) : 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u)
        if (c + u < c1) acc += v[u];
    }
  }
  __shared__ double sh[FINP_SPLIT][32];
  sh[w][threadIdx.x & 31] = acc;
  __syncthreads();
  double tot = sh[0][threadIdx.x & 31];
#pragma unroll
  for (int k = 1; k < FINP_SPLIT; ++k) tot += sh[k][threadIdx.x & 31];
  return tot;   // meaningful in warp 0
}

// ... and the ell reduction (S3): each CTA sums its 16 events' ell_i in lane order into
// ell_part[block]; the CTA that draws the last ticket sums ell_part in a fixed order (thread
// k: blocks k, k + 128, ...; then a fixed shared-memory tree) into st->ell and re-arms the
// ticket.  Replaces k_ell_reduce (one launch and a one-CTA pass over N) on the PAIRS path.
template <int D>
__device__ __forceinline__ void fin1p_block(int blk, int nblk, const double* __restrict__ part,
                                            SlotView sv, int N,
                                            const double* __restrict__ rec, double* __restrict__ rl,
                                            double* __restrict__ rates, const FinConst* __restrict__ fcp,
                                            double* __restrict__ rec_rho, float* __restrict__ rec32_rho,
                                            double* __restrict__ ell_part, int* ticket, EvalStatus* st,
                                            double* __restrict__ lrho, WalkMap wm,
                                            EvalStatus* mirror = nullptr) {
  const long long q = (long long)blk * 32 + (threadIdx.x & 31);   // (walk position, M' or X')
  const int i = (int)(q >> 1);
  // K1P = 2 partials per event
  const double* p0 = part + q;
  long long stride = 0;
  int nslots = 1;
  if (sv.coff) {
    const int c = min(i, N - 1) / sv.chunk;
    p0 = part + (sv.coff[c] + (i - c * sv.chunk)) * 2 + (q & 1);
    stride = (long long)sv.chunk * 2;
    nslots = sv.cn[c];
  }
  const double M = finp_slot_sum(p0, stride, nslots, i < N);
  __shared__ int last;
  __shared__ double red[FINP_THREADS];
  if (threadIdx.x < 32) {
    const double X = __shfl_down_sync(0xffffffffu, M, 1);
    double e = 0.0;
    if (i < N && (threadIdx.x & 1) == 0)
      e = fin1_event<D>(i, M, X, rec, rl, rates, *fcp, rec_rho, rec32_rho, &st->range32, lrho, wm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_down_sync(0xffffffffu, e, o);
    __threadfence();   // every lane: its range flag before the ticket (the mirror reads it)
    __syncwarp();
    if (threadIdx.x == 0) {
      ell_part[blk] = e;
      __threadfence();
      last = atomicAdd(ticket, 1) == nblk - 1;
    }
  }
  __syncthreads();
  if (last) {   // CTA-uniform
    __threadfence();
    // fixed order: thread k sums blocks k, k + 128, ...; a shuffle-down tree in each warp; the
    // FINP_SPLIT warp sums in warp order (one barrier instead of a 7-level shared-memory tree)
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += FINP_THREADS) s += __ldcg(ell_part + b);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = red[0];
#pragma unroll
      for (int w = 1; w < FINP_SPLIT; ++w) tot += red[w];
      st->ell = tot;
      if (!(tot > -INFINITY)) st->undefined = 1;
      *ticket = 0;
      __threadfence();
    }
    if (mirror) {   // the status into the caller's pinned host copy (no device-to-host copy)
      __syncthreads();
      constexpr int NW = (int)(sizeof(EvalStatus) / sizeof(int));
      static_assert(sizeof(EvalStatus) % sizeof(int) == 0, "EvalStatus is copied in words");
      const int* src = reinterpret_cast<const int*>(st);
      volatile int* dst = reinterpret_cast<volatile int*>(mirror);
      // (no system fence: the host reads it after the stream has completed)
      for (int k = threadIdx.x; k < NW; k += FINP_THREADS) dst[k] = __ldcg(src + k);
    }
  }
  __syncthreads();   // last / red reused by the caller's next block
}

template <int D>
__global__ void __launch_bounds__(FINP_THREADS) k_fin1p(const double* __restrict__ part, SlotView sv,
                                                        int N, const double* __restrict__ rec,
                                                        double* __restrict__ rl, double* __restrict__ rates,
                                                        const FinConst* __restrict__ fcp,
                                                        double* __restrict__ rec_rho,
                                                        float* __restrict__ rec32_rho,
                                                        double* __restrict__ ell_part, int* ticket,
                                                        EvalStatus* st, double* __restrict__ lrho,
                                                        WalkMap wm, EvalStatus* mirror,
                                                        int* counters, int W, int early) {
  // early: the gradient pass's grid fills every SM slot, so its CTAs may launch (and stage
  // the exp table) while this kernel runs; else at the end (a small grid launched early gets
  // packed onto busy SMs: N = 2000, +11 us per call)
  if (early) pdl_trigger();
  pdl_wait();
  // re-arm the pass-1 item counters of the W logical ranks (hawkes_engine.cuh run_rates: the
  // PAIRS path has no counter memset; pass 1 is complete here, pass 2's counters untouched)
  if (counters && blockIdx.x == 0 && threadIdx.x < W) counters[4 * threadIdx.x + 2] = 0;
  fin1p_block<D>(blockIdx.x, gridDim.x, part, sv, N, rec, rl, rates, fcp, rec_rho, rec32_rho,
                 ell_part, ticket, st, lrho, wm, mirror);
  if (!early) pdl_trigger();
}

template <int D>
__device__ __forceinline__ void fin2p_block(int blk, const double* __restrict__ part, SlotView sv,
                                            int N, double* __restrict__ grad,
                                            const int* __restrict__ perm,
                                            double* __restrict__ grad2 = nullptr) {
  constexpr int K = Layout<D>::K2;
  const long long q = (long long)blk * 32 + (threadIdx.x & 31);   // (walk position, d)
  const bool live = q < (long long)N * D;
  const int p = (int)(q / D), d = (int)(q % D);
  const double* p0 = part + (long long)p * K + d;
  long long stride = 0;
  int nslots = 1;
  if (sv.coff) {
    const int c = min(p, N - 1) / sv.chunk;
    p0 = part + (sv.coff[c] + (p - c * sv.chunk)) * K + d;
    stride = (long long)sv.chunk * K;
    nslots = sv.cn[c];
  }
  const double g = finp_slot_sum(p0, stride, nslots, live);
  if (threadIdx.x < 32 && live) {
    const long long o = perm ? (long long)perm[p] * D + d : q;
    grad[o] = g;
    if (grad2) grad2[o] = g;   // hawkes_grad_at: the caller's array as well (no copy launch)
  }
  __syncthreads();   // finp_slot_sum's shared buffer is reused by the next block
}

template <int D>
__global__ void __launch_bounds__(FINP_THREADS) k_fin2p(const double* __restrict__ part, SlotView sv,
                                                        int N, double* __restrict__ grad,
                                                        const int* __restrict__ perm,
                                                        int* counters, int W,
                                                        double* __restrict__ grad2) {
  pdl_wait();
  // re-arm the pass-2 item counters (as k_fin1p does pass 1's)
  if (counters && blockIdx.x == 0 && threadIdx.x < W) counters[4 * threadIdx.x + 3] = 0;
  fin2p_block<D>(blockIdx.x, part, sv, N, grad, perm, grad2);
}

template <int D>
__global__ void k_rho_to_rec(double* __restrict__ rec, float* __restrict__ rec32,
                             const double* __restrict__ rl, int N) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  // both records: an fp32 context may evaluate with the fp64 kernels (range guard)
  if (rec32) rec32[(long long)i * Layout32<D>::REC + Layout32<D>::RHO] = (float)rl[2 * (long long)i];
  rec[(long long)i * Layout<D>::REC + Layout<D>::RHO] = rl[2 * (long long)i];
}

// Spatial walk order (hawkes_plan.h): the records the pair kernels stream, gathered in walk
// order, rec_p[p] = rec[perm[p]] (x, t; rho' is written by the rate finalize), and each
// 128-event tile's box {lo[D], hi[D], tmin, tmax} for the kernels' culling.  One CTA per tile,
// once per evaluation (the locations move between evaluations).
template <int D>
__global__ void __launch_bounds__(128) k_walk_records(const double* __restrict__ rec,
                                                      const int* __restrict__ perm, int N, int npad,
                                                      double* __restrict__ rec_p,
                                                      double* __restrict__ boxes) {
  using L = Layout<D>;
  const int p = blockIdx.x * 128 + threadIdx.x;
  const bool live = p < N;
  double v[D + 1];
  const int i = perm[min(p, N - 1)];
  HK_CHECK(i >= 0 && i < N);
#pragma unroll
  for (int d = 0; d <= D; ++d) v[d] = rec[(long long)i * L::REC + d];
  if (p < npad) {
#pragma unroll
    for (int d = 0; d <= D; ++d) rec_p[(long long)p * L::REC + d] = v[d];
  }
  __shared__ double lo[4][D + 1], hi[4][D + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int d = 0; d <= D; ++d) {
    double a = live ? v[d] : INFINITY, b = live ? v[d] : -INFINITY;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
      lo[w][d] = a;
      hi[w][d] = b;
    }
  }
  __syncthreads();
  if (threadIdx.x <= D) {
    const int d = threadIdx.x;
    const double a = fmin(fmin(lo[0][d], lo[1][d]), fmin(lo[2][d], lo[3][d]));
    const double b = fmax(fmax(hi[0][d], hi[1][d]), fmax(hi[2][d], hi[3][d]));
    double* o = boxes + (long long)blockIdx.x * (2 * D + 2);
    if (d < D) {
      o[d] = a;
      o[D + d] = b;
    } else {
      o[2 * D] = a;
      o[2 * D + 1] = b;
    }
  }
}

// the fp32 records in walk order (their rho' is written by the rate finalize)
template <int D>
__global__ void __launch_bounds__(128) k_walk_records32(const float* __restrict__ rec32,
                                                        const int* __restrict__ perm, int N, int npad,
                                                        float* __restrict__ rec32_p) {
  using L = Layout32<D>;
  const int p = blockIdx.x * 128 + threadIdx.x;
  if (p >= npad) return;
  const int i = perm[min(p, N - 1)];
  HK_CHECK(i >= 0 && i < N);
#pragma unroll
  for (int q = 0; q < L::RHO; ++q) rec32_p[(long long)p * L::REC + q] = rec32[(long long)i * L::REC + q];
}

// ---- HMC transition (Neal 2011): counter-based random numbers on the device.
// Philox-4x32-10 (Salmon et al. 2011): 10 rounds of the two 32x32->64 multiplies with the
// Weyl key schedule; the counter is (iteration lo, hi, block, lane) and the key the seed, so
// every rank (and every world size) draws the same numbers without any state.
__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

// 53-bit uniform in (0, 1) from two words (high 27 bits of a, high 26 of b)
__device__ __forceinline__ double u53(unsigned a, unsigned b) {
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6) + 0.5) * (1.0 / 9007199254740992.0);
}

// Delta ell of a block move (summation order: hawkes_moves.cuh), one CTA: the
// tree sums part[] of the outside-S terms (written by k_move_delta_rows) in a fixed tree,
// then the k moved events' terms log(lambda_n'/lambda_n) from their combined rows (stored
// in rows_out for the commit) one by one in slot order.  rates[n] = (lambda, mu, xi,
// Lambda); Lambda' = 2^64 lambda is the kernels' scaled unit.  With decide != 0 (MH sweep)
// it also takes the Metropolis decision of block st->mh_cur: log alpha = dell +
// st->mh_hastings, accept iff log u < log alpha (u: Philox block (it, b, MH_ACCEPT_TAG), the
// same stream as hawkes_mh.cuh).
__device__ __forceinline__ double mh_accept_uniform(unsigned klo, unsigned khi, unsigned long long it,
                                                    unsigned b) {
  const uint4 w = philox10(make_uint4((unsigned)it, (unsigned)(it >> 32), b, 0xC0000000u),
                           make_uint2(klo, khi));
  return u53(w.x, w.y);
}

constexpr int MOVE_FINAL_THREADS = 1024;   // 32 warps: one per moved event for k <= 32
__global__ void __launch_bounds__(MOVE_FINAL_THREADS) k_move_terms_final(
    const double* __restrict__ rates, const double* __restrict__ rows_part, int nsplit,
    const int* __restrict__ idx, int k, const double* __restrict__ part, int nb, double tx2,
    double h2, double floor_, double* __restrict__ rows_out, EvalStatus* st, int decide,
    int* __restrict__ acc_out, double* __restrict__ la_out) {
  __shared__ double sh[256];
  __shared__ double sterm[MOVE_MAX];
  const double S = 18446744073709551616.0;   // 2^64
  for (int q = threadIdx.x >> 5; q < k; q += MOVE_FINAL_THREADS / 32) {   // a warp per moved event
    double M, X;
    const double t = move_term_in(rates[4 * (long long)idx[q]] * S, rows_part, q, nsplit, tx2, h2,
                                  floor_, M, X);
    if ((threadIdx.x & 31) == 0) {
      sterm[q] = t;
      rows_out[2 * q] = M;
      rows_out[2 * q + 1] = X;
    }
  }
  // the cooperative sweep's sum (cta_sum256 over its 256-thread CTAs), on threads 0-255
  double v = 0.0;
  if (threadIdx.x < 256)
    for (int i = threadIdx.x; i < nb; i += 256) v += part[i];
  v = cta_sum256(v, sh);
  if (threadIdx.x == 0) {
    double dl = v;
    for (int q = 0; q < k; ++q) dl += sterm[q];
    st->dell = dl;
    if (decide) {
      const int b = st->mh_cur;
      const double la = (dl > -INFINITY) ? dl + st->mh_hastings : -INFINITY;   // NaN -> -inf
      const double u = mh_accept_uniform(st->mh_key_lo, st->mh_key_hi, st->mh_it, (unsigned)b);
      const int acc = log(u) < la ? 1 : 0;
      st->accepted = acc;
      acc_out[b] = acc;
      la_out[b] = la;
      st->mh_block = b + 1;
    }
  }
}

__global__ void k_sum_partials(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// Commit an accepted move: cached rates, ell and the moved events' records.
template <int D>
__global__ void k_move_commit(double* __restrict__ rates, const double* __restrict__ delta,
                              const double* __restrict__ rows, const int* __restrict__ slot_of,
                              const int* __restrict__ idx, const double* __restrict__ new_x, int k,
                              int N, double tx2, double h2, double* __restrict__ rec,
                              float* __restrict__ rec32, double* __restrict__ xcur, EvalStatus* st,
                              int gated) {
  if (gated && !st->accepted) return;   // block MH: the decision is on the device
  const double S1 = 1.0 / 18446744073709551616.0;   // 2^-64
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n == 0) st->ell += st->dell;
  if (n < N) {
    const int q = slot_of[n];
    double mu, xi;
    if (q < 0) {
      mu = __dadd_rn(rates[4 * (long long)n + 1], __dmul_rn(__dmul_rn(delta[2 * (long long)n], tx2), S1));
      xi = __dadd_rn(rates[4 * (long long)n + 2], __dmul_rn(__dmul_rn(delta[2 * (long long)n + 1], h2), S1));
      rates[4 * (long long)n] = __dadd_rn(rates[4 * (long long)n],
          __dmul_rn(fma(delta[2 * (long long)n], tx2, delta[2 * (long long)n + 1] * h2), S1));
    } else {
      mu = __dmul_rn(__dmul_rn(rows[2 * q], tx2), S1);
      xi = __dmul_rn(__dmul_rn(rows[2 * q + 1], h2), S1);
      rates[4 * (long long)n] = __dmul_rn(fma(rows[2 * q], tx2, rows[2 * q + 1] * h2), S1);
    }
    rates[4 * (long long)n + 1] = mu;
    rates[4 * (long long)n + 2] = xi;
  }
  if (n < k) {
    const int m = idx[n];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double v = new_x[n * D + d];
      rec[(long long)m * Layout<D>::REC + d] = v;
      xcur[(long long)m * D + d] = v;
      if (rec32) {
        const float hi = (float)v;
        rec32[(long long)m * Layout32<D>::REC + Layout32<D>::XH + d] = hi;
        rec32[(long long)m * Layout32<D>::REC + Layout32<D>::XL + d] = (float)(v - (double)hi);
      }
    }
  }
}

__global__ void k_scatter_slots(int* __restrict__ slot_of, const int* __restrict__ idx, int k, int set) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < k) slot_of[idx[q]] = set ? q : -1;
}

// sum of ell_n over all rows in a fixed order (one CTA): deterministic for any W (ROWS;
// PAIRS reduces ell in k_fin1p)
__global__ void k_ell_reduce(const double* __restrict__ rl, int N, EvalStatus* st) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < N; i += 1024) s += rl[2 * (long long)i + 1];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    st->ell = sh[0];
    if (!(sh[0] > -INFINITY)) st->undefined = 1;
  }
}

// HAS_G1 (ROWS): g_i = rho'_i G1'_i + sum of the G2' partials; PAIRS: the partials alone
template <int D, bool HAS_G1>
__global__ void k_fin2(const double* __restrict__ part, long long npad, int nchunks,
                       const int* __restrict__ tiles, int N, const double* __restrict__ G1,
                       const double* __restrict__ rl, double* __restrict__ grad) {
  using L = Layout<D>;
  const int i = tiles[blockIdx.x] * RT + threadIdx.x;
  if (i >= N) return;
  double G[D];
#pragma unroll
  for (int d = 0; d < D; ++d) G[d] = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const double* p = part + ((long long)c * npad + i) * L::K2;
#pragma unroll
    for (int d = 0; d < D; ++d) G[d] += p[d];
  }
  if (HAS_G1) {
    const double rho = rl[2 * (long long)i];
#pragma unroll
    for (int d = 0; d < D; ++d) grad[(long long)i * D + d] = fma(rho, G1[(long long)i * D + d], G[d]);
  } else {
#pragma unroll
    for (int d = 0; d < D; ++d) grad[(long long)i * D + d] = G[d];
  }
}

// rows of this rank's tiles -> contiguous send buffer (tile-list order), K values per row
__global__ void k_pack_rows(const double* __restrict__ src, int K, const int* __restrict__ tiles,
                            int ntiles, int N, double* __restrict__ dst) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)ntiles * RT * K;
  if (idx >= total) return;
  const int k = (int)(idx % K);
  const long long r = idx / K;
  const int i = tiles[r / RT] * RT + (int)(r % RT);
  dst[idx] = (i < N) ? src[(long long)i * K + k] : 0.0;
}

// gathered buffers of all ranks -> rows (inverse of k_pack_rows for every rank)
__global__ void k_unpack_rows(const double* __restrict__ src, int K, const int* __restrict__ all_tiles,
                              int max_tiles, int W, int N, double* __restrict__ dst) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per_rank = (long long)max_tiles * RT * K;
  if (idx >= per_rank * W) return;
  const int rank = (int)(idx / per_rank);
  const long long o = idx % per_rank;
  const int k = (int)(o % K);
  const long long r = o / K;
  const int tile = all_tiles[rank * max_tiles + (int)(r / RT)];
  if (tile < 0) return;
  const int i = tile * RT + (int)(r % RT);
  if (i < N) dst[(long long)i * K + k] = src[idx];
}

// leapfrog pieces: every rank holds the full gradient, so every rank updates all
// rows identically (no position exchange needed)
// p += h (g1 + g2): the potential's gradient is the sum of the selected log densities'
__global__ void k_kick(double* __restrict__ p, const double* __restrict__ g1,
                       const double* __restrict__ g2, long long n, double h) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double g = (g1 ? g1[i] : 0.0) + (g2 ? g2[i] : 0.0);
  p[i] = fma(h, g, p[i]);
}

template <int D>
__global__ void k_drift(double* __restrict__ x, double* __restrict__ p,
                        const double* __restrict__ minv, const double* __restrict__ lo,
                        const double* __restrict__ hi, int N, double eps,
                        int* __restrict__ bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const long long k = (long long)i * D + d;
    double pv = p[k];
    double xv = fma(eps * (minv ? minv[k] : 1.0), pv, x[k]);
    if (lo) {
      const double a = lo[k], b = hi[k];
      for (int it = 0; it < 64 && (xv < a || xv > b); ++it) {  // one bounce per round
        xv = (xv < a) ? 2.0 * a - xv : 2.0 * b - xv;
        pv = -pv;
      }
    }
    if (!(fabs(xv) <= 1e100)) atomicOr(bad, 1);
    x[k] = xv;
    p[k] = pv;
  }
}

__global__ void k_kinetic(const double* __restrict__ p, const double* __restrict__ minv, long long n,
                          EvalStatus* st) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += 1024) {
    const double v = p[i];
    s += (minv ? minv[i] : 1.0) * v * v;
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) st->kinetic = 0.5 * sh[0];
}

// standard normals z[2q], z[2q+1] from block (it, q): Box-Muller of (u1, u2)
__device__ __forceinline__ double2 hmc_normal_pair(uint2 key, unsigned long long it, unsigned q) {
  const uint4 w = philox10(make_uint4((unsigned)it, (unsigned)(it >> 32), q, 0u), key);
  const double u1 = u53(w.x, w.y), u2 = u53(w.z, w.w);
  const double rad = sqrt(-2.0 * log(u1));
  double s, c;
  sincospi(2.0 * u2, &s, &c);
  return make_double2(rad * c, rad * s);
}

// p = Minv^{-1/2} z (Minv = nullptr: identity), or z itself into p when raw != 0
__global__ void k_hmc_momenta(double* __restrict__ p, const double* __restrict__ minv, long long n,
                              uint2 key, unsigned long long it, int raw) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * q >= n) return;
  const double2 z = hmc_normal_pair(key, it, (unsigned)q);
  const long long e = 2 * q;
  p[e] = (minv && !raw) ? z.x * rsqrt(minv[e]) : z.x;
  if (e + 1 < n) p[e + 1] = (minv && !raw) ? z.y * rsqrt(minv[e + 1]) : z.y;
}

// after the first potential evaluation at x0 and k_kinetic(p0)
__global__ void k_hmc_begin(EvalStatus* st, int use_h, int use_b) {
  st->lp0 = (use_h ? st->ell : 0.0) + (use_b ? st->bmds : 0.0);
  st->kin0 = st->kinetic;
  // ell(x0) itself, not the undefined flag: a cached evaluation of x0 (rates reused from an
  // earlier call) does not run k_ell_reduce again, so the flag would stay clear
  st->undef0 = (use_h && !(st->ell > -INFINITY)) ? 1 : 0;
}

// after the trajectory and k_kinetic(p1): Metropolis accept iff log u < H0 - H1.  A
// trajectory that left the support (ell = -inf) or diverged (|x| > 1e100, flagged by
// k_drift / k_pack_x in bit 0 of *bad) has H1 = +inf and is rejected; its flag is cleared.
__global__ void k_hmc_decide(EvalStatus* st, int* bad, int use_h, int use_b, uint2 key,
                             unsigned long long it) {
  const double lp1 = (use_h ? st->ell : 0.0) + (use_b ? st->bmds : 0.0);
  const bool diverged = (use_h && st->undefined) || (*bad & 1) || !(lp1 > -INFINITY) ||
                        !(st->kinetic < INFINITY);
  const double la = diverged ? -INFINITY : (lp1 - st->kinetic) - (st->lp0 - st->kin0);
  const uint4 w = philox10(make_uint4((unsigned)it, (unsigned)(it >> 32), 0xffffffffu, 1u), key);
  const double u = u53(w.x, w.y);
  st->log_alpha = la;
  st->accepted = (!st->undef0 && log(u) < la) ? 1 : 0;
  if (*bad & 1) atomicAnd(bad, ~1);
  if (use_h) st->undefined = 0;
}

// the chain's new state: x' when accepted, else x0 (xstage holds x0 throughout)
__global__ void k_hmc_select(double* __restrict__ xstage, const double* __restrict__ x1, long long n,
                             const EvalStatus* st) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && st->accepted) xstage[i] = x1[i];
}

// diagnostics: the fast exp on an array (tests pin its accuracy)
__global__ void k_diag_exp(const double* __restrict__ a, double* __restrict__ out, long long n,
                           const int2* __restrict__ gtab) {
  __shared__ int2 tab[EXP_TABLE];
  for (int q = threadIdx.x; q < EXP_TABLE; q += blockDim.x) tab[q] = gtab[q];
  __syncthreads();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fexp(a[i], tab);
}

// diagnostics: dependent-DFMA throughput probe (FP64 pipe peak)
__global__ void k_diag_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
         a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int k = 0; k < iters; ++k) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  const double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}

// diagnostics: FP64-pipe throughput for several operand patterns (ops per thread per iter = 8)
__global__ void k_diag_mode(double* out, int iters, int mode, const int2* __restrict__ gtab) {
  __shared__ int2 tab[EXP_TABLE];
  for (int q = threadIdx.x; q < EXP_TABLE; q += blockDim.x) tab[q] = gtab[q];
  __syncthreads();
  double a[8], b[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    a[q] = 1e-3 * (threadIdx.x + q);
    b[q] = 0.5 + 1e-4 * q;
  }
  const double m = 0.999999, c = 1e-7;
  if (mode == 0) {
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = fma(a[q], m, c);
  } else if (mode == 1) {      // three distinct register operands
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = fma(a[q], b[q], b[(q + 1) & 7]);
  } else if (mode == 2) {      // DADD of two registers
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = a[q] + b[q];
  } else if (mode == 3) {      // DMUL of two registers
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = a[q] * b[q];
  } else if (mode == 4) {      // fast exp, 8 independent chains (9 FP64 ops each)
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = -fexp(-a[q] * 1e-3, tab);
  } else if (mode == 5) {      // two-register DFMA with one constant
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = fma(a[q], b[q], c);
  } else if (mode == 6) {      // alternating DFMA / DADD
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = (q & 1) ? a[q] + b[q] : fma(a[q], b[q], c);
  } else if (mode == 10) {     // alternating DFMA / DMUL
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = (q & 1) ? a[q] * b[q] : fma(a[q], b[q], c);
  } else if (mode == 11) {     // alternating DFMA / (DADD written as DFMA with a runtime 1.0)
    const double one = gtab ? 1.0 + 0.0 * (double)iters : 1.0;
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = (q & 1) ? fma(a[q], one, b[q]) : fma(a[q], b[q], c);
  } else if (mode == 13) {     // DFMA stream + an independent I2F.F64 per DFMA (pipe sharing)
    int acc = threadIdx.x;
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        a[q] = fma(a[q], m, c);
        acc ^= __double2loint(__int2double_rn(acc + q));
      }
    a[0] += acc;
  } else if (mode == 14) {     // I2F.F64 stream alone
    int acc = threadIdx.x;
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc ^= __double2loint(__int2double_rn(acc + q));
    a[0] += acc;
  } else if (mode == 15) {     // fast exp with kf = I2F(k) in place of y - shift
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double x = -a[q] * 1e-3;
        const unsigned ahi = min((unsigned)__double2hiint(x), EXP_AMIN_HI);
        const double ac = __hiloint2double((int)ahi, __double2loint(x));
        const double y = fma(ac, EXP_K, EXP_SHIFT);
        const int kk = __double2loint(y);
        const double r = fma(__int2double_rn(kk), -EXP_C, ac);
        const int2 T = tab[kk & (EXP_TABLE - 1)];
        const double p = fma(EXP_C2, r, 1.0) * r;
        const double Tm = __hiloint2double(T.y + kk * (1 << EXP_BIAS_SHIFT), T.x);
        a[q] = -fma(Tm, p, Tm);
      }
  } else if (mode == 9) {      // one dependent DFMA chain per thread (latency probe)
    for (int k = 0; k < iters; ++k)
#pragma unroll
      for (int q = 0; q < 8; ++q) a[0] = fma(a[0], m, c);
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += a[q];
  if (s == 12345.678) out[0] = s;
}


}  // namespace hk
