// hawkes_bmds.cuh -- Bayesian MDS log density and location gradient (sm_100a, fp64).
//
// The flu application models observed dissimilarities y_{nn'} ~ N(delta_{nn'}, sigma^2)
// truncated to y > 0, delta_{nn'} = |x_n - x_n'|, so (Eq. bmdsLikelihood,
// P:L176-180, with the normal constant kept)
//   log p(Y | X) = sum_{n > n'} -1/2 log(2 pi sigma^2) - (y - delta)^2 / (2 sigma^2)
//                              - log Phi(delta / sigma)
//   d log p / d x_n = - sum_{n' != n} r'(delta) (x_n - x_n') / delta,
//   r'(delta) = -(y - delta)/sigma^2 + phi(delta/sigma) / (sigma Phi(delta/sigma)).
// HMC over X needs this gradient next to the Hawkes one.  One 128-thread CTA per
// event n: threads stride over n' (row n of Y is contiguous, so the loads coalesce), the D
// gradient components and the value (pairs n' < n only, so each pair counts once) are
// reduced over the CTA in a fixed tree.  Per pair: one rsqrt and one table exp (plus an erfc
// and a log1p for the few pairs with delta < 9 sigma); the per-pair chain is long and
// dependent, so the kernel needs many warps.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "hawkes_kernels.cuh"

namespace hk {

struct BmdsConst {
  double inv_s;        // 1/sigma
  double inv_s2;       // 1/sigma^2
  double half_log;     // 1/2 log(2 pi sigma^2)
  double mhalf_inv_s2; // -1/(2 sigma^2)
  double lphi_c;       // log(1/(sigma sqrt(2 pi))): phi(z)/sigma = e^(r2 mhalf_inv_s2 + lphi_c)
};

constexpr int BMDS_THREADS = 128;

// Per ordered pair: 1/delta = rsqrt(r2) gives delta = r2/delta and replaces the division in
// the gradient weight; phi(z)/sigma = e^(-r2/(2 sigma^2)) / (sigma sqrt(2 pi)) comes straight
// from r2 through the kernels' table exp (constant folded into the exponent); beyond
// z = 9 the tail 1 - Phi(z) is below 1.2e-19, so 1/Phi(z) is 1 in double and log Phi(z)
// adds under 1.2e-19 per pair -- the erfc, log1p and the division by Phi are skipped
// there (most pairs of a spread-out configuration; whole warps skip the branch).
// The kernel is latency-bound (ncu at the flu shape: FP64 pipe 42 %, 28 warps/SM, DRAM only
// Y once).  Tried and slower: 4 events per CTA sharing each x_n' load (1.7x: the larger
// register tile cut the warps in flight); unroll 1 or 4 instead of 2 (+14 %); forcing 10-12
// CTAs/SM with launch bounds (spills, +8-53 %) -- shared memory (exp table 16 KB + the
// reduction) allows 9 CTAs anyway.
template <int D>
__global__ void __launch_bounds__(BMDS_THREADS) k_bmds(const double* __restrict__ x,
                                                       const double* __restrict__ Y, int N,
                                                       BmdsConst c, const int2* __restrict__ gtab,
                                                       double* __restrict__ grad,
                                                       double* __restrict__ row_value) {
  __shared__ int2 tab[EXP_TABLE];
  __shared__ double red[BMDS_THREADS][D + 1];
  const int n = blockIdx.x;
  const int tid = threadIdx.x;
  for (int t = tid; t < EXP_TABLE; t += BMDS_THREADS) tab[t] = gtab[t];
  double xn[D];
#pragma unroll
  for (int d = 0; d < D; ++d) xn[d] = x[(long long)n * D + d];
  const double* yrow = Y + (long long)n * N;
  double g[D], v = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) g[d] = 0.0;
  __syncthreads();
#pragma unroll 2
  for (int m = tid; m < N; m += BMDS_THREADS) {
    if (m == n) continue;
    double u[D], r2 = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      u[d] = xn[d] - x[(long long)m * D + d];
      r2 = fma(u[d], u[d], r2);
    }
    // hawkes_set_bmds mirrored the lower triangle (Eq. bmdsLikelihood's n > n') into the
    // upper one, so row n holds y_{nn'} for every n' and the loads coalesce
    const double y = yrow[m];
    const bool apart = r2 > 0.0;
    const double inv_d = apart ? rsqrt(r2) : 0.0;
    const double delta = r2 * inv_d;
    const double z = delta * c.inv_s;
    double q = 0.0, lphi = 0.0;
    if (z < 9.0) {
      q = 0.5 * erfc(z * 0.70710678118654752440);   // 1 - Phi(z), z >= 0
      lphi = log1p(-q);
    }
    const double e = y - delta;
    if (m < n) v -= c.half_log + 0.5 * e * e * c.inv_s2 + lphi;
    if (apart) {
      double phis = fexp(fma(r2, c.mhalf_inv_s2, c.lphi_c), tab);   // phi(z) / sigma
      if (z < 9.0) phis = phis / (1.0 - q);
      const double s = (e * c.inv_s2 - phis) * inv_d;                // -r'(delta) / delta
#pragma unroll
      for (int d = 0; d < D; ++d) g[d] = fma(s, u[d], g[d]);
    }
  }
  // fixed-order tree over the CTA
#pragma unroll
  for (int d = 0; d < D; ++d) red[tid][d] = g[d];
  red[tid][D] = v;
  __syncthreads();
  for (int w = BMDS_THREADS / 2; w > 0; w >>= 1) {
    if (tid < w) {
#pragma unroll
      for (int d = 0; d <= D; ++d) red[tid][d] += red[tid + w][d];
    }
    __syncthreads();
  }
  if (tid == 0) {
#pragma unroll
    for (int d = 0; d < D; ++d) grad[(long long)n * D + d] = red[0][d];
    row_value[n] = red[0][D];
  }
}

// mirror the lower triangle into the upper one (device copy of Y), flag bad entries
__global__ void k_bmds_mirror(double* __restrict__ Y, int N, int* __restrict__ bad) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)N * N) return;
  const int n = (int)(idx / N), m = (int)(idx % N);
  if (n > m) {
    const double y = Y[idx];
    if (!(y > 0.0) || !(y <= 1e100)) atomicOr(bad, 2);
    Y[(long long)m * N + n] = y;
  }
}

}  // namespace hk
