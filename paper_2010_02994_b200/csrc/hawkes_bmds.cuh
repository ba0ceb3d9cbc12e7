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

// ---- unordered-pair BMDS (each pair {n, m} evaluated once) ----------------------------
// Tasks are pairs (a <= b) of 32-event blocks, dealt statically to warps.  Lane l owns row
// i = 32a + l; in step s = 0..31 it pairs with column j = 32b + (l + s) mod 32 (diagonal
// tasks: only j > i), whose x comes from a warp-private shared copy and whose gradient sums
// rotate one lane per step through warp shuffles (as in the Hawkes sym kernel).  The task's
// 32 x 32 block of Y is staged in warp-private shared memory with coalesced loads; step s
// reads Y[l][(l + s) mod 32], two wavefronts (the ideal for 8-byte loads).  The pair's value
// goes to the row, +s u to the row's gradient and -s u to the column's.  Row partials go to
// slot b, column partials to slot a (slot NB for diagonal tasks), so every (slot, event) is
// written exactly once and k_bmds_sym_fin sums the NB + 1 slots in order.  Each lane
// takes two pairs per step (columns (l + s) and (l + s + 16) mod 32, 16 steps), their main
// chains branch-free so they interleave (128 registers, 16 warps/SM): 5 % over one pair
// per step.  Half the pair work of k_bmds: 2.3 vs 3.79 ms at N = 20k; 0.19 vs 0.28 ms at
// the flu size (N = 4733), where ~5 tasks per warp and their staging latency limit it.
constexpr int BSYM_WARPS = 4;

template <int D>
__host__ __device__ constexpr size_t bmds_sym_smem() {
  return (size_t)EXP_TABLE * sizeof(int2) + (size_t)BSYM_WARPS * (32 * 32 + 32 * D) * sizeof(double);
}

template <int D>
__global__ void __launch_bounds__(32 * BSYM_WARPS) k_bmds_sym(const double* __restrict__ x,
                                                              const double* __restrict__ Y, int N,
                                                              BmdsConst c, const int2* __restrict__ gtab,
                                                              double* __restrict__ part, long long ntasks) {
  constexpr int K = D + 1;
  extern __shared__ __align__(16) unsigned char bs_smem[];
  int2* tab = reinterpret_cast<int2*>(bs_smem);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* Ys = reinterpret_cast<double*>(tab + EXP_TABLE) + warp * (32 * 32 + 32 * D);   // [32][32]
  double* xs = Ys + 32 * 32;                                                               // [32][D]
  for (int t = threadIdx.x; t < EXP_TABLE; t += blockDim.x) tab[t] = gtab[t];
  __syncthreads();
  const int NB = (N + 31) / 32;
  const long long gw = (long long)blockIdx.x * BSYM_WARPS + warp, W = (long long)gridDim.x * BSYM_WARPS;
  for (long long t = gw; t < ntasks; t += W) {
    // t = b (b + 1) / 2 + a, 0 <= a <= b
    int b = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
    while ((long long)b * (b + 1) / 2 > t) --b;
    while ((long long)(b + 1) * (b + 2) / 2 <= t) ++b;
    const int a = (int)(t - (long long)b * (b + 1) / 2);
    const bool diag = a == b;
    const int i = 32 * a + lane;
    const bool irow = i < N;
    double xi[D];
#pragma unroll
    for (int d = 0; d < D; ++d) xi[d] = x[(long long)min(i, N - 1) * D + d];
    const int j0 = 32 * b;
    {
      const int jl = j0 + lane;
#pragma unroll
      for (int d = 0; d < D; ++d) xs[lane * D + d] = x[(long long)min(jl, N - 1) * D + d];
      for (int r = 0; r < 32; ++r) {
        const int ir = 32 * a + r;
        Ys[r * 32 + lane] = (ir < N && jl < N) ? Y[(long long)ir * N + jl] : 1.0;
      }
    }
    __syncwarp();
    // two pairs per lane and step (columns (l + s) and (l + s + 16) mod 32, s = 0..15): two
    // independent dependency chains per lane, whose column sums rotate together
    double gr[D], gc[2][D], v = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) gr[d] = gc[0][d] = gc[1][d] = 0.0;
#pragma unroll 1
    for (int s = 0; s < 16; ++s) {
      // both pairs' main chains branch-free (a dead pair -- padding, or j <= i on a diagonal
      // task -- computes on a clamped column and is selected to 0), so the compiler can
      // interleave them; the erfc / log1p tail (z < 9) stays a branch, rarely taken
      double u[2][D], r2[2], inv_d[2], z[2], e[2], phis[2];
      bool live[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cidx = (lane + s + 16 * h) & 31;
        const int j = j0 + cidx;
        live[h] = irow && j < N && (!diag || j > i);
        r2[h] = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          u[h][d] = xi[d] - xs[cidx * D + d];
          r2[h] = fma(u[h][d], u[h][d], r2[h]);
        }
        const double y = Ys[lane * 32 + cidx];
        const bool apart = r2[h] > 0.0;
        inv_d[h] = apart ? rsqrt(r2[h]) : 0.0;
        const double delta = r2[h] * inv_d[h];
        z[h] = delta * c.inv_s;
        e[h] = y - delta;
        phis[h] = apart ? fexp(fma(r2[h], c.mhalf_inv_s2, c.lphi_c), tab) : 0.0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double lphi = 0.0;
        if (z[h] < 9.0) {
          const double q = 0.5 * erfc(z[h] * 0.70710678118654752440);
          lphi = log1p(-q);
          phis[h] = phis[h] / (1.0 - q);
        }
        const double sw = live[h] ? (e[h] * c.inv_s2 - phis[h]) * inv_d[h] : 0.0;
        if (live[h]) v -= c.half_log + 0.5 * e[h] * e[h] * c.inv_s2 + lphi;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          gr[d] = fma(sw, u[h][d], gr[d]);
          gc[h][d] = fma(-sw, u[h][d], gc[h][d]);
        }
      }
      // rotate both column sums one lane down: lane l then holds columns (l + s + 1) and
      // (l + s + 17) mod 32
      const int nxt = (lane + 1) & 31;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        gc[0][d] = __shfl_sync(0xffffffffu, gc[0][d], nxt);
        gc[1][d] = __shfl_sync(0xffffffffu, gc[1][d], nxt);
      }
    }
    __syncwarp();
    // lane l now holds, for column (l + 16) mod 32, the sums over rows l' = l + 16 + t (mod 32,
    // t < 16: its gc[0] half) and, for column l, those over rows l - 16 - t (gc[1]): the
    // column's total is its gc[1] plus the gc[0] of lane (l + 16) mod 32
    if (irow) {
      double* o = part + ((long long)b * N + i) * K;
#pragma unroll
      for (int d = 0; d < D; ++d) o[d] = gr[d];
      o[D] = v;
    }
    const int jl = j0 + lane;
#pragma unroll
    for (int d = 0; d < D; ++d) gc[1][d] += __shfl_sync(0xffffffffu, gc[0][d], (lane + 16) & 31);
    if (jl < N) {
      double* o = part + ((long long)(diag ? NB : a) * N + jl) * K;
#pragma unroll
      for (int d = 0; d < D; ++d) o[d] = gc[1][d];
      o[D] = 0.0;
    }
  }
}

// every event's NB + 1 slots in index order (slots a < block(n) hold column roles, slots
// b >= block(n) row roles, slot NB the diagonal task's column role).  One thread per
// (event, component): consecutive threads read consecutive doubles of a slot (coalesced), and
// each sum runs over the slots in the same order as one thread per event did (bitwise the
// same result); at the flu size that is 33k independent sums instead of 4733 (ncu: the
// per-event form took 88 us, long-scoreboard bound, next to the pair kernel's 154 us)
template <int D>
__global__ void k_bmds_sym_fin(const double* __restrict__ part, int N, double* __restrict__ grad,
                               double* __restrict__ row_value) {
  constexpr int K = D + 1;
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)N * K) return;
  const int n = (int)(q / K), k = (int)(q % K);
  const int NB = (N + 31) / 32;
  const long long stride = (long long)N * K;
  const double* p = part + q;
  double acc = 0.0;
#pragma unroll 8
  for (int sl = 0; sl <= NB; ++sl) acc += __ldg(p + sl * stride);
  if (k < D)
    grad[(long long)n * D + k] = acc;
  else
    row_value[n] = acc;
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
