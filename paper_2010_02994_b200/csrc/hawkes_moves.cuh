// hawkes_moves.cuh -- block Metropolis-Hastings over locations: Delta ell for moving k events.
//
// The paper's DC and Alaska samplers update locations with "a Metropolis-Hastings kernel
// with block-wise updates over sets of individual location variables".  Moving
// the events S to new positions leaves every Lambda_n unchanged (P:L92-93 has no x) and
// changes lambda_n only through the pairs that touch S:
//   n not in S:  lambda_n' = lambda_n + sum_{m in S} [lambda_nm(x_m') - lambda_nm(x_m)]
//   n in S:      lambda_n' = sum_j lambda_nj(X')            (full row, O(N))
//   Delta ell = sum_n log(lambda_n' / lambda_n)              (Eq. 1)
// so a proposal costs O(k N) instead of the O(N^2) of a fresh evaluation.  Pair terms use
// the same scaled-domain exps as the pass kernels (alpha mu 2^64, beta xi 2^64).
// Summation order of Delta ell (shared by the launch path and the cooperative sweep, which
// tests compare bitwise): the terms of the events outside S in fixed 256-event trees (the
// moved events contribute 0 there), the tree sums over the 256-event blocks in a fixed
// tree, then the k moved events' terms added one by one in slot order.  The events outside
// S get their terms in the same pass that computes their rate changes.
#pragma once
#include "hawkes_kernels.cuh"

namespace hk {

constexpr int MOVE_MAX = 256;   // events per proposal (one shared-memory batch)

template <int D>
struct MoveArgs {
  const double* rec;       // event records (x, t, ...)
  const int* gid;
  const int* slot_of;      // N: index into the proposal, or -1
  const int* idx;          // k moved events
  const double* new_x;     // k x D proposed locations
  int k, N;
  PassConst c;
  const int2* tab;
  const double* rates;     // N x 4 (lambda, mu, xi, Lambda) at the current state
  double tx2, h2, floor_;  // Lambda' = M' tau_x^2 + X' h^2; at or below floor_: lambda = 0
  double* part;            // ceil(N/256): tree sums of the outside-S terms
};

// Delta-ell term of an event outside S from its rate changes (scaled units, L0 = Lambda')
__device__ __forceinline__ double move_term_out(double L0, double dM, double dX, double tx2, double h2,
                                                double floor_) {
  const double d = fma(dM, tx2, dX * h2);
  return (d == 0.0) ? 0.0 : ((L0 + d > floor_) ? log1p(d / L0) : -INFINITY);
}

// term of a moved event from its full row at X', by one warp: lane l sums the split ranges
// l, l + 32, ... in order, a shuffle-down tree combines the lanes (a fixed order); M', X'
// and the term are valid in lane 0.  (One thread walking the up to 64 ranges put a chain of
// dependent L2 loads on the MH sweep's critical path.)
__device__ __forceinline__ double move_term_in(double L0, const double* __restrict__ rows_part, int q,
                                               int nsplit, double tx2, double h2, double floor_,
                                               double& M, double& X) {
  const int lane = threadIdx.x & 31;
  M = 0.0;
  X = 0.0;
  for (int s = lane; s < nsplit; s += 32) {
    M += __ldcg(rows_part + 2 * ((long long)q * nsplit + s));
    X += __ldcg(rows_part + 2 * ((long long)q * nsplit + s) + 1);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    M += __shfl_down_sync(0xffffffffu, M, o);
    X += __shfl_down_sync(0xffffffffu, X, o);
  }
  const double L1 = fma(M, tx2, X * h2);
  return ((L1 > floor_) ? log(L1) : -INFINITY) - log(L0);
}

// fixed-order sum over the first 256 threads of a CTA (every thread calls it; red: 16
// doubles of shared memory): a shuffle-down tree in each of warps 0-7, then warp 0 combines
// the 8 warp sums the same way.  The result is valid in thread 0; one barrier instead of the
// eight of a shared-memory tree (the MH sweep's block step is a chain of such sums).  The
// two-value form sums (a, b) pairs in the same order.
__device__ __forceinline__ void cta_sum256x2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  if (lane == 0 && warp < 8) {
    red[warp] = a;
    red[8 + warp] = b;
  }
  __syncthreads();
  if (warp == 0) {
    a = lane < 8 ? red[lane] : 0.0;
    b = lane < 8 ? red[8 + lane] : 0.0;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b += __shfl_down_sync(0xffffffffu, b, o);
    }
  }
}
__device__ __forceinline__ double cta_sum256(double v, double* red) {
  double z = 0.0;
  cta_sum256x2(v, z, red);
  return v;
}

// pair term parts (scaled) for event n at xn against event m at xm, times/ties from records
template <int D>
__device__ __forceinline__ void move_pair(const double* xn, double tn, int gn, const double* xm,
                                          double tm, int gm, const PassConst& c,
                                          const int2* __restrict__ tab, double& eb, double& es) {
  double r2 = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double dx = xm[d] - xn[d];
    r2 = fma(dx, dx, r2);
  }
  const double dt = tn - tm;
  eb = gm == gn ? 0.0 : fexp(fma(c.kx, r2, fma(c.kt * dt, dt, c.lnc_b)), tab);
  es = gm < gn ? fexp(fma(c.ks, r2, fma(-c.omega, dt, c.lnc_s)), tab) : 0.0;
}

// rows not in S: (delta M', delta X') from the k moved events and their Delta-ell terms,
// tree-summed over the CTA's 256 events into part[blk] (CTA blk of the delta role)
template <int D>
__device__ __forceinline__ void move_delta_body(const MoveArgs<D>& a, const int2* __restrict__ tab,
                                                double* __restrict__ dout, int blk, double* dyn) {
  using L = Layout<D>;
  double* red = dyn;                          // [256]
  double* sx_old = dyn + 256;                 // [k][D]
  double* sx_new = sx_old + a.k * D;          // [k][D]
  double* st = sx_new + a.k * D;              // [k]
  int* sg = reinterpret_cast<int*>(st + a.k); // [k]
  for (int q = threadIdx.x; q < a.k; q += blockDim.x) {
    const int m = a.idx[q];
    const double* rm = a.rec + (long long)m * L::REC;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      sx_old[q * D + d] = rm[d];
      sx_new[q * D + d] = a.new_x[q * D + d];
    }
    st[q] = rm[D];
    sg[q] = a.gid[m];
  }
  __syncthreads();
  const int n = blk * blockDim.x + threadIdx.x;
  double term = 0.0;
  if (n < a.N) {
    double dM = 0.0, dX = 0.0;
    if (a.slot_of[n] < 0) {
      const double* rn = a.rec + (long long)n * L::REC;
      double xn[D];
#pragma unroll
      for (int d = 0; d < D; ++d) xn[d] = rn[d];
      const double tn = rn[D];
      const int gn = a.gid[n];
      for (int q = 0; q < a.k; ++q) {
        double eb0, es0, eb1, es1;
        move_pair<D>(xn, tn, gn, sx_old + q * D, st[q], sg[q], a.c, tab, eb0, es0);
        move_pair<D>(xn, tn, gn, sx_new + q * D, st[q], sg[q], a.c, tab, eb1, es1);
        dM += eb1 - eb0;
        dX += es1 - es0;
      }
      term = move_term_out(a.rates[4 * (long long)n] * 18446744073709551616.0, dM, dX, a.tx2,
                           a.h2, a.floor_);
    }
    dout[2 * (long long)n] = dM;
    dout[2 * (long long)n + 1] = dX;
  }
  const double tsum = cta_sum256(term, red);
  if (threadIdx.x == 0) a.part[blk] = tsum;
}

// rows in S: full (M', X') at the proposed configuration.  Block (q, s) sums the j range
// [s*len, (s+1)*len), len = move_split_len(N), for moved event q (strided per thread, fixed tree);
// k_move_rows_combine adds the split partials in order.
// j-range length: 256 events per CTA for small N (latency), at most MOVE_NSPLIT ranges for
// large N (the in-order combine of k_move_terms_final stays short)
constexpr int MOVE_NSPLIT = 64;
__host__ __device__ inline int move_split_len(int N) {
  const int per = (N + MOVE_NSPLIT - 1) / MOVE_NSPLIT;
  return per <= 256 ? 256 : ((per + 255) / 256) * 256;
}

template <int D>
__device__ __forceinline__ void move_rows_body(const MoveArgs<D>& a, const int2* __restrict__ tab,
                                               double* __restrict__ rows_part, int q, int split,
                                               int nsplit, double* dyn) {
  using L = Layout<D>;
  double* red = dyn;   // 16 doubles (cta_sum256x2)
  const int n = a.idx[q];
  double xn[D];
#pragma unroll
  for (int d = 0; d < D; ++d) xn[d] = a.new_x[q * D + d];
  const double tn = a.rec[(long long)n * L::REC + D];
  const int gn = a.gid[n];
  const int len = move_split_len(a.N);
  const int j0 = split * len, j1 = min(a.N, j0 + len);
  double M = 0.0, X = 0.0;
  for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
    const double* rj = a.rec + (long long)j * L::REC;
    const int sj = a.slot_of[j];
    const double* xj = sj >= 0 ? a.new_x + sj * D : rj;
    double eb, es;
    move_pair<D>(xn, tn, gn, xj, rj[D], a.gid[j], a.c, tab, eb, es);
    M += eb;
    X += es;
  }
  cta_sum256x2(M, X, red);
  if (threadIdx.x == 0) {
    const long long o = 2 * ((long long)q * nsplit + split);
    rows_part[o] = M;
    rows_part[o + 1] = X;
  }
}

// One launch, two CTA roles: CTAs [0, nb_delta) update the rows outside S
// (move_delta_body), the k * nsplit others sum the moved events' full rows at X' over
// move_split_len(N)-event j ranges (move_rows_body).  Dynamic shared memory: the exp table,
// then the k moved events (delta role) or the reduction buffers (rows role).
template <int D>
__host__ __device__ constexpr size_t move_smem_bytes(int k) {
  return (size_t)EXP_TABLE * sizeof(int2) +
         ((size_t)(256 + k * (2 * D + 1)) * sizeof(double) + (size_t)k * sizeof(int) > 512 * sizeof(double)
              ? (size_t)(256 + k * (2 * D + 1)) * sizeof(double) + (size_t)k * sizeof(int)
              : 512 * sizeof(double));
}

template <int D>
__global__ void __launch_bounds__(256) k_move_delta_rows(MoveArgs<D> a, const int2* __restrict__ gtab,
                                                         double* __restrict__ dout,
                                                         double* __restrict__ rows_part, int nb_delta,
                                                         int nsplit) {
  extern __shared__ __align__(16) unsigned char mv_smem[];
  int2* tab = reinterpret_cast<int2*>(mv_smem);
  double* dyn = reinterpret_cast<double*>(tab + EXP_TABLE);
  for (int t = threadIdx.x; t < EXP_TABLE; t += blockDim.x) tab[t] = gtab[t];
  __syncthreads();
  if ((int)blockIdx.x < nb_delta) {
    move_delta_body<D>(a, tab, dout, blockIdx.x, dyn);
  } else {
    const int u = blockIdx.x - nb_delta;
    move_rows_body<D>(a, tab, rows_part, u / nsplit, u % nsplit, nsplit, dyn);
  }
}

}  // namespace hk
