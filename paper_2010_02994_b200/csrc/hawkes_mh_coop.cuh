// hawkes_mh_coop.cuh -- the block Metropolis-Hastings sweep as ONE persistent
// cooperative kernel.
//
// The launch-based sweep (hawkes_mh.cuh + hawkes_moves.cuh, replayed as a CUDA graph) pays
// four dependent kernel launches per block; at the paper's catalog sizes (N = 2925 / 3982)
// the pair work of a block is ~1 us and the launches dominate.  Here one grid of
// co-resident CTAs (cudaLaunchCooperativeKernel) walks all blocks with two grid-wide
// barriers per block:
//   A  every CTA draws the block's k proposals itself (same Philox stream, same values),
//      keeps them in shared memory and stamps the events' slots as (block << 8) | slot in a
//      global map -- identical concurrent writes, and no clearing between blocks, so no
//      barrier is needed before phase B
//   B  rows outside S (the k moved events' pair changes, their Delta-ell terms and the
//      terms' 256-event tree sums) and the moved rows at X', grid-stride over the same work
//      units as k_move_delta_rows                                          | grid.sync
//   D  every CTA forms the moved events' terms, sums everything in the same fixed order,
//      takes the Metropolis decision (identical everywhere), and commits its share of the
//      rates / records                                                     | grid.sync
// (A third barrier, for the per-event terms as a phase of their own, cost 2.5-3 us per block.)
// Arithmetic and reduction orders are those of the launch-based path (hawkes_moves.cuh;
// tests check the two agree bitwise).
#pragma once
#include <cooperative_groups.h>

#include "hawkes_mh.cuh"

namespace hk {

template <int D>
struct MhCoopArgs {
  double* rec;             // Npad x REC records (x rewritten on commit)
  float* rec32;            // fp32 records or nullptr
  const int* gid;
  const int* blocks;       // n_blocks x k event indices
  int n_blocks, k, N, nsplit;
  const double* centre;    // N x D region centres
  const double* size;      // N region sizes
  int kind;
  double* xcur;            // N x D current locations
  double* rates;           // N x 4 (lambda, mu, xi, Lambda)
  double* delta;           // Npad x 2
  double* rows_part;       // k x nsplit x 2
  double* part;            // ceil(N/256) term sums
  int* stamp;              // N: (block << 8) | slot of the events moved so far, -1 initially
  const int2* gtab;
  PassConst c;
  double tx2, h2, floor_;
  EvalStatus* st;
  int* acc_out;
  double* la_out;
};

// slot of event n in block b: every CTA stamps the block's events with (b << 8) | slot in
// phase A (identical values, so the concurrent writes agree); the map is cleared to -1 at
// the start of each sweep, so a stamp of another block can never read as a member
struct StampSlots {
  const int* stamp;
  int b;
  __device__ __forceinline__ int operator()(int n) const {
    const int v = stamp[n];
    return (v >> 8) == b ? (v & 255) : -1;
  }
};

template <int D>
__host__ __device__ constexpr size_t mh_coop_smem(int k) {
  return (size_t)EXP_TABLE * sizeof(int2) + (size_t)k * (2 * D + 1) * sizeof(double) +
         512 * sizeof(double) + (size_t)4 * k * sizeof(double) + (size_t)2 * k * sizeof(int);
}

template <int D>
__global__ void __launch_bounds__(256) k_mh_sweep_coop(MhCoopArgs<D> a) {
  namespace cg = cooperative_groups;
  using L = Layout<D>;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char sm[];
  int2* tab = reinterpret_cast<int2*>(sm);
  const int k = a.k, N = a.N, nb = (N + 255) / 256, nsplit = a.nsplit;
  double* sx_old = reinterpret_cast<double*>(tab + EXP_TABLE);   // [k][D]
  double* sx_new = sx_old + k * D;                               // [k][D]
  double* stt = sx_new + k * D;                                  // [k] times
  double* red = stt + k;                                         // [512] reductions
  double* srow = red + 512;                                      // [k][2] moved rows (M', X')
  double* sterm = srow + 2 * k;                                  // [k] moved events' terms
  double* sL0 = sterm + k;                                       // [k] their Lambda' before
  int* sraw = reinterpret_cast<int*>(sL0 + k);                   // [k] event of slot q
  int* sg = sraw + k;                                            // [k] tie group of slot q
  __shared__ int s_acc;
  __shared__ double s_hast;
  const int tid = threadIdx.x;
  for (int t = tid; t < EXP_TABLE; t += blockDim.x) tab[t] = a.gtab[t];
  const uint2 key = make_uint2(a.st->mh_key_lo, a.st->mh_key_hi);
  const unsigned long long it = a.st->mh_it;
  const double scale = a.st->mh_scale;
  const double S = 18446744073709551616.0, S1 = 1.0 / S;   // 2^64, 2^-64
  const int len = move_split_len(N);

  for (int b = 0; b < a.n_blocks; ++b) {
    // ---- A: the block's proposals, drawn identically by every CTA
    double logh = 0.0;
    if (tid < k) {
      const int n = a.blocks[(long long)b * k + tid];
      sraw[tid] = n;
      a.stamp[n] = (b << 8) | tid;
      double y[D];
      logh = mh_propose_one<D>(n, tid, b, key, it, scale, a.kind, a.xcur, a.centre, a.size, y);
      const double* rn = a.rec + (long long)n * L::REC;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        sx_old[tid * D + d] = rn[d];
        sx_new[tid * D + d] = y[d];
      }
      stt[tid] = rn[D];
      sg[tid] = a.gid[n];
      // read before any CTA's phase-D commit can rewrite it (written by another CTA's commit
      // of an earlier block: bypass L1)
      sL0[tid] = __ldcg(a.rates + 4 * (long long)n) * S;
    }
    logh = cta_sum256(logh, red);
    if (tid == 0) s_hast = logh;
    __syncthreads();
    const StampSlots slots{a.stamp, b};

    // ---- B: rows outside S (delta units) and the moved rows (row units)
    for (int u = blockIdx.x; u < nb + k * nsplit; u += gridDim.x) {
      if (u < nb) {
        const int n = u * 256 + tid;
        double term = 0.0;
        if (n < N) {
          double dM = 0.0, dX = 0.0;
          if (slots(n) < 0) {
            const double* rn = a.rec + (long long)n * L::REC;
            double xn[D];
#pragma unroll
            for (int d = 0; d < D; ++d) xn[d] = rn[d];
            const double tn = rn[D];
            const int gn = a.gid[n];
            for (int q = 0; q < k; ++q) {
              double eb0, es0, eb1, es1;
              move_pair<D>(xn, tn, gn, sx_old + q * D, stt[q], sg[q], a.c, tab, eb0, es0);
              move_pair<D>(xn, tn, gn, sx_new + q * D, stt[q], sg[q], a.c, tab, eb1, es1);
              dM += eb1 - eb0;
              dX += es1 - es0;
            }
            term = move_term_out(a.rates[4 * (long long)n] * S, dM, dX, a.tx2, a.h2, a.floor_);
          }
          a.delta[2 * (long long)n] = dM;
          a.delta[2 * (long long)n + 1] = dX;
        }
        const double tsum = cta_sum256(term, red);
        if (tid == 0) a.part[u] = tsum;
        __syncthreads();
      } else {
        const int q = (u - nb) / nsplit, split = (u - nb) % nsplit;
        double xn[D];
#pragma unroll
        for (int d = 0; d < D; ++d) xn[d] = sx_new[q * D + d];
        const double tn = stt[q];
        const int gn = sg[q];
        const int j0 = split * len, j1 = min(N, j0 + len);
        double M = 0.0, X = 0.0;
        for (int j = j0 + tid; j < j1; j += blockDim.x) {
          const double* rj = a.rec + (long long)j * L::REC;
          const int sj = slots(j);
          const double* xj = sj >= 0 ? sx_new + sj * D : rj;
          double eb, es;
          move_pair<D>(xn, tn, gn, xj, rj[D], a.gid[j], a.c, tab, eb, es);
          M += eb;
          X += es;
        }
        cta_sum256x2(M, X, red);
        if (tid == 0) {
          const long long o = 2 * ((long long)q * nsplit + split);
          a.rows_part[o] = M;
          a.rows_part[o + 1] = X;
        }
        __syncthreads();
      }
    }
    grid.sync();

    // ---- D: the moved events' terms, the sum in the fixed order, the decision, the commit
    for (int q = tid >> 5; q < k; q += 8) {   // one warp per moved event
      double M, X;
      const double t = move_term_in(sL0[q], a.rows_part, q, nsplit, a.tx2, a.h2, a.floor_, M, X);
      if ((tid & 31) == 0) {
        sterm[q] = t;
        srow[2 * q] = M;
        srow[2 * q + 1] = X;
      }
    }
    double v = 0.0;
    for (int i = tid; i < nb; i += 256) v += __ldcg(a.part + i);
    v = cta_sum256(v, red);
    if (tid == 0) {
      double dl = v;
      for (int q = 0; q < k; ++q) dl += sterm[q];
      const double la = (dl > -INFINITY) ? dl + s_hast : -INFINITY;   // NaN -> -inf
      const double u = mh_uniforms(key, it, (unsigned)b, MH_ACCEPT_TAG).x;
      const int acc = log(u) < la ? 1 : 0;
      s_acc = acc;
      if (blockIdx.x == 0) {
        a.st->dell = dl;
        a.st->mh_hastings = s_hast;
        a.st->accepted = acc;
        a.acc_out[b] = acc;
        a.la_out[b] = la;
        if (acc) a.st->ell += dl;
      }
    }
    __syncthreads();
    if (s_acc) {
      for (int n = blockIdx.x * 256 + tid; n < N; n += gridDim.x * 256) {
        const int q = slots(n);
        double mu, xi;
        if (q < 0) {
          mu = __dadd_rn(a.rates[4 * (long long)n + 1], __dmul_rn(__dmul_rn(a.delta[2 * (long long)n], a.tx2), S1));
          xi = __dadd_rn(a.rates[4 * (long long)n + 2], __dmul_rn(__dmul_rn(a.delta[2 * (long long)n + 1], a.h2), S1));
          a.rates[4 * (long long)n] = __dadd_rn(a.rates[4 * (long long)n],
              __dmul_rn(fma(a.delta[2 * (long long)n], a.tx2, a.delta[2 * (long long)n + 1] * a.h2), S1));
        } else {
          mu = __dmul_rn(__dmul_rn(srow[2 * q], a.tx2), S1);
          xi = __dmul_rn(__dmul_rn(srow[2 * q + 1], a.h2), S1);
          a.rates[4 * (long long)n] = __dmul_rn(fma(srow[2 * q], a.tx2, srow[2 * q + 1] * a.h2), S1);
        }
        a.rates[4 * (long long)n + 1] = mu;
        a.rates[4 * (long long)n + 2] = xi;
      }
      for (int q = blockIdx.x * 256 + tid; q < k; q += gridDim.x * 256) {
        const int m = sraw[q];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const double val = sx_new[q * D + d];
          a.rec[(long long)m * L::REC + d] = val;
          a.xcur[(long long)m * D + d] = val;
          if (a.rec32) {
            const float hi = (float)val;
            a.rec32[(long long)m * Layout32<D>::REC + Layout32<D>::XH + d] = hi;
            a.rec32[(long long)m * Layout32<D>::REC + Layout32<D>::XL + d] = (float)(val - (double)hi);
          }
        }
      }
    }
    grid.sync();
  }
}

}  // namespace hk
