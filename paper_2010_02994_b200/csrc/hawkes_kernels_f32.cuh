// hawkes_kernels_f32.cuh -- fp32-accumulate variant of the two pass kernels (sm_100a).
//
// Same algebra as the fp64 kernels (hawkes_kernels.cuh: g_i = rho_i G1_i + G2_i, one
// background exp per pair and one self-excitation exp where its indicator can be
// non-zero), with
//  - pair arithmetic in fp32: locations and times stored as hi/lo float pairs
//    (v = hi + lo exactly to ~48 bits), differences formed as (hi_j - hi_i) + (lo_j - lo_i),
//    so absolute times of 1e4 (DC-shaped hours) keep ~1e-7 relative differences
//    (SURVEY.md §8(c) reading 17);
//  - exponents in the log2 domain with every constant (log2 e, the kernel weight, alpha or
//    beta, and a power-of-two scale 2^-E that puts the largest possible term near 2^20)
//    folded in, evaluated by one MUFU ex2.approx.ftz each;
//  - fp32 sums over one 128-event j-tile, promoted to the fp64 item accumulators after each
//    tile ("fp32-accumulate").
// Terms more than 2^146 below the largest possible term (exponent < ~-101) flush to 0.
#pragma once
#include "hawkes_kernels.cuh"

namespace hk {

template <int D>
struct Layout32 {
  static constexpr int XH = 0, XL = D, TH = 2 * D, TL = 2 * D + 1, RHO = 2 * D + 2;
  static constexpr int REC = ((2 * D + 3 + 3) / 4) * 4;  // floats per record (16 B multiple)
};

struct PassConst32 {
  float kx, kt, ks;   // -log2(e)/(2 tau_x^2), -log2(e)/(2 tau_t^2), -log2(e)/(2 h^2)
  float omega;        // omega log2(e)
  float cb, cs;       // log2(alpha w_b) - E, log2(beta w_s) - E
};

__device__ __forceinline__ float ex2f(float a) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a));
  return r;
}

template <int D>
struct RowState32 {
  float xh[D], xl[D];
  float th, tl;
  int g;
};

template <int D, int KIND>
__device__ __forceinline__ void pair32_pass1(const float* __restrict__ rj, int gj,
                                             const RowState32<D>& row, float& M, float& X,
                                             float (&G)[D], const PassConst32& c) {
  using L = Layout32<D>;
  float dx[D];
#pragma unroll
  for (int d = 0; d < D; ++d) dx[d] = (rj[L::XH + d] - row.xh[d]) + (rj[L::XL + d] - row.xl[d]);
  float r2 = dx[0] * dx[0];
#pragma unroll
  for (int d = 1; d < D; ++d) r2 = fmaf(dx[d], dx[d], r2);
  const float dt = (row.th - rj[L::TH]) + (row.tl - rj[L::TL]);
  float eb = ex2f(fmaf(c.kx, r2, fmaf(c.kt * dt, dt, c.cb)));
  if (KIND == KIND_MIXED) eb = (gj == row.g) ? 0.f : eb;
  if (KIND == KIND_LATER) {
    M += eb;
#pragma unroll
    for (int d = 0; d < D; ++d) G[d] = fmaf(eb, dx[d], G[d]);
  } else {
    float es = ex2f(fmaf(c.ks, r2, fmaf(-c.omega, dt, c.cs)));
    if (KIND == KIND_MIXED) es = (gj < row.g) ? es : 0.f;
    M += eb;
    X += es;
    const float cc = eb + es;
#pragma unroll
    for (int d = 0; d < D; ++d) G[d] = fmaf(cc, dx[d], G[d]);
  }
}

template <int D, int KIND>
__device__ __forceinline__ void pair32_pass2(const float* __restrict__ rj, int gj,
                                             const RowState32<D>& row, float (&G)[D],
                                             const PassConst32& c) {
  using L = Layout32<D>;
  float dx[D];
#pragma unroll
  for (int d = 0; d < D; ++d) dx[d] = (rj[L::XH + d] - row.xh[d]) + (rj[L::XL + d] - row.xl[d]);
  float r2 = dx[0] * dx[0];
#pragma unroll
  for (int d = 1; d < D; ++d) r2 = fmaf(dx[d], dx[d], r2);
  const float dt = (row.th - rj[L::TH]) + (row.tl - rj[L::TL]);
  const float rho = rj[L::RHO];
  float eb = ex2f(fmaf(c.kx, r2, fmaf(c.kt * dt, dt, c.cb)));
  if (KIND == KIND_MIXED) eb = (gj == row.g) ? 0.f : eb;
  float cc;
  if (KIND == KIND_EARLIER) {
    cc = rho * eb;
  } else {
    float es = ex2f(fmaf(c.ks, r2, fmaf(c.omega, dt, c.cs)));
    if (KIND == KIND_MIXED) es = (gj > row.g) ? es : 0.f;
    cc = rho * (eb + es);
  }
#pragma unroll
  for (int d = 0; d < D; ++d) G[d] = fmaf(cc, dx[d], G[d]);
}

struct PassArgs32 {
  const float* rec;      // Npad x REC floats
  const int* gid;
  const int2* items;
  int* counter;
  double* part;          // [chunks][Npad][K] (fp64, same layout as the fp64 path)
  long long npad;
  int N;
  int n_items;
  int chunk;
  PassConst32 c;
};

template <int D, int PASS, int R>
__global__ void __launch_bounds__(THREADS, 4) pass_kernel_f32(PassArgs32 a) {
  using L = Layout32<D>;
  using L64 = Layout<D>;
  constexpr int REC = L::REC;
  constexpr int RT = THREADS * R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + STAGES * TILE_J * REC * sizeof(float));
  __shared__ int s_item;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t parity = 0;
  const PassConst32 c = a.c;
  const int N = a.N;

  for (;;) {
    if (tid == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= a.n_items) break;
    const int2 w = a.items[it];
    const int row0 = w.x * RT;
    const int j0 = w.y * a.chunk;
    const int j1 = min(N, j0 + a.chunk);
    const int ntiles = (j1 - j0 + TILE_J - 1) / TILE_J;
    const int rlast = min(row0 + RT, N) - 1;
    const int g_first = a.gid[row0];
    const int g_last = a.gid[rlast];

    RowState32<D> row[R];
    double M[R], X[R], G[R][D];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = min(row0 + tid + r * THREADS, N - 1);
      const float* ri = a.rec + (long long)i * REC;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        row[r].xh[d] = ri[L::XH + d];
        row[r].xl[d] = ri[L::XL + d];
      }
      row[r].th = ri[L::TH];
      row[r].tl = ri[L::TL];
      row[r].g = a.gid[i];
      M[r] = 0.0;
      X[r] = 0.0;
#pragma unroll
      for (int d = 0; d < D; ++d) G[r][d] = 0.0;
    }

    if (tid == 0) {
      for (int s = 0; s < STAGES && s < ntiles; ++s) {
        const int jt = j0 + s * TILE_J;
        const int cnt = min(TILE_J, j1 - jt);
        tma_load_1d(stage + s * TILE_J * REC, a.rec + (long long)jt * REC,
                    (uint32_t)(cnt * REC * sizeof(float)), &bars[s]);
      }
    }

    for (int tl = 0; tl < ntiles; ++tl) {
      const int s = tl % STAGES;
      const int jt = j0 + tl * TILE_J;
      const int cnt = min(TILE_J, j1 - jt);
      const int gj_first = a.gid[jt];
      const int gj_last = a.gid[jt + cnt - 1];
      mbar_wait(&bars[s], (parity >> s) & 1u);
      parity ^= (1u << s);
      const float* st = stage + s * TILE_J * REC;
      const int kind = (gj_last < g_first) ? KIND_EARLIER
                                           : ((gj_first > g_last) ? KIND_LATER : KIND_MIXED);
      float m32[R], x32[R], g32[R][D];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        m32[r] = 0.f;
        x32[r] = 0.f;
#pragma unroll
        for (int d = 0; d < D; ++d) g32[r][d] = 0.f;
      }
      if (kind == KIND_EARLIER) {
#pragma unroll 4
        for (int jj = 0; jj < cnt; ++jj) {
          const float* rj = st + jj * REC;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (PASS == 1)
              pair32_pass1<D, KIND_EARLIER>(rj, 0, row[r], m32[r], x32[r], g32[r], c);
            else
              pair32_pass2<D, KIND_EARLIER>(rj, 0, row[r], g32[r], c);
          }
        }
      } else if (kind == KIND_LATER) {
#pragma unroll 4
        for (int jj = 0; jj < cnt; ++jj) {
          const float* rj = st + jj * REC;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (PASS == 1)
              pair32_pass1<D, KIND_LATER>(rj, 0, row[r], m32[r], x32[r], g32[r], c);
            else
              pair32_pass2<D, KIND_LATER>(rj, 0, row[r], g32[r], c);
          }
        }
      } else {
        for (int jj = 0; jj < cnt; ++jj) {
          const float* rj = st + jj * REC;
          const int gj = a.gid[jt + jj];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (PASS == 1)
              pair32_pass1<D, KIND_MIXED>(rj, gj, row[r], m32[r], x32[r], g32[r], c);
            else
              pair32_pass2<D, KIND_MIXED>(rj, gj, row[r], g32[r], c);
          }
        }
      }
      // promote the tile's fp32 sums
#pragma unroll
      for (int r = 0; r < R; ++r) {
        M[r] += (double)m32[r];
        X[r] += (double)x32[r];
#pragma unroll
        for (int d = 0; d < D; ++d) G[r][d] += (double)g32[r][d];
      }
      __syncthreads();
      if (tid == 0 && tl + STAGES < ntiles) {
        const int jn = j0 + (tl + STAGES) * TILE_J;
        const int cn = min(TILE_J, j1 - jn);
        tma_load_1d(stage + s * TILE_J * REC, a.rec + (long long)jn * REC,
                    (uint32_t)(cn * REC * sizeof(float)), &bars[s]);
      }
    }

#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = row0 + tid + r * THREADS;
      if (i < N) {
        if (PASS == 1) {
          double* o = a.part + ((long long)w.y * a.npad + i) * L64::K1;
          o[0] = M[r];
          o[1] = X[r];
#pragma unroll
          for (int d = 0; d < D; ++d) o[2 + d] = G[r][d];
        } else {
          double* o = a.part + ((long long)w.y * a.npad + i) * L64::K2;
#pragma unroll
          for (int d = 0; d < D; ++d) o[d] = G[r][d];
        }
      }
    }
  }
}

}  // namespace hk
