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
  float st, oms;      // sqrt(-kt) and -omega / st: rebased times u = st (t - T0) (REB = 1)
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
__global__ void __launch_bounds__(THREADS, D <= 4 ? 4 : 3) pass_kernel_f32(PassArgs32 a) {
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

// --------------------------------------------------------------------------------------
// fp32 unordered-pair kernel: hawkes_kernels_sym.cuh's chunk-pair mapping (R rows per lane,
// 32-step skewed column schedule, column sums rotating through warp shuffles) with the
// fp32 pair arithmetic above.  Row sums are fp32 over one 128-column tile and promoted to
// fp64 after it; column sums are fp32 over the 128 rows of a row tile and promoted when
// they are added to the fp64 partial slot.
#include "hawkes_kernels_sym.cuh"

namespace hk {

// Two rows of one lane against one column, packed into f32x2 instructions (sm_100
// FADD2/FMUL2/FFMA2): every FP32 instruction serves two pairs; the two exps stay on MUFU.
// Row data are stored negated (nxh = -x_hi, ...) so differences are packed adds.
template <int D>
struct RowPair32 {
  float2 nxh[D], nxl[D];
  float2 nth, ntl, rho;
  float2 nrt;      // REB 1: -(t - T0) of the two rows, T0 the current column tile's first time
  float2 nxr[D];   // REB 2: -(x - O) of the two rows, O the current column tile's first location
  int ga, gb;
};

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }

// GEN (spatial walk, as in the fp64 kernels): either event may be the later one; the
// self-excitation term uses |dt| and goes to the later event (pass 1: the row's X or the
// column's; pass 2: rho' of the later event in the coefficient).
// REB = 1 (time walk): the column's time arrives as t_j - T0 and the rows' as -(t_i - T0), T0
// the column tile's first time (sym_kernel_f32), so dt is one packed add instead of three;
// REB = 2 (spatial walk): the same for the locations, relative to the column tile's first one
template <int D, int PASS, bool MASK, bool SELF, bool GEN = false, int REB = 0>
__device__ __forceinline__ void sym32_pair2(const RowPair32<D>& rp, const float (&cxh)[D],
                                            const float (&cxl)[D], float cth, float ctl,
                                            float crho, bool dead_a, bool dead_b, float2& rM,
                                            float2& rX, float2 (&rG)[D], float2& cM, float2& cX,
                                            float2 (&cG)[D], const PassConst32& c) {
  float2 dx[D];
#pragma unroll
  for (int d = 0; d < D; ++d)
    dx[d] = REB == 2 ? __fadd2_rn(f2(cxh[d]), rp.nxr[d])
                     : __fadd2_rn(__fadd2_rn(f2(cxh[d]), rp.nxh[d]), __fadd2_rn(f2(cxl[d]), rp.nxl[d]));
  float2 r2 = __fmul2_rn(dx[0], dx[0]);
#pragma unroll
  for (int d = 1; d < D; ++d) r2 = __ffma2_rn(dx[d], dx[d], r2);
  // REB = 1: dt holds du = st dt (the times arrive scaled), so k_t dt^2 = -du^2 needs no multiply
  const float2 dt = REB == 1 ? __fadd2_rn(f2(cth), rp.nrt)
                         : __fadd2_rn(__fadd2_rn(f2(cth), rp.nth), __fadd2_rn(f2(ctl), rp.ntl));
  const float2 ab = REB == 1 ? __ffma2_rn(f2(c.kx), r2, __ffma2_rn(make_float2(-dt.x, -dt.y), dt, f2(c.cb)))
                             : __ffma2_rn(f2(c.kx), r2, __ffma2_rn(__fmul2_rn(f2(c.kt), dt), dt, f2(c.cb)));
  const float2 adt = GEN ? make_float2(fabsf(dt.x), fabsf(dt.y)) : dt;
  const float2 as = SELF ? __ffma2_rn(f2(c.ks), r2, __ffma2_rn(f2(REB == 1 ? c.oms : -c.omega), adt, f2(c.cs)))
                         : make_float2(0.f, 0.f);
  float2 eb = make_float2(ex2f(ab.x), ex2f(ab.y));
  float2 es = SELF ? make_float2(ex2f(as.x), ex2f(as.y)) : make_float2(0.f, 0.f);
  if (MASK) {
    eb.x = dead_a ? 0.f : eb.x;
    es.x = dead_a ? 0.f : es.x;
    eb.y = dead_b ? 0.f : eb.y;
    es.y = dead_b ? 0.f : es.y;
  }
  if (PASS == 1) {   // rates only (the gradient comes out of pass 2)
    rM = __fadd2_rn(rM, eb);
    cM = __fadd2_rn(cM, eb);
    if (SELF) {
      if (GEN) {
        const bool la = __float_as_int(dt.x) < 0, lb = __float_as_int(dt.y) < 0;   // row later
        rX = __fadd2_rn(rX, make_float2(la ? es.x : 0.f, lb ? es.y : 0.f));
        cX = __fadd2_rn(cX, make_float2(la ? 0.f : es.x, lb ? 0.f : es.y));
      } else {
        cX = __fadd2_rn(cX, es);
      }
    }
  } else {
    // the pair's App. A coefficient rho'_i mu' + rho'_j (mu' + xi'), the same for both events
    // (GEN: rho'_i mu' + rho'_j mu' + rho'_later xi')
    float2 cc;
    if (GEN) {
      const float2 rl = make_float2(__float_as_int(dt.x) < 0 ? rp.rho.x : crho,
                                    __float_as_int(dt.y) < 0 ? rp.rho.y : crho);
      const float2 rs = __fadd2_rn(rp.rho, f2(crho));
      cc = SELF ? __ffma2_rn(rs, eb, __fmul2_rn(rl, es)) : __fmul2_rn(rs, eb);
    } else {
      cc = __ffma2_rn(rp.rho, eb, __fmul2_rn(f2(crho), SELF ? __fadd2_rn(eb, es) : eb));
    }
    const float2 ncc = make_float2(-cc.x, -cc.y);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      rG[d] = __ffma2_rn(cc, dx[d], rG[d]);
      cG[d] = __ffma2_rn(ncc, dx[d], cG[d]);
    }
  }
}

template <int D, int PASS, bool MASK, int SR, bool SELF, bool SOA, bool GEN, bool PIECE, int REB = 0>
__device__ __forceinline__ void sym32_group_t(const RowPair32<D> (&rp)[SR / 2],
                                            const float* __restrict__ grp, int cg0, bool cvalid0,
                                            int ridx0, int cidx0, bool diag, int s0, int s1,
                                            float2 (&rM)[SR / 2], float2 (&rX)[SR / 2],
                                            float2 (&rG)[SR / 2][D],
                                            float (&cacc)[2 + D], const PassConst32& c) {
  using L = Layout32<D>;
  constexpr int REC = L::REC;
  const int lane = threadIdx.x & 31;
  if (!PIECE) s0 = 0, s1 = 32;   // PIECE: a step range (hawkes_kernels_sym.cuh sym_group)
  if (PIECE && s0) rotate_cols<D, PASS>(cacc, (lane + s0) & 31);
#pragma unroll 2
  for (int s = s0; s < s1; ++s) {
    const int src = (lane + s) & 31;
    // AoS record in the stage, or (SOA) the warp's transposed copy: float4 unit u of column
    // e at [u][e], read without bank conflicts
    float rbuf[REC];
    const float* rc;
    if (SOA) {
      const float4* g4 = reinterpret_cast<const float4*>(grp);
#pragma unroll
      for (int u = 0; u < REC / 4; ++u) {
        const float4 w = g4[u * 32 + src];
        rbuf[4 * u] = w.x;
        rbuf[4 * u + 1] = w.y;
        rbuf[4 * u + 2] = w.z;
        rbuf[4 * u + 3] = w.w;
      }
      rc = rbuf;
    } else {
      rc = grp + src * REC;
    }
    float cxh[D], cxl[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      cxh[d] = rc[L::XH + d];
      cxl[d] = rc[L::XL + d];
    }
    const float cth = rc[L::TH], ctl = rc[L::TL];
    const float crho = PASS == 2 ? rc[L::RHO] : 0.f;
    int cg = 0;
    bool cv = true;
    if (MASK) {
      cg = __shfl_sync(0xffffffffu, cg0, src);
      cv = __shfl_sync(0xffffffffu, (int)cvalid0, src) != 0;
    }
    // a padding column of a ragged tile holds stale shared memory (NaN patterns included):
    // zero its values so the masked terms are exactly 0 (0 * NaN would not be)
    const float crho_v = (MASK && !cv) ? 0.f : crho;
    if (MASK && !cv) {
#pragma unroll
      for (int d = 0; d < D; ++d) cxh[d] = cxl[d] = 0.f;
    }
    const float cth_v = (MASK && !cv) ? 0.f : cth, ctl_v = (MASK && !cv) ? 0.f : ctl;
    float2 cM = make_float2(cacc[0], 0.f), cX = make_float2(cacc[1], 0.f), cG[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cG[d] = make_float2(cacc[2 + d], 0.f);
#pragma unroll
    for (int h = 0; h < SR / 2; ++h) {
      bool da = false, db = false;
      if (MASK) {
        const int ia = ridx0 + 32 * (2 * h), ib = ridx0 + 32 * (2 * h + 1);
        da = !cv || rp[h].ga < 0 || cg == rp[h].ga || (diag && cidx0 + src <= ia);
        db = !cv || rp[h].gb < 0 || cg == rp[h].gb || (diag && cidx0 + src <= ib);
      }
      sym32_pair2<D, PASS, MASK, SELF, GEN, REB>(rp[h], cxh, cxl, cth_v, ctl_v, crho_v, da, db, rM[h],
                                                  rX[h], rG[h], cM, cX, cG, c);
    }
    if (PASS == 1) {
      cacc[0] = cM.x + cM.y;
      cacc[1] = cX.x + cX.y;
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) cacc[2 + d] = cG[d].x + cG[d].y;
    }
    const int nxt = (lane + 1) & 31;
    if (PASS == 1) {
      cacc[0] = __shfl_sync(0xffffffffu, cacc[0], nxt);
      cacc[1] = __shfl_sync(0xffffffffu, cacc[1], nxt);
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) cacc[2 + d] = __shfl_sync(0xffffffffu, cacc[2 + d], nxt);
    }
  }
  if (PIECE && s1 != 32) rotate_cols<D, PASS>(cacc, (lane - s1) & 31);
}

// REB kernels: the unmasked tile pairs whose column tile passed the span test take the
// rebased times / locations (reb), the others -- and every masked tile pair -- the hi/lo
// differences
template <int D, int PASS, bool MASK, int SR, bool SELF, bool SOA, bool GEN, bool PIECE, int REB>
__device__ __forceinline__ void sym32_group(const RowPair32<D> (&rp)[SR / 2],
                                            const float* __restrict__ grp, int cg0, bool cvalid0,
                                            int ridx0, int cidx0, bool diag, int s0, int s1,
                                            float2 (&rM)[SR / 2], float2 (&rX)[SR / 2],
                                            float2 (&rG)[SR / 2][D],
                                            float (&cacc)[2 + D], const PassConst32& c, bool reb) {
  if (REB && !MASK && reb)
    sym32_group_t<D, PASS, MASK, SR, SELF, SOA, GEN, PIECE, REB>(rp, grp, cg0, cvalid0, ridx0, cidx0, diag,
                                                                  s0, s1, rM, rX, rG, cacc, c);
  else
    sym32_group_t<D, PASS, MASK, SR, SELF, SOA, GEN, PIECE, 0>(rp, grp, cg0, cvalid0, ridx0, cidx0, diag,
                                                                   s0, s1, rM, rX, rG, cacc, c);
}

struct SymArgs32 {
  const float* rec;          // records in the walk's order (time order, or spatial: rec32_p)
  const double* boxes;       // GEN: per 128-event tile {lo[D], hi[D], tmin, tmax} (fp64)
  int ties;                  // GEN: the catalog has equal times
  const int* gid;
  const PairItem* items;   // chunk pairs and their slot blocks (hawkes_kernels_sym.cuh)
  int* counter;
  double* part;
  long long npad;
  int N;
  int n_items;
  int chunk;
  int nchunks;
  int piece;                 // host side: the plan is made of pieces (SymArgs.piece)
  PassConst32 c;
};

// box bounds in the fp32 kernels' log2 domain (the 2^-E scale folded into cb, cs): a term
// whose bound is below -127 is flushed by ex2.approx.ftz
template <int D>
__device__ __forceinline__ void box_bounds32(const double* lo_a, const double* hi_a, const double* lo_b,
                                             const double* hi_b, const PassConst32& c, bool& bg, bool& self) {
  double r2 = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double g = fmax(0.0, fmax(lo_b[d] - hi_a[d], lo_a[d] - hi_b[d]));
    r2 = fma(g, g, r2);
  }
  const float dt = (float)fmax(0.0, fmax(lo_b[D] - hi_a[D], lo_a[D] - hi_b[D]));
  const float r2f = (float)r2;
  bg = fmaf(c.kx, r2f, fmaf(c.kt * dt, dt, c.cb)) > -127.f;
  self = fmaf(c.ks, r2f, c.cs - c.omega * dt) > -127.f;
}

template <int D, int PASS, int SR, bool SOA, bool GEN = false, bool PIECE = false>
__global__ void __launch_bounds__(THREADS, D <= 2 ? 4 : (D <= 4 ? 3 : 2)) sym_kernel_f32(SymArgs32 a) {
  static_assert(32 * SR == TILE_J, "row tiles and column tiles must coincide");
  constexpr int SRT = 32 * SR;
  using L = Layout32<D>;
  using L64 = Layout<D>;
  constexpr int REC = L::REC;
  constexpr int K = PASS == 1 ? K1P : L64::K2;
  constexpr int KR = PASS == 1 ? (GEN ? 2 : 1) : D;
  // rebased differences (below): times on the time walk, locations on the spatial walk
#ifdef HK_NO_TREB   // A/B: hi/lo time differences in every pair
  constexpr bool TREB = false;
#else
  constexpr bool TREB = SOA && !GEN;
#endif
#ifdef HK_NO_XREB   // A/B: hi/lo location differences in every pair
  constexpr bool XREB = false;
#else
  constexpr bool XREB = SOA && GEN;
#endif
  constexpr int REBK = TREB ? 1 : (XREB ? 2 : 0);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + STAGES * TILE_J * REC * sizeof(float));
  double* red = reinterpret_cast<double*>(bars + STAGES);   // [4 warps][SRT][KR]
  float* soa = reinterpret_cast<float*>(red + 4 * SRT * KR);  // [4 warps][REC/4][32] float4
  __shared__ int s_item;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* mysoa = soa + warp * 32 * REC;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  pdl_wait();
  uint32_t parity = 0;
  const PassConst32 c = a.c;
  const int N = a.N;

  // (drawing the next item's index early -- during the item's last tile pair -- was measured
  // slower at small N, where an item is one tile pair: a CTA then holds its next item for a
  // whole item, N = 5000 +6 %; profiles/r02_latency_prefetch.jsonl)
  for (;;) {
    if (tid == 0) s_item = atomicAdd(a.counter, 1);
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    if (it >= a.n_items) break;
    const PairItem w = a.items[it];
    const bool diag = w.a == w.b;
    const int r0 = w.a * a.chunk;
    const int r1 = min(N, r0 + a.chunk);
    const int c0 = w.b * a.chunk;
    const int c1 = min(N, c0 + a.chunk);
    const int n_rt = (r1 - r0 + SRT - 1) / SRT;
    const int n_ct = (c1 - c0 + TILE_J - 1) / TILE_J;
    if (GEN && !diag) {   // item-level cull by the chunks' union boxes (see sym_items)
      double lo_a[D + 1], hi_a[D + 1], lo_b[D + 1], hi_b[D + 1];
#pragma unroll
      for (int d = 0; d <= D; ++d) {
        lo_a[d] = lo_b[d] = INFINITY;
        hi_a[d] = hi_b[d] = -INFINITY;
      }
      for (int q = 0; q < n_rt + n_ct; ++q) {
        const bool ra = q < n_rt;
        const double* b = a.boxes + (long long)((ra ? r0 : c0) / TILE_J + (ra ? q : q - n_rt)) * (2 * D + 2);
        double* lo = ra ? lo_a : lo_b;
        double* hi = ra ? hi_a : hi_b;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          lo[d] = fmin(lo[d], b[d]);
          hi[d] = fmax(hi[d], b[D + d]);
        }
        lo[D] = fmin(lo[D], b[2 * D]);
        hi[D] = fmax(hi[D], b[2 * D + 1]);
      }
      bool bg, self;
      box_bounds32<D>(lo_a, hi_a, lo_b, hi_b, c, bg, self);
      if (!bg && !self) {
        for (int q = tid; q < (r1 - r0) * K; q += THREADS) a.part[w.ro * K + q] = 0.0;
        for (int q = tid; q < (c1 - c0) * K; q += THREADS) a.part[w.co * K + q] = 0.0;
        continue;
      }
    }

    TileWalk prod{0, 0};
    if (tid == 0) {
      for (int s = 0; s < STAGES && prod.rt < n_rt; ++s, prod.next(n_ct, diag)) {
        const int jt = c0 + prod.ct * TILE_J;
        const int cnt = min(TILE_J, c1 - jt);
        tma_load_1d(stage + s * TILE_J * REC, a.rec + (long long)jt * REC,
                    (uint32_t)(cnt * REC * sizeof(float)), &bars[s]);
      }
    }

    int k = 0;
    for (int rt = 0; rt < n_rt; ++rt) {
      const int row0 = r0 + rt * SRT;
      const bool rows_full = row0 + SRT <= r1;
      RowPair32<D> rp[SR / 2];
      double rM[SR], rX[SR], rG[SR][D];
#pragma unroll
      for (int h = 0; h < SR / 2; ++h) {
        const int ia = row0 + lane + 32 * (2 * h), ib = ia + 32;
        const float* ra = a.rec + (long long)min(ia, N - 1) * REC;
        const float* rb = a.rec + (long long)min(ib, N - 1) * REC;
#pragma unroll
        for (int d = 0; d < D; ++d) {
          rp[h].nxh[d] = make_float2(-ra[L::XH + d], -rb[L::XH + d]);
          rp[h].nxl[d] = make_float2(-ra[L::XL + d], -rb[L::XL + d]);
        }
        rp[h].nth = make_float2(-ra[L::TH], -rb[L::TH]);
        rp[h].ntl = make_float2(-ra[L::TL], -rb[L::TL]);
        rp[h].rho = make_float2(ra[L::RHO], rb[L::RHO]);
        rp[h].ga = ia < N ? a.gid[ia] : -1;
        rp[h].gb = ib < N ? a.gid[ib] : -1;
      }
#pragma unroll
      for (int r = 0; r < SR; ++r) {
        rM[r] = 0.0;
        rX[r] = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) rG[r][d] = 0.0;
      }
      const double* rbox = GEN ? a.boxes + (long long)(row0 / TILE_J) * (2 * D + 2) : nullptr;
      const int rlast = min(row0 + SRT, r1) - 1;
      const int g_rlast = a.gid[rlast];
      const float th_rlast = a.rec[(long long)rlast * REC + L::TH];
      const float tl_rlast = a.rec[(long long)rlast * REC + L::TL];

      for (int ct = diag ? rt : 0; ct < n_ct; ++ct, ++k) {
        const int s = k % STAGES;
        const int jt = c0 + ct * TILE_J;
        const int cnt = min(TILE_J, c1 - jt);
        mbar_wait(&bars[s], (parity >> s) & 1u);
        parity ^= (1u << s);
        const float* st = stage + s * TILE_J * REC;
        const int cl = warp * 32 + lane;
        const bool cvalid = cl < cnt;
        const int cj = jt + min(cl, cnt - 1);
        const int cg = a.gid[cj];
        double* cpart = a.part + (w.co + (cj - c0)) * K;
        float cacc[2 + D];
#pragma unroll
        for (int q = 0; q < 2 + D; ++q) cacc[q] = 0.f;
        float2 rM32[SR / 2], rX32[SR / 2], rG32[SR / 2][D];
#pragma unroll
        for (int h = 0; h < SR / 2; ++h) {
          rM32[h] = make_float2(0.f, 0.f);
          rX32[h] = make_float2(0.f, 0.f);
#pragma unroll
          for (int d = 0; d < D; ++d) rG32[h][d] = make_float2(0.f, 0.f);
        }
        const bool diag_tile = diag && ct == rt;
        const bool strict = !diag_tile && rows_full && cnt == TILE_J && (GEN ? !a.ties : g_rlast < a.gid[jt]);
        // temporal culling as in the fp64 kernel, in the log2 domain: ex2.approx.ftz
        // returns 0 below 2^-126 (with the 2^-E scale already folded into cb, cs); GEN: the
        // two tiles' boxes in space and time
        bool self_live, bg_live;
        if (GEN) {
          const double* cb = a.boxes + (long long)(jt / TILE_J) * (2 * D + 2);
          double lo_r[D + 1], hi_r[D + 1], lo_c[D + 1], hi_c[D + 1];
#pragma unroll
          for (int d = 0; d < D; ++d) {
            lo_r[d] = rbox[d];
            hi_r[d] = rbox[D + d];
            lo_c[d] = cb[d];
            hi_c[d] = cb[D + d];
          }
          lo_r[D] = rbox[2 * D];
          hi_r[D] = rbox[2 * D + 1];
          lo_c[D] = cb[2 * D];
          hi_c[D] = cb[2 * D + 1];
          box_bounds32<D>(lo_r, hi_r, lo_c, hi_c, c, bg_live, self_live);
        } else {
          const float dtmin = fmaxf((st[L::TH] - th_rlast) + (st[L::TL] - tl_rlast), 0.f);
          self_live = c.cs - c.omega * dtmin > -127.f;
          bg_live = fmaf(c.kt * dtmin, dtmin, c.cb) > -127.f;
        }
        const float* grp = st + warp * 32 * REC;
        // TREB (time walk: tiles are time ranges): times relative to T0 = this column tile's
        // first time -- the column's t_j - T0 replaces its t_hi in the transposed copy, the
        // rows' -(t_i - T0) is formed here, so each pair's dt is one packed add.  The rounding
        // of t - T0 is u32 |t - T0| <= u32 (|dt| + span of the tile), against u32 |dt| for the
        // hi/lo difference: the same order for every pair whose terms survive the flush
        // ... only where the column tile's time span is short against the time scales: its
        // rounding adds u32 (omega log2e span) to the self-excitation exponent and u32 (2 |k_t|
        // dt span) to the background one, so omega log2e span <= 64 and |k_t| span^2 <= 64 keep
        // both within the hi/lo form's error class (a sparse-in-time catalog with a large omega
        // keeps the hi/lo differences: fuzz seed 44 without this guard, 1.5x the fp32 gate)
        bool treb = false;
        if (TREB && strict) {   // (masked tile pairs read the hi/lo times)
          const float* lastc = st + (cnt - 1) * REC;
          const float span = (lastc[L::TH] - st[L::TH]) + (lastc[L::TL] - st[L::TL]);
          treb = c.omega * span <= 64.f && c.kt * span * span >= -64.f;
        }
        if (treb) {
          const float T0h = st[L::TH], T0l = st[L::TL];
#pragma unroll
          for (int h = 0; h < SR / 2; ++h)
            rp[h].nrt = __fmul2_rn(f2(c.st), __fadd2_rn(__fadd2_rn(rp[h].nth, f2(T0h)), __fadd2_rn(rp[h].ntl, f2(T0l))));
        }
        // XREB (spatial walk: tiles are compact in space): the same for the locations, relative
        // to O = the column tile's first location, where the column tile's extent E around O
        // (its box) keeps u32 |k| E^2-sized exponent errors small: |k| E^2 <= 64 for both
        // kernels' k (log2 domain)
        bool xreb = false;
        if (XREB && strict) {
          const double* cbx = a.boxes + (long long)(jt / TILE_J) * (2 * D + 2);
          float e = 0.f;
#pragma unroll
          for (int d = 0; d < D; ++d) {
            const double o = (double)st[L::XH + d] + (double)st[L::XL + d];
            e = fmaxf(e, (float)fmax(cbx[D + d] - o, o - cbx[d]));
          }
          xreb = fminf(c.kx, c.ks) * e * e >= -64.f;
        }
        if (xreb) {
#pragma unroll
          for (int h = 0; h < SR / 2; ++h)
#pragma unroll
            for (int d = 0; d < D; ++d)
              rp[h].nxr[d] = __fadd2_rn(__fadd2_rn(rp[h].nxh[d], f2(st[L::XH + d])),
                                        __fadd2_rn(rp[h].nxl[d], f2(st[L::XL + d])));
        }
        if (SOA) {   // this lane's column record -> the warp's [unit][32] float4 buffer
          const float4* rc4 = reinterpret_cast<const float4*>(grp + lane * REC);
          float4* g4 = reinterpret_cast<float4*>(mysoa);
          if (treb || xreb) {
            float v[REC];
#pragma unroll
            for (int u = 0; u < REC / 4; ++u) {
              const float4 w4 = rc4[u];
              v[4 * u] = w4.x;
              v[4 * u + 1] = w4.y;
              v[4 * u + 2] = w4.z;
              v[4 * u + 3] = w4.w;
            }
            if (treb) v[L::TH] = c.st * ((v[L::TH] - st[L::TH]) + (v[L::TL] - st[L::TL]));
            if (xreb) {
#pragma unroll
              for (int d = 0; d < D; ++d)
                v[L::XH + d] = (v[L::XH + d] - st[L::XH + d]) + (v[L::XL + d] - st[L::XL + d]);
            }
#pragma unroll
            for (int u = 0; u < REC / 4; ++u)
              g4[u * 32 + lane] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
          } else {
#pragma unroll
            for (int u = 0; u < REC / 4; ++u) g4[u * 32 + lane] = rc4[u];
          }
          __syncwarp();
          grp = mysoa;
        }
        if (!strict)   // PIECE: as sym_items; the masked tiles keep the hi/lo differences
          sym32_group<D, PASS, true, SR, true, SOA, GEN, PIECE, REBK>(rp, grp, cg, cvalid, row0 + lane,
                                                                      jt + warp * 32, diag_tile, w.s0, w.s1,
                                                                      rM32, rX32, rG32, cacc, c, treb || xreb);
        else if (self_live)
          sym32_group<D, PASS, false, SR, true, SOA, GEN, PIECE, REBK>(rp, grp, cg, cvalid, row0 + lane,
                                                                       jt + warp * 32, false, w.s0, w.s1,
                                                                       rM32, rX32, rG32, cacc, c, treb || xreb);
        else if (bg_live)
          sym32_group<D, PASS, false, SR, false, SOA, GEN, PIECE, REBK>(rp, grp, cg, cvalid, row0 + lane,
                                                                        jt + warp * 32, false, w.s0, w.s1,
                                                                        rM32, rX32, rG32, cacc, c, treb || xreb);
#pragma unroll
        for (int h = 0; h < SR / 2; ++h) {
          rM[2 * h] += (double)rM32[h].x;
          rM[2 * h + 1] += (double)rM32[h].y;
          if (GEN && PASS == 1) {
            rX[2 * h] += (double)rX32[h].x;
            rX[2 * h + 1] += (double)rX32[h].y;
          }
#pragma unroll
          for (int d = 0; d < D; ++d) {
            rG[2 * h][d] += (double)rG32[h][d].x;
            rG[2 * h + 1][d] += (double)rG32[h][d].y;
          }
        }
        if (cvalid) {
          if (PASS == 1) {
#pragma unroll
            for (int q = 0; q < 2; ++q) cpart[q] = (rt ? cpart[q] : 0.0) + (double)cacc[q];
          } else {
#pragma unroll
            for (int d = 0; d < D; ++d) cpart[d] = (rt ? cpart[d] : 0.0) + (double)cacc[2 + d];
          }
        }
        __syncthreads();
        if (tid == 0 && prod.rt < n_rt) {
          const int jn = c0 + prod.ct * TILE_J;
          const int cn = min(TILE_J, c1 - jn);
          tma_load_1d(stage + s * TILE_J * REC, a.rec + (long long)jn * REC,
                      (uint32_t)(cn * REC * sizeof(float)), &bars[s]);
          prod.next(n_ct, diag);
        }
      }
#pragma unroll
      for (int r = 0; r < SR; ++r) {
        double* o = red + ((long long)warp * SRT + lane + 32 * r) * KR;
        if (PASS == 1) {
          o[0] = rM[r];
          if (GEN) o[1] = rX[r];
        } else {
#pragma unroll
          for (int d = 0; d < D; ++d) o[d] = rG[r][d];
        }
      }
      __syncthreads();
      for (int q = tid; q < SRT * KR; q += THREADS) {
        const int rr = q / KR, kk = q % KR;
        if (row0 + rr >= N) continue;
        double v = red[(0 * SRT + rr) * KR + kk];
        v += red[(1 * SRT + rr) * KR + kk];
        v += red[(2 * SRT + rr) * KR + kk];
        v += red[(3 * SRT + rr) * KR + kk];
        double* o = a.part + (w.ro + (row0 + rr - r0)) * K;
        if (PASS == 1 && !GEN) {
          o[0] = v;
          o[1] = 0.0;
        } else {
          o[kk] = v;
        }
      }
      __syncthreads();
    }
  }
  pdl_trigger();   // out of items (as sym_kernel)
}

}  // namespace hk
