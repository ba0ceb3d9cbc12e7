// hawkes_kernels_sym.cuh -- unordered-pair ("symmetric") pass kernels, fp64 (sm_100a).
//
// SURVEY.md §8(f) NEXT-1.  mu_ij = mu_ji, and for t_i < t_j only xi_ji is non-zero
// (P:L98-99), so one evaluation of the two exps of an unordered pair {i, j} (i earlier)
// serves both events:
//   pass 1  row i: M += mu'                 col j: M += mu', X += xi'   (rates only)
//   pass 2  c = rho'_i mu' + rho'_j (mu' + xi'):   g_i += c dx,   g_j -= c dx
// with dx = x_j - x_i and the scaled-domain terms of hawkes_kernels.cuh (mu' = alpha mu 2^64,
// xi' = beta xi_ji 2^64).  App. A's coefficient of the pair is the same for both events
// ((mu_ij/lambda_i + mu_ji/lambda_j)/tau_x^2 + (xi_ij/lambda_i + xi_ji/lambda_j)/h^2 with
// xi_ij = 0), so the whole gradient comes out of pass 2 and pass 1 computes the rates alone
// (K1P = 2 partials per event: M', X').  Work items are chunk pairs (a, b), a <= b.  For a < b every event
// of chunk a precedes every event of chunk b in the time-sorted catalog; a diagonal item
// (a, a) visits only the upper triangle of its tile pairs and masks j <= i (by index, which
// is time order) on the diagonal tiles.  An item writes the row partial of chunk a's events
// into slot b and the column partial of chunk b's events into slot a (slot C for diagonal
// items) of a [C + 1][Npad][K] array, so every (slot, event) is written exactly once and
// the fixed-order finalize sums C + 1 slots.
//
// Mapping: a CTA (4 warps) holds a row tile of 32*R events (lane l owns rows l + 32r, all
// four warps hold the same rows) and streams column tiles of 128 events via TMA; warp w
// takes columns [32w, 32w+32) of each tile.  Lane l loads column l of its group, then in
// step s = 0..31 pairs its R rows with column (l + s) mod 32, obtained by warp shuffle,
// while the column's accumulators rotate one lane down per step: after 32 steps every
// row has met every column and lane l again holds column l's sums.  Row sums stay in
// registers across the column tiles and are reduced over the 4 warps in a fixed order.
#pragma once
#include "hawkes_kernels.cuh"

namespace hk {

constexpr int SYM_RMAX = 4;               // largest rows-per-lane variant
// -DHK_SYM_FOLD: pass 2 folds -ln lambda_j (staged beside the records) into the
// self-excitation exponent, so rho'_j xi' comes out of one exp and the coefficient costs one
// add and one fma instead of add, mul, fma: one FP64 instruction less per pair, but measured
// 5 % SLOWER (11.39 vs 10.83 ms at N = 100k, profiles/r02_ab_fold.jsonl): the per-tile bound of
// the staged -ln lambda (a warp max) makes the step loop's convergence non-uniform and the
// column's extra shared load sits on the exponent's dependency chain.  Off by default.
#ifdef HK_SYM_FOLD
constexpr bool SYM_FOLD = true;
#else
constexpr bool SYM_FOLD = false;
#endif
#ifdef HK_NO_REB1   // A/B: the rate pass without rebased times
constexpr bool REB1 = false;
#else
constexpr bool REB1 = true;
#endif
#ifdef HK_REB2      // A/B: the gradient pass with rebased times
constexpr bool REB2 = true;
#else
constexpr bool REB2 = false;
#endif
constexpr int K1P = 2;                    // pass-1 partials of the unordered-pair kernels: M', X' 
// a term whose exponent is below this adds nothing (fexp clamps at -707, and the finalize
// treats sums below N e^-700 as zero): tile pairs whose bound is lower skip the term
constexpr double CULL_EXPONENT = -708.0;
// V bits (DESIGN.md §4 "shared-memory banks"): 2 = the exp table in TAB_COPIES interleaved
// copies, lane l reading copy l & 15, so a half-warp's 16 lookups hit 16 distinct bank pairs;
// 4 = each warp transposes its 32-column group once per tile into a private structure-of-
// arrays buffer of double2 pairs, so the 32 steps read columns without bank conflicts
// 16 copies of the 256-entry table (32 KB); the 1024-entry table (8 KB) fits 4, the 2048-entry one 2
constexpr int TAB_COPIES = EXP_TABLE == 256 ? 16 : (EXP_TABLE == 1024 ? 4 : 2);

// One work item of the unordered-pair kernels: chunk pair (a, b), a <= b, and where its
// partial sums go.  The slot arrays are item-indexed and compact per rank (hawkes_engine.cuh
// build_plan_pairs): for each chunk c, one block of `chunk` events per slot that this rank's
// items write for c's events, the slots in ascending slot id (row role of item (c, b): slot b;
// column role of item (a, c), a < c: slot a; column role of the diagonal item (c, c): slot C),
// so a rank holds ~1/W of the partials and the finalize adds them in the same fixed order for
// every W.  ro / co: the event offsets of this item's row block (chunk a's events) and column
// block (chunk b's events) in the slot array.
// s0, s1: the skewed steps [s0, s1) of every tile pair this item runs (hawkes_plan.h
// pairs_layout splits the lightest items of a small plan into 2 or 4 step ranges, "pieces",
// each with its own row and column slot blocks; a whole item runs [0, 32)).
struct PairItem {
  int a, b;
  long long ro, co;
  int s0, s1;
};

// lane l takes v from lane src(l): the column-sum rotation of a step range that does not
// start (or end) at step 0 (or 32)
template <int D, int PASS, class T>
__device__ __forceinline__ void rotate_cols(T (&cacc)[2 + D], int src) {
  if (PASS == 1) {
    cacc[0] = __shfl_sync(0xffffffffu, cacc[0], src);
    cacc[1] = __shfl_sync(0xffffffffu, cacc[1], src);
  } else {
#pragma unroll
    for (int d = 0; d < D; ++d) cacc[2 + d] = __shfl_sync(0xffffffffu, cacc[2 + d], src);
  }
}

struct SymArgs {
  const double* rec;     // records in the item walk's order (time order, or spatial: rec_p)
  const double* boxes;   // GEN: per 128-event tile {lo[D], hi[D], tmin, tmax} (spatial order)
  int ties;              // GEN: the catalog has equal times (every tile pair takes the masked path)
  const double* lrho;    // pass 2: -ln lambda_j per event (npad), staged beside the records
  const int* gid;
  const PairItem* items; // chunk pairs and their slot blocks
  int* counter;
  double* part;          // item-indexed slot blocks (PairItem), K per event
  const int2* tab;
  long long npad;
  int N;
  int n_items;
  int piece;             // host side: the plan is made of pieces (launch the PIECE kernel)
  int chunk;
  int nchunks;           // slot nchunks holds the column-role sums of diagonal items
  PassConst c;          // by value: DFMA constant-bank operands
};

template <int D>
struct SymRow {
  double x[D];
  double t;
  double rho;
  double u;   // rate pass, REB: st (t - T0), T0 the current column tile's first time
  int g;
};

// one unordered pair, pass 1; MASK: tie (same time) or padding column -> no contribution.
// GEN (spatial order, hawkes_plan.h): the column may be earlier or later than the row; the
// self-excitation term is that of the later event, exponent k_s r^2 - omega |dt|, added to
// the row's X (row later) or the column's (column later).
// REB (time walk, strict tile pairs passing the span test in sym_items): the column's time
// arrives as u_j = st (t_j - T0) and the row's as u_i, so du = u_j - u_i = st dt and the
// background exponent's k_t dt^2 = -du^2 needs no multiply (one FP64 instruction less per pair)
template <int D, bool MASK, bool SELF, int TS, bool GEN = false, bool REB = false>
__device__ __forceinline__ void sym_pair1(const SymRow<D>& row, const double (&cx)[D], double ct,
                                          bool dead, double& rM, double& rX, double& cM, double& cX,
                                          const PassConst& c, const int2* __restrict__ tab) {
  double dx[D];
#pragma unroll
  for (int d = 0; d < D; ++d) dx[d] = cx[d] - row.x[d];
  double r2 = dx[0] * dx[0];
#pragma unroll
  for (int d = 1; d < D; ++d) r2 = fma(dx[d], dx[d], r2);
  const double dt = REB ? ct - row.u : ct - row.t;   // >= 0: the column is the later event
  const int lane_off = TS > 1 ? (int)(threadIdx.x & (TS - 1)) * 8 : 0;
  // the exp's k -> double on the conversion pipe (I2F.F64) in pass 1 as well: with the product
  // form's fewer FP64 instructions it pays at D = 2 (N = 100k 8.84 -> 8.81 ms, Alaska-shaped
  // time walk -1.2 %, DC-shaped spatial walk -0.3 %; profiles/r02_ab_final_variants.jsonl); it
  // cost 0.6-2.6 % before, and D >= 3 is unmeasured, so it stays off there
#if defined(HK_PASS1_I2F)      // A/B: for every D <= 5
  constexpr bool I2F1 = D <= 5;
#elif defined(HK_PASS1_NO_I2F)   // A/B: off
  constexpr bool I2F1 = false;
#else
  constexpr bool I2F1 = D <= 2;
#endif
#ifndef HK_NO_EXPFMA
  // product-form exps (fexp_tp): each accumulation is one fma(Tm, P, sum) -- 25 FP64
  // instructions per unordered pair instead of 27 (100 + 51.5 other per 4-pair step), measured
  // 9.00 -> 8.85 ms at N = 100k (profiles/r02_ab_expfma.jsonl; -DHK_NO_EXPFMA: the old form)
  double Tb, Pb, Ts = 0.0, Ps = 0.0;
  if (REB) {   // dt holds du = u_j - u_i here
    fexp_tp<TS, I2F1>(fma(c.kx, r2, fma(-dt, dt, c.lnc_b)), tab, lane_off, Tb, Pb);
    if (SELF) fexp_tp<TS, I2F1>(fma(c.ks, r2, fma(c.oms, dt, c.lnc_s)), tab, lane_off, Ts, Ps);
  } else {
    fexp_tp<TS, I2F1>(fma(c.kx, r2, fma(c.kt * dt, dt, c.lnc_b)), tab, lane_off, Tb, Pb);
    if (SELF)
      fexp_tp<TS, I2F1>(fma(c.ks, r2, fma(-c.omega, GEN ? fabs(dt) : dt, c.lnc_s)), tab, lane_off, Ts, Ps);
  }
  if (MASK) {
    Tb = dead ? 0.0 : Tb;
    Ts = dead ? 0.0 : Ts;
  }
  rM = fma(Tb, Pb, rM);
  cM = fma(Tb, Pb, cM);
  if (SELF) {
    if (GEN) {   // the later event takes xi (dt != 0 here: ties are masked)
      const bool row_later = __double2hiint(dt) < 0;
      rX = fma(row_later ? Ts : 0.0, Ps, rX);
      cX = fma(row_later ? 0.0 : Ts, Ps, cX);
    } else {
      cX = fma(Ts, Ps, cX);
    }
  }
  return;
#endif
  double eb = fexp<TS, I2F1>(fma(c.kx, r2, fma(c.kt * dt, dt, c.lnc_b)), tab, lane_off);
  double es = SELF ? fexp<TS, I2F1>(fma(c.ks, r2, fma(-c.omega, GEN ? fabs(dt) : dt, c.lnc_s)), tab, lane_off)
                   : 0.0;
  if (MASK) {
    eb = dead ? 0.0 : eb;
    es = dead ? 0.0 : es;
  }
  rM += eb;
  cM += eb;
  if (SELF) {
    if (GEN) {   // the later event takes xi (dt != 0 here: ties are masked)
      const bool row_later = __double2hiint(dt) < 0;
      rX += row_later ? es : 0.0;
      cX += row_later ? 0.0 : es;
    } else {
      cX += es;
    }
  }
}

template <int D, bool MASK, bool SELF, int TS, bool GEN = false, bool REB = false>
__device__ __forceinline__ void sym_pair2(const SymRow<D>& row, const double (&cx)[D], double ct,
                                          double crho, double cL, bool dead, double (&rG)[D],
                                          double (&cG)[D], const PassConst& c,
                                          const int2* __restrict__ tab) {
  double dx[D];
#pragma unroll
  for (int d = 0; d < D; ++d) dx[d] = cx[d] - row.x[d];
  double r2 = dx[0] * dx[0];
#pragma unroll
  for (int d = 1; d < D; ++d) r2 = fma(dx[d], dx[d], r2);
  const double dt = REB ? ct - row.u : ct - row.t;   // REB: du (sym_pair1)
  const int lane_off = TS > 1 ? (int)(threadIdx.x & (TS - 1)) * 8 : 0;
#ifdef HK_PASS2_NO_I2F
  constexpr bool I2F = false;
#else
  constexpr bool I2F = D <= 5;
#endif
#if defined(HK_PASS2_EXPFMA) && !defined(HK_SYM_FOLD)
  // A/B only: product-form exps (fexp_tp) in pass 2 too -- mu' = Tb Pb once (it is needed
  // twice), mu' + xi' as one fma: 4 FP64 instructions fewer per 4-pair step, but measured 0.9 %
  // SLOWER at N = 100k (10.62 vs 10.52 ms; the 128-register build rematerialises two exp
  // constants per step, and at 3 CTAs/SM, without them, 10.98 ms; profiles/r02_ab_expfma.jsonl)
  {
    double Ts = 0.0, Ps = 0.0;
#ifdef HK_EXPFMA_MIX   // mu' by fexp (it is needed as a value), xi' in product form
    double eb = fexp<TS, I2F>(fma(c.kx, r2, fma(c.kt * dt, dt, c.lnc_b)), tab, lane_off);
    if (SELF)
      fexp_tp<TS, I2F>(fma(c.ks, r2, fma(-c.omega, GEN ? fabs(dt) : dt, c.lnc_s)), tab, lane_off, Ts, Ps);
    if (MASK) {
      eb = dead ? 0.0 : eb;
      Ts = dead ? 0.0 : Ts;
    }
#else
    double Tb, Pb;
    if (REB) {
      fexp_tp<TS, I2F>(fma(c.kx, r2, fma(-dt, dt, c.lnc_b)), tab, lane_off, Tb, Pb);
      if (SELF) fexp_tp<TS, I2F>(fma(c.ks, r2, fma(c.oms, dt, c.lnc_s)), tab, lane_off, Ts, Ps);
    } else {
      fexp_tp<TS, I2F>(fma(c.kx, r2, fma(c.kt * dt, dt, c.lnc_b)), tab, lane_off, Tb, Pb);
      if (SELF)
        fexp_tp<TS, I2F>(fma(c.ks, r2, fma(-c.omega, GEN ? fabs(dt) : dt, c.lnc_s)), tab, lane_off, Ts, Ps);
    }
    if (MASK) {
      Tb = dead ? 0.0 : Tb;
      Ts = dead ? 0.0 : Ts;
    }
    const double eb = Tb * Pb;
#endif
    double cc;
    if (GEN) {   // rho'_i mu' + rho'_j mu' + rho'_later xi'
      const double rlater = __double2hiint(dt) < 0 ? row.rho : crho;
      cc = SELF ? fma(row.rho + crho, eb, (rlater * Ts) * Ps) : (row.rho + crho) * eb;
    } else {
      cc = fma(row.rho, eb, crho * (SELF ? fma(Ts, Ps, eb) : eb));
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      rG[d] = fma(cc, dx[d], rG[d]);
      cG[d] = fma(-cc, dx[d], cG[d]);
    }
    return;
  }
#endif
  double eb = REB ? fexp<TS, I2F>(fma(c.kx, r2, fma(-dt, dt, c.lnc_b)), tab, lane_off)
                  : fexp<TS, I2F>(fma(c.kx, r2, fma(c.kt * dt, dt, c.lnc_b)), tab, lane_off);
#ifdef HK_SYM_FOLD
  // rho'_j xi' = beta xi_ji / lambda_j: the column's cL = lnc_s - 64 ln 2 - ln lambda_j
  double es = SELF ? fexp<TS, I2F>(fma(c.ks, r2, fma(-c.omega, dt, cL)), tab, lane_off) : 0.0;
#else   // xi' alone, weighted by rho' of the later event below
  double es = SELF ? (REB ? fexp<TS, I2F>(fma(c.ks, r2, fma(c.oms, dt, c.lnc_s)), tab, lane_off)
                          : fexp<TS, I2F>(fma(c.ks, r2, fma(-c.omega, GEN ? fabs(dt) : dt, c.lnc_s)), tab, lane_off))
                   : 0.0;
#endif
  if (MASK) {
    eb = dead ? 0.0 : eb;
    es = dead ? 0.0 : es;
  }
  // the pair's App. A coefficient, the same for both events
#ifdef HK_SYM_FOLD
  const double rs = row.rho + crho;
  const double cc = SELF ? fma(rs, eb, es) : rs * eb;
#else
  double cc;
  if (GEN) {   // rho'_i mu' + rho'_j mu' + rho'_later xi'
    const double rlater = __double2hiint(dt) < 0 ? row.rho : crho;
    cc = SELF ? fma(row.rho + crho, eb, rlater * es) : (row.rho + crho) * eb;
  } else {
    cc = fma(row.rho, eb, crho * (SELF ? eb + es : eb));
  }
#endif
#pragma unroll
  for (int d = 0; d < D; ++d) {
    rG[d] = fma(cc, dx[d], rG[d]);
    cG[d] = fma(-cc, dx[d], cG[d]);
  }
}

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// 32 skewed steps of one warp: its lanes' R rows x its 32-column group.
template <int D, int PASS, bool MASK, int SYM_R, bool SELF, int TS, bool SOA, bool GEN, bool PIECE,
          bool REB = false>
__device__ __forceinline__ void sym_group(const SymRow<D> (&row)[SYM_R],
                                          const double* __restrict__ grp,
                                          const double* __restrict__ lgrp, int cg0, bool cvalid0,
                                          int ridx0, int cidx0, bool diag, int s0, int s1,
                                          double (&rM)[SYM_R], double (&rX)[SYM_R], double (&rG)[SYM_R][D],
                                          double (&cacc)[2 + D], const PassConst& c,
                                          const int2* __restrict__ tab) {
  constexpr int REC = Layout<D>::REC;
  const int lane = threadIdx.x & 31;
  // PIECE: a step range [s0, s1) (whole items: the constant 0..32 loop).  Starting at s0,
  // lane l must hold column (l + s0)'s sums at the first step.
  if (!PIECE) s0 = 0, s1 = 32;
  if (PIECE && s0) rotate_cols<D, PASS>(cacc, (lane + s0) & 31);
  // unrolling by 2: pass 1 -2.8 %, pass 2 +1.4 % (N = 100k, accurate exp;
  // profiles/r02_ab_unroll.jsonl)
#ifdef HK_PASS2_UNR2   // A/B: pass 2 unrolled by 2 as well
  constexpr int UNR = 2;
#else
  constexpr int UNR = PASS == 1 ? 2 : 1;
#endif
#pragma unroll UNR
  for (int s = s0; s < s1; ++s) {
    const int src = (lane + s) & 31;
    // column (l + s) mod 32 of this warp's group: from the staged tile (AoS records), or
    // from the warp's transposed copy (SOA: component pair p of column e at [p][e])
    double cx[D];
    double ct, crho = 0.0, cL = 0.0;
    if (SOA) {   // pass 2: (x, t, rho', cL) of the column, cL in the pair after (x, t, rho')
      const double2* g2 = reinterpret_cast<const double2*>(grp);
      constexpr int NP = (PASS == 2 && SYM_FOLD) ? (D + 4) / 2 : (PASS == 2 ? (D + 3) / 2 : (D + 2) / 2);
      double v[2 * NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double2 w = g2[p * 32 + src];
        v[2 * p] = w.x;
        v[2 * p + 1] = w.y;
      }
#pragma unroll
      for (int d = 0; d < D; ++d) cx[d] = v[d];
      ct = v[D];
      if (PASS == 2) {
        crho = v[D + 1];
        if constexpr (SYM_FOLD) cL = v[D + 2];
      }
    } else {
      const double* rc = grp + src * REC;
#pragma unroll
      for (int d = 0; d < D; ++d) cx[d] = rc[d];
      ct = rc[D];
      if (PASS == 2) {
        crho = rc[D + 1];
        if constexpr (SYM_FOLD) cL = c.lnc_sr + lgrp[src];
      }
    }
    int cg = 0;
    bool cv = true;
    if (MASK) {
      cg = __shfl_sync(0xffffffffu, cg0, src);
      cv = __shfl_sync(0xffffffffu, (int)cvalid0, src) != 0;
      // a padding column of a ragged tile holds stale shared memory (any bit pattern, NaN
      // included): select its values to 0 so the masked terms below are exactly 0 (0 * NaN
      // would not be)
      if (!cv) {
#pragma unroll
        for (int d = 0; d < D; ++d) cx[d] = 0.0;
        ct = 0.0;
        crho = 0.0;
        cL = 0.0;
      }
    }
    double cG[D];
#pragma unroll
    for (int d = 0; d < D; ++d) cG[d] = cacc[2 + d];
#pragma unroll
    for (int r = 0; r < SYM_R; ++r) {
      // masked tiles: padding column or row, equal times, and (diagonal tiles) the
      // lower triangle j <= i, which the transposed tile pair covers
      const bool dead = MASK && (!cv || row[r].g < 0 || cg == row[r].g ||
                                 (diag && cidx0 + src <= ridx0 + 32 * r));
      if (PASS == 1)
        sym_pair1<D, MASK, SELF, TS, GEN, REB>(row[r], cx, ct, dead, rM[r], rX[r], cacc[0], cacc[1], c, tab);
      else
        sym_pair2<D, MASK, SELF, TS, GEN, REB>(row[r], cx, ct, crho, cL, dead, rG[r], cG, c, tab);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) cacc[2 + d] = cG[d];
    // rotate the column sums one lane down: lane l now holds column (l + s + 1) mod 32
    const int nxt = (lane + 1) & 31;
    if (PASS == 1) {
      cacc[0] = shfl(cacc[0], nxt);
      cacc[1] = shfl(cacc[1], nxt);
    }
    if (PASS == 2) {
#pragma unroll
      for (int d = 0; d < D; ++d) cacc[2 + d] = shfl(cacc[2 + d], nxt);
    }
  }
  // ... and ending at s1: lane l holds column (l + s1)'s; back to column l
  if (PIECE && s1 != 32) rotate_cols<D, PASS>(cacc, (lane - s1) & 31);
}

// Smallest squared distance and time gap between two boxes {lo[D], tlo} / {hi[D], thi} and a
// tile box b = {lo[D], hi[D], tmin, tmax}.
template <int D>
__device__ __forceinline__ void box_gaps(const double (&lo)[D + 1], const double (&hi)[D + 1],
                                         const double* __restrict__ b, double& r2min, double& dtmin) {
  r2min = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double g = fmax(0.0, fmax(b[d] - hi[d], lo[d] - b[D + d]));
    r2min = fma(g, g, r2min);
  }
  dtmin = fmax(0.0, fmax(b[2 * D] - hi[D], lo[D] - b[2 * D + 1]));
}

// Can any pair of the two boxes (space D + time) have a term above the exp's clamp?
template <int D>
__device__ __forceinline__ bool box_pair_live(const double (&lo_a)[D + 1], const double (&hi_a)[D + 1],
                                              const double (&lo_b)[D + 1], const double (&hi_b)[D + 1],
                                              const PassConst& c) {
  double r2min = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double g = fmax(0.0, fmax(lo_b[d] - hi_a[d], lo_a[d] - hi_b[d]));
    r2min = fma(g, g, r2min);
  }
  const double dtmin = fmax(0.0, fmax(lo_b[D] - hi_a[D], lo_a[D] - hi_b[D]));
  return fma(c.kx, r2min, fma(c.kt * dtmin, dtmin, c.lnc_b)) > CULL_EXPONENT ||
         fma(c.ks, r2min, c.lnc_s - c.omega * dtmin) > CULL_EXPONENT;
}

// Tile walk of one item: row tiles rt = 0..n_rt-1, column tiles ct = (diag ? rt : 0)..n_ct-1
// (a diagonal item (a, a) visits only the upper triangle of its tile pairs).
struct TileWalk {
  int rt, ct;
  __device__ __forceinline__ void next(int n_ct, bool diag) {
    if (++ct == n_ct) {
      ++rt;
      ct = diag ? rt : 0;
    }
  }
};

// Shared-memory layout of the pass kernels: the column-tile stages (records, and the staged
// -ln lambda of -DHK_SYM_FOLD), the stage barriers, the exp table (TS interleaved copies),
// the 4 warps' row-sum buffers (KR per row) and the per-warp SoA column copies (SOAW doubles
// per column).
template <int D, int TS, int KR, int SOAW, int LST>
struct SymSmem {
  static constexpr int REC = Layout<D>::REC;
  static constexpr size_t bytes() {
    return (size_t)STAGES * TILE_J * REC * sizeof(double) + (size_t)STAGES * LST * sizeof(double) +
           STAGES * sizeof(uint64_t) + (size_t)EXP_TABLE * TS * sizeof(int2) +
           (size_t)4 * TILE_J * KR * sizeof(double) + (size_t)4 * 32 * SOAW * sizeof(double);
  }
  double* stage;
  double* lstage;
  uint64_t* bars;
  int2* tab;
  double* red;
  double* soa;
  __device__ __forceinline__ explicit SymSmem(unsigned char* raw) {
    stage = reinterpret_cast<double*>(raw);
    lstage = stage + STAGES * TILE_J * REC;
    bars = reinterpret_cast<uint64_t*>(lstage + STAGES * LST);
    tab = reinterpret_cast<int2*>(bars + STAGES);
    red = reinterpret_cast<double*>(tab + EXP_TABLE * TS);
    soa = red + 4 * TILE_J * KR;
  }
};

template <int D, int PASS, int V, bool GEN = false>
struct SymCfg {
  static constexpr bool FOLD = PASS == 2 && SYM_FOLD;
  static constexpr int TS = (V & 2) ? TAB_COPIES : 1;
  // row sums reduced over warps: M (time order: a row is never the later event of its pairs),
  // M and X (GEN), or G
  static constexpr int KR = PASS == 1 ? (GEN ? 2 : 1) : D;
  static constexpr int LST = FOLD ? TILE_J : 0;          // -ln lambda of the staged columns
  static constexpr int SOAW = FOLD ? 2 * ((D + 4) / 2) : Layout<D>::REC;   // doubles per column
  using Smem = SymSmem<D, TS, KR, (V & 4) ? SOAW : 0, LST>;
};

// kernel prologue: the exp table into shared memory (TS copies), the stage barriers
template <int TS>
__device__ __forceinline__ void sym_prologue(const int2* __restrict__ gtab, int2* tab, uint64_t* bars) {
  const int tid = threadIdx.x;
  // all of a thread's table loads in flight at once, then the stores (a load-store loop pays
  // one L2 round trip per entry: 7 % of the gradient pass's samples at N = 5000)
  static_assert(EXP_TABLE * TS % THREADS == 0, "whole table rows per thread");
  constexpr int PER = EXP_TABLE * TS / THREADS;
  int2 v[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) v[k] = __ldg(gtab + (tid + k * THREADS) / TS);
#pragma unroll
  for (int k = 0; k < PER; ++k) tab[tid + k * THREADS] = v[k];
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
}

// One pass over the work items of a.counter (chunk pairs), pulled until exhausted; the
// shared-memory pointers come from the caller's layout, parity carries the stage barriers'
// phases across calls (every issued stage is consumed before this returns).
// GEN: spatial order (hawkes_plan.h morton_order): no time order between or inside chunks,
// so the general-direction pair bodies; tile pairs and whole items are culled by the
// bounding boxes of their tiles (a.boxes) in space and time.
template <int D, int PASS, int SYM_R, int V, bool GEN, bool PIECE, class Sm>
__device__ __forceinline__ void sym_items(const SymArgs& a, const Sm& sm, int* s_item_p,
                                          uint32_t& parity) {
  static_assert(32 * SYM_R == TILE_J, "row tiles and column tiles must coincide");
  constexpr int SYM_RT = 32 * SYM_R;
  using L = Layout<D>;
  constexpr int REC = L::REC;
  constexpr int K = PASS == 1 ? K1P : L::K2;
  using Cfg = SymCfg<D, PASS, V, GEN>;
  constexpr int KR = Cfg::KR;
  constexpr bool SOA = (V & 4) != 0;
  constexpr int TS = Cfg::TS;
  constexpr bool FOLD = Cfg::FOLD;
  constexpr int LST = Cfg::LST;
  constexpr int SOAW = Cfg::SOAW;
  double* stage = sm.stage;
  double* lstage = sm.lstage;
  uint64_t* bars = sm.bars;
  double* red = sm.red;
  int& s_item = *s_item_p;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int2* mytab = sm.tab;   // REPL: fexp or-s the lane's copy into the index
  double* mysoa = sm.soa + warp * 32 * SOAW;
  // stage s <- column tile [jt, jt + cnt): the records, and (pass 2) -ln lambda rounded up to
  // an even count (16-byte bulk copies; lrho has npad >= N + 1 entries or N even)
  auto load_stage = [&](int s, int jt, int cnt) {
    HK_CHECK(s >= 0 && s < STAGES && cnt >= 1 && cnt <= TILE_J && jt >= 0 && jt + cnt <= a.npad &&
             jt % TILE_J == 0);
    if (FOLD)
      tma_load_1d_x2(stage + s * TILE_J * REC, a.rec + (long long)jt * REC,
                     (uint32_t)(cnt * REC * sizeof(double)), lstage + s * LST, a.lrho + jt,
                     (uint32_t)(((cnt + 1) & ~1) * sizeof(double)), &bars[s]);
    else
      tma_load_1d(stage + s * TILE_J * REC, a.rec + (long long)jt * REC,
                  (uint32_t)(cnt * REC * sizeof(double)), &bars[s]);
  };
  const PassConst c = a.c;
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
    HK_CHECK(w.a >= 0 && w.a <= w.b && w.b < a.nchunks && w.ro >= 0 && w.co >= 0 && 0 <= w.s0 &&
             w.s0 < w.s1 && w.s1 <= 32);
    const bool diag = w.a == w.b;
    const int r0 = w.a * a.chunk;                 // chunk a: rows
    const int r1 = min(N, r0 + a.chunk);
    const int c0 = w.b * a.chunk;                 // chunk b: columns
    const int c1 = min(N, c0 + a.chunk);
    const int n_rt = (r1 - r0 + SYM_RT - 1) / SYM_RT;
    const int n_ct = (c1 - c0 + TILE_J - 1) / TILE_J;
    if (GEN && !diag) {
      // item-level cull: the union boxes of the two chunks; a dead item still owns its
      // slots (row role: slot b of chunk a's events; column role: slot a of chunk b's)
      const double* bx = a.boxes;
      double lo_a[D + 1], hi_a[D + 1], lo_b[D + 1], hi_b[D + 1];
#pragma unroll
      for (int d = 0; d <= D; ++d) {
        lo_a[d] = lo_b[d] = INFINITY;
        hi_a[d] = hi_b[d] = -INFINITY;
      }
      for (int q = 0; q < n_rt; ++q) {
        const double* b = bx + (long long)(r0 / TILE_J + q) * (2 * D + 2);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          lo_a[d] = fmin(lo_a[d], b[d]);
          hi_a[d] = fmax(hi_a[d], b[D + d]);
        }
        lo_a[D] = fmin(lo_a[D], b[2 * D]);
        hi_a[D] = fmax(hi_a[D], b[2 * D + 1]);
      }
      for (int q = 0; q < n_ct; ++q) {
        const double* b = bx + (long long)(c0 / TILE_J + q) * (2 * D + 2);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          lo_b[d] = fmin(lo_b[d], b[d]);
          hi_b[d] = fmax(hi_b[d], b[D + d]);
        }
        lo_b[D] = fmin(lo_b[D], b[2 * D]);
        hi_b[D] = fmax(hi_b[D], b[2 * D + 1]);
      }
      if (!box_pair_live<D>(lo_a, hi_a, lo_b, hi_b, c)) {
        for (int q = tid; q < (r1 - r0) * K; q += THREADS) a.part[w.ro * K + q] = 0.0;
        for (int q = tid; q < (c1 - c0) * K; q += THREADS) a.part[w.co * K + q] = 0.0;
        continue;
      }
    }

    TileWalk prod{0, 0};
    if (tid == 0) {
      for (int s = 0; s < STAGES && prod.rt < n_rt; ++s, prod.next(n_ct, diag)) {
        const int jt = c0 + prod.ct * TILE_J;
        load_stage(s, jt, min(TILE_J, c1 - jt));
      }
    }

    int k = 0;
    for (int rt = 0; rt < n_rt; ++rt) {
      const int row0 = r0 + rt * SYM_RT;
      const bool rows_full = row0 + SYM_RT <= r1;
      SymRow<D> row[SYM_R];
      double rM[SYM_R], rX[SYM_R], rG[SYM_R][D];
#pragma unroll
      for (int r = 0; r < SYM_R; ++r) {
        const int i = row0 + lane + 32 * r;
        const double* ri = a.rec + (long long)min(i, N - 1) * REC;
#pragma unroll
        for (int d = 0; d < D; ++d) row[r].x[d] = ri[d];
        row[r].t = ri[D];
        row[r].rho = ri[D + 1];
        row[r].g = i < N ? a.gid[i] : -1;   // -1: padding row (masked)
        rM[r] = 0.0;
        rX[r] = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) rG[r][d] = 0.0;
      }
      // GEN: this row tile's box (tiles are TILE_J-aligned in the walk's order)
      double rlo[D + 1], rhi[D + 1];
      if (GEN) {
        const double* b = a.boxes + (long long)(row0 / TILE_J) * (2 * D + 2);
#pragma unroll
        for (int d = 0; d < D; ++d) {
          rlo[d] = b[d];
          rhi[d] = b[D + d];
        }
        rlo[D] = b[2 * D];
        rhi[D] = b[2 * D + 1];
      }
      const int rlast = min(row0 + SYM_RT, r1) - 1;
      const int g_rlast = a.gid[rlast];
      const double t_rlast = a.rec[(long long)rlast * REC + D];

      for (int ct = diag ? rt : 0; ct < n_ct; ++ct, ++k) {
        const int s = k % STAGES;
        const int jt = c0 + ct * TILE_J;
        const int cnt = min(TILE_J, c1 - jt);
        mbar_wait(&bars[s], (parity >> s) & 1u);
        parity ^= (1u << s);
        const double* st = stage + s * TILE_J * REC;
        // this lane's column in its warp's group (padding columns of a ragged tile read
        // stale stage data and are masked out)
        const int cl = warp * 32 + lane;
        const bool cvalid = cl < cnt;
        const int cj = jt + min(cl, cnt - 1);
        const int cg = a.gid[cj];
        // column sums: accumulated over this item's row tiles in its own slot
        HK_CHECK(cj >= c0 && cj < c1);
        double* cpart = a.part + (w.co + (cj - c0)) * K;
        const bool first = rt == 0;   // every column tile is first visited by row tile 0
        double cacc[2 + D];
        if (first || !cvalid) {
#pragma unroll
          for (int q = 0; q < 2 + D; ++q) cacc[q] = 0.0;
        } else if (PASS == 1) {
          cacc[0] = cpart[0];
          cacc[1] = cpart[1];
        } else {
          cacc[0] = cacc[1] = 0.0;
#pragma unroll
          for (int d = 0; d < D; ++d) cacc[2 + d] = cpart[d];
        }
        const bool diag_tile = diag && ct == rt;
        const bool strict = !diag_tile && rows_full && cnt == TILE_J &&
                            (GEN ? !a.ties : g_rlast < a.gid[jt]);
        // temporal culling (NEXT-2 on time-compact tiles): with dt >= dtmin for every pair
        // of this tile pair, the self-excitation exponent is <= lnc_s - omega dtmin and the
        // background one <= lnc_b + k_t dtmin^2; below the exp's clamp they add nothing.
        // GEN: the same bounds from the two tiles' boxes, with r^2 >= r2min as well.
        double dtmin, r2min = 0.0;
        if (GEN) {
          const double* b = a.boxes + (long long)(jt / TILE_J) * (2 * D + 2);
          box_gaps<D>(rlo, rhi, b, r2min, dtmin);
        } else {
          dtmin = fmax(st[D] - t_rlast, 0.0);
        }
        const double* grp = st + warp * 32 * REC;
        const double* lgrp = lstage + s * LST + warp * 32;
        // pass 2's self-excitation exponent carries the column's cL = lnc_s - 64 ln2 - ln
        // lambda_j: its bound takes the largest cL of this warp's 32 columns
        double self_bound = c.lnc_s;
        if (FOLD) {
          double cLmax = cvalid ? c.lnc_sr + lgrp[lane] : -INFINITY;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) cLmax = fmax(cLmax, __shfl_xor_sync(0xffffffffu, cLmax, o));
          self_bound = cLmax;
        }
        const bool self_live = fma(c.ks, r2min, self_bound - c.omega * dtmin) > CULL_EXPONENT;
        const bool bg_live = fma(c.kx, r2min, fma(c.kt * dtmin, dtmin, c.lnc_b)) > CULL_EXPONENT;
        // REB (rate pass, time walk, strict tile pairs): times rebased to T0 = the column tile's
        // first time and scaled by st, u = st (t - T0), where the tile's span keeps the rounding
        // of u within the fp64 exponents' error class: omega span <= 256, |k_t| span^2 <= 64
        // (rows precede T0 here, so |u_i| <= st dt and |u_j| <= st span)
        bool reb = false;
        if constexpr (!GEN && SOA && !FOLD && (PASS == 1 ? REB1 : REB2)) {
          if (strict) {
            const double span = st[(cnt - 1) * REC + D] - st[D];
            reb = c.omega * span <= 256.0 && -c.kt * span * span <= 64.0;
          }
          if (reb) {
#pragma unroll
            for (int r = 0; r < SYM_R; ++r) row[r].u = c.st * (row[r].t - st[D]);
          }
        }
        if (SOA) {   // this lane's column record (+ cL) -> the warp's [pair][32] double2 buffer
          const double* rc = grp + lane * REC;
          double2* g2 = reinterpret_cast<double2*>(mysoa);
          double v[SOAW];
#pragma unroll
          for (int q = 0; q < REC; ++q) v[q] = rc[q];
          if (reb) v[D] = c.st * (v[D] - st[D]);
          if constexpr (FOLD) v[D + 2] = c.lnc_sr + lgrp[lane];
#pragma unroll
          for (int q = (FOLD ? D + 3 : REC); q < SOAW; ++q) v[q] = 0.0;
#pragma unroll
          for (int p = 0; p < SOAW / 2; ++p) g2[p * 32 + lane] = make_double2(v[2 * p], v[2 * p + 1]);
          __syncwarp();
          grp = mysoa;
        }
        // PIECE (a plan of pieces, hawkes_plan.h): the item's step range; whole items run the
        // constant 32-step loop (a kernel instantiation of its own: carrying both in one
        // kernel made the gradient pass 5 % slower at N = 100k)
        if (!strict)
          sym_group<D, PASS, true, SYM_R, true, TS, SOA, GEN, PIECE>(row, grp, lgrp, cg, cvalid, row0 + lane,
                                                                     jt + warp * 32, diag_tile, w.s0, w.s1,
                                                                     rM, rX, rG, cacc, c, mytab);
        else if (self_live) {
          if (reb)
            sym_group<D, PASS, false, SYM_R, true, TS, SOA, GEN, PIECE, true>(row, grp, lgrp, cg, cvalid,
                                                                              row0 + lane, jt + warp * 32, false,
                                                                              w.s0, w.s1, rM, rX, rG, cacc, c, mytab);
          else
            sym_group<D, PASS, false, SYM_R, true, TS, SOA, GEN, PIECE>(row, grp, lgrp, cg, cvalid, row0 + lane,
                                                                        jt + warp * 32, false, w.s0, w.s1, rM,
                                                                        rX, rG, cacc, c, mytab);
        } else if (bg_live) {
          if (reb)
            sym_group<D, PASS, false, SYM_R, false, TS, SOA, GEN, PIECE, true>(row, grp, lgrp, cg, cvalid,
                                                                               row0 + lane, jt + warp * 32, false,
                                                                               w.s0, w.s1, rM, rX, rG, cacc, c, mytab);
          else
            sym_group<D, PASS, false, SYM_R, false, TS, SOA, GEN, PIECE>(row, grp, lgrp, cg, cvalid,
                                                                         row0 + lane, jt + warp * 32, false,
                                                                         w.s0, w.s1, rM, rX, rG, cacc, c, mytab);
        }
        // else: nothing survives; lane l still holds column l's sums (no rotation needed)
        if (cvalid) {
          if (PASS == 1) {
            cpart[0] = cacc[0];
            cpart[1] = cacc[1];
          } else {
#pragma unroll
            for (int d = 0; d < D; ++d) cpart[d] = cacc[2 + d];
          }
        }
        __syncthreads();   // stage s fully consumed
        if (tid == 0 && prod.rt < n_rt) {
          const int jn = c0 + prod.ct * TILE_J;
          load_stage(s, jn, min(TILE_J, c1 - jn));
          prod.next(n_ct, diag);
        }
      }
      // row sums of this row tile: reduce the 4 warps' partials in a fixed order
#pragma unroll
      for (int r = 0; r < SYM_R; ++r) {
        double* o = red + ((long long)warp * SYM_RT + lane + 32 * r) * KR;
        if (PASS == 1) {
          o[0] = rM[r];
          if (GEN) o[1] = rX[r];
        } else {
#pragma unroll
          for (int d = 0; d < D; ++d) o[d] = rG[r][d];
        }
      }
      __syncthreads();
      for (int q = tid; q < SYM_RT * KR; q += THREADS) {
        const int rr = q / KR, kk = q % KR;
        if (row0 + rr >= N) continue;
        double v = red[(0 * SYM_RT + rr) * KR + kk];
        v += red[(1 * SYM_RT + rr) * KR + kk];
        v += red[(2 * SYM_RT + rr) * KR + kk];
        v += red[(3 * SYM_RT + rr) * KR + kk];
        HK_CHECK(row0 + rr < a.N && kk < K);
        double* o = a.part + (w.ro + (row0 + rr - r0)) * K;   // row block (slot b)
        if (PASS == 1 && !GEN) {
          o[0] = v;      // M
          o[1] = 0.0;    // X: xi_ij = 0 for a later j
        } else {
          o[kk] = v;     // (GEN pass 1: M and X)
        }
      }
      __syncthreads();
    }
  }
}

// CTAs per SM: 4 (<= 128 registers) for the D <= 2 time-walk gradient pass, 3 (<= 168) for
// the other D <= 4 kernels, 2 above.  At N = 100k the gradient pass at 128 registers has no
// spills and runs 1.5 % faster (more warps hide its dependency latency), the rate pass 1.2 %
// slower (profiles/r02_ab_occ4.jsonl) and the spatial-walk gradient pass 2 % slower (DC shape);
// -DHK_SYM_OCC4 asks for 4 everywhere (A/B).
template <int D, int PASS, bool GEN>
constexpr int sym_min_ctas() {
#if defined(HK_SYM_OCC4)
  return D <= 4 ? 4 : 2;
#elif defined(HK_SYM_GRAD_OCC3)   // A/B: the D <= 2 gradient pass at 3 CTAs/SM as well
  return D <= 4 ? 3 : 2;
#else
  return (D <= 2 && PASS == 2 && !GEN) ? 4 : (D <= 4 ? 3 : 2);
#endif
}
template <int D, int PASS, int SYM_R, int V, bool GEN = false, bool PIECE = false>
__global__ void __launch_bounds__(THREADS, sym_min_ctas<D, PASS, GEN>()) sym_kernel(SymArgs a) {
  using Cfg = SymCfg<D, PASS, V, GEN>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const typename Cfg::Smem sm(smem_raw);
  __shared__ int s_item;
  sym_prologue<Cfg::TS>(a.tab, sm.tab, sm.bars);   // the table is written at creation
  pdl_wait();
  uint32_t parity = 0;
  sym_items<D, PASS, SYM_R, V, GEN, PIECE>(a, sm, &s_item, parity);
  // the dependent grid launches once every CTA is out of items: triggering at the start lets
  // its CTAs take SM slots while this grid still runs, which at small N (grid < 148) packs
  // the next pass's CTAs onto busy SMs (N = 2000: +11 us per call)
  pdl_trigger();
}

}  // namespace hk
