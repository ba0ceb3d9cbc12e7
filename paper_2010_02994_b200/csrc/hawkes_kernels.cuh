// hawkes_kernels.cuh -- sm_100a kernels for the O(N^2) Hawkes rate and gradient passes.
//
// Math (PAPER.md, see include/hawkes.h for the full statement):
//   mu_ij = mu0/(tau_x^D tau_t) phi_D(dx/tau_x) phi(dt/tau_t) I[t_i != t_j]
//   xi_ij = theta omega/h^D e^{-omega dt} phi_D(dx/h) I[t_j < t_i]
//   lambda_i = sum_j mu_ij + xi_ij
//   g_i = sum_j [(mu_ij rho_i + mu_ji rho_j)/tau_x^2 + (xi_ij rho_i + xi_ji rho_j)/h^2] (x_j - x_i)
//                                                                            (App. A)
// with rho = 1/lambda.  Because mu is symmetric, g_i splits into a part that needs only
// row-i data (accumulated in the rate pass) and a part weighted by rho_j (gradient pass):
//   g_i = rho_i * G1_i + G2_i
//   G1_i = sum_j (mu_ij/tau_x^2 + xi_ij/h^2) dx_ij                  [pass 1, with lambda]
//   G2_i = sum_j rho_j (mu_ij/tau_x^2 + xi_ji/h^2) dx_ij            [pass 2]
// so each pass evaluates the background exp for every pair and the self-excitation exp
// only for the half of the pairs where the relevant indicator can be non-zero.
//
// Scaled domain: every pair exponent carries log(alpha*w*2^64) (alpha = 1/tau_x^2 or
// 1/h^2, w the kernel weight), so the exp returns alpha*mu_ij*2^64 (resp. beta*xi_ij*2^64)
// directly; sums stay scaled, rho' = 2^-64/lambda, and g_i = rho'_i G1'_i + G2'_i exactly
// as above.
//
// Layout: each event is one record of REC doubles {x_0..x_{D-1}, t, rho', pad} (32 B for
// D <= 2); a CTA owns RT = THREADS*R rows (thread k: rows row0 + k + r*THREADS), and
// streams j-tiles of TILE_J records through shared memory with 1-D TMA bulk copies
// (cp.async.bulk + mbarrier, STAGES deep).  Every lane reads the same record (broadcast).
// Work items (row tile, j chunk) are pulled from a global counter by a persistent grid;
// each item writes its own partial sums, reduced later in a fixed order (deterministic,
// independent of the number of ranks).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hk {

// -DHK_CHECKED (tools/checked_run.sh): device-side bounds checks on the pass kernels' item
// decode, bulk-copy ranges, partial-slot stores and walk permutation -- compute-sanitizer is
// closed on the GPU pool, so the checked build runs the GPU test-suite instead.  A failed check
// prints its site and traps (the launch then fails with an error).
#ifdef HK_CHECKED
#define HK_CHECK(cond)                                                                    \
  do {                                                                                    \
    if (!(cond)) {                                                                        \
      printf("HK_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__,      \
             __LINE__, (int)blockIdx.x, (int)threadIdx.x);                                \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define HK_CHECK(cond) \
  do {                 \
  } while (0)
#endif

constexpr int THREADS = 128;
constexpr int TILE_J = 128;
constexpr int STAGES = 4;

template <int D>
struct Layout {
  static constexpr int REC = ((D + 3) / 2) * 2;   // doubles per event record (even)
  static constexpr int T = D;                     // offset of t
  static constexpr int RHO = D + 1;               // offset of rho'
  static constexpr int K1 = ((D + 3) / 2) * 2;    // pass-1 partial: M', X', G1'[D] (padded)
  static constexpr int K2 = ((D + 1) / 2) * 2;    // pass-2 partial: G2'[D] (padded)
};

struct PassConst {
  double kx, kt, ks;   // -1/(2 tau_x^2), -1/(2 tau_t^2), -1/(2 h^2)
  double omega;
  double lnc_b;        // log(mu0/((2pi)^{(D+1)/2} tau_x^D tau_t) / tau_x^2 * 2^64)
  double lnc_s;        // log(theta omega/((2pi)^{D/2} h^D) / h^2 * 2^64)
  double lnc_sr;       // lnc_s - 64 ln 2: the unordered-pair gradient pass folds -ln lambda_j
                       // into the self-excitation exponent (hawkes_kernels_sym.cuh)
  double st;           // sqrt(-kt) = 1/(sqrt2 tau_t): rebased times u = st (t - T0) (rate pass)
  double oms;          // -omega / st: -omega dt = oms du
};

// ---------------------------------------------------------------- table fp64 exp
// e^a for the pair kernels.  On sm_100 an FP64 instruction holds its SM sub-partition's
// dispatch for two cycles and every other instruction for one (measured: the FP64 pipe
// utilisation of a kernel tracks 2*n_fp64 / (2*n_fp64 + n_other)), so this exp is
// built to minimise both: 7 FP64 instructions and 5 integer/shared-memory ones.
//   a' = max(a, AMIN)            one unsigned min on the high word (AMIN = -707: for
//                                negative doubles a larger high word means a larger |a|;
//                                positive a, high bit clear, pass through)
//   y  = a' * 1024/ln2 + 1.5*2^52 rounds to an integer: y's low word is
//                                k = rint(a' * 1024/ln2) = 1024m + j
//   r  = a' - k ln2/1024         |r| <= ln2/2048
//   T  = 2^(j/1024) from a 1024-entry (8 KB) shared table whose high words are
//        pre-biased by -(j << 10), so that one integer multiply-add, hi + (k << 10), also
//        adds m to the exponent field
//   e^a = T 2^m (1 + p(r)),  p(r) = r (1 + r (c2 + c3 r))  (minimax, tools/fit_exp_poly.py
//        1024 3: |rel. err.| <= 9.4e-17 on |r| <= ln2/2048, so the result is within a few
//        ulp of e^a': u-accurate, like the oracle's libm exp -- SURVEY.md §7 asks for
//        <~1e-15 because gradient components cancel).  1024 entries measured 0.4 % faster
//        in the gradient pass than 2048 (-DHK_EXP2048; profiles/r02_ab_table.jsonl)
// Round 1 shipped degree 2 (6 FP64, 8.1e-13; -DHK_EXP_FAST keeps it for A/B): its error
// is systematic per table cell, so a gradient component's error reached ~7000 u S_nd and
// the plain relative error exceeded 1e-9 from kappa ~ 8e3 (profiles/r02_plain_error_r01kernel.jsonl),
// where a u-accurate sum stays below it up to kappa ~ 1e6.
// Arguments below AMIN return e^(a') ~ e^-707 instead of a smaller number (callers treat
// sums below N e^-700 as zero; reading R23).  Arguments must be < ~700
// (guaranteed by the validated kernel constants).
#if defined(HK_EXP256)   // the 256-entry, degree-3 exp (tools/fit_exp_poly.py 256 3: 2.4e-14)
constexpr double EXP_K = 369.3299304675746;                // 256/ln2
constexpr double EXP_C = 0.0027076061740622863;            // ln2/256
constexpr double EXP_C2 = 0.5000000632802307;
constexpr double EXP_C3 = 0.1666666688540192;
constexpr int EXP_TABLE = 256;
constexpr int EXP_BIAS_SHIFT = 12;                          // 20 - log2(EXP_TABLE)
constexpr int EXP_DEGREE = 3;
#elif defined(HK_EXP2048) || defined(HK_EXP_FAST)   // 2048 entries (16 KB)
constexpr double EXP_K = 2954.639443740597;                 // 2048/ln2
constexpr double EXP_C = 3.3845077175778579e-04;            // ln2/2048
constexpr int EXP_TABLE = 2048;
constexpr int EXP_BIAS_SHIFT = 9;                           // 20 - log2(EXP_TABLE)
#if defined(HK_EXP_FAST)  // round 1: degree 2, 8.1e-13
constexpr double EXP_C2 = 0.499999996420339;
constexpr double EXP_C3 = 0.0;                              // unused
constexpr int EXP_DEGREE = 2;
#else                     // degree 3, 5.9e-18
constexpr double EXP_C2 = 0.5000000009888816;               // 0x1.000000087e92ep-1
constexpr double EXP_C3 = 0.16666666670097202;              // 0x1.5555555683162p-3
constexpr int EXP_DEGREE = 3;
#endif
#else   // default: 1024 entries (8 KB), degree 3 (tools/fit_exp_poly.py 1024 3: 9.4e-17)
constexpr double EXP_K = 1477.3197218702985;                // 1024/ln2
constexpr double EXP_C = 6.7690154351557158e-04;            // ln2/1024
constexpr int EXP_TABLE = 1024;
constexpr int EXP_BIAS_SHIFT = 10;                          // 20 - log2(EXP_TABLE)
constexpr double EXP_C2 = 0.5000000039557457;               // 0x1.00000021fac6ep-1
constexpr double EXP_C3 = 0.16666666680410733;              // 0x1.5555555a0e463p-3
constexpr int EXP_DEGREE = 3;
#endif
constexpr double EXP_SHIFT = 6755399441055744.0;            // 1.5 * 2^52
constexpr unsigned EXP_AMIN_HI = 0xC0861800u;               // high word of -707.0

#ifdef HK_ABLATE_TABMASK
__constant__ int g_ablate_tabmask = 0;
#endif

// STRIDE > 1: the table is stored interleaved in STRIDE copies (entry j of copy c at
// j*STRIDE + c) and tab points at this thread's copy (see sym_kernel)
template <int STRIDE = 1, bool KF_I2F = false>
__device__ __forceinline__ double fexp(double a, const int2* __restrict__ tab, int lane_off = 0) {
  static_assert(STRIDE == 1 || STRIDE == 2 || STRIDE == 4 || STRIDE == 16, "interleaved copies");
  const unsigned ahi = min((unsigned)__double2hiint(a), EXP_AMIN_HI);
  const double ac = __hiloint2double((int)ahi, __double2loint(a));
  const double y = fma(ac, EXP_K, EXP_SHIFT);
  const int k = __double2loint(y);
  // k as a double: y - shift (FP64 pipe) or I2F.F64 (a quarter-rate conversion pipe beside
  // it), both exact, so both forms give the same bits.  The conversion pays where the FP64
  // pipe is the tighter limit: sym_kernel's gradient pass for D <= 5 (-1.4 % at D = 2,
  // N = 100k; -0.5 to -2.8 % for D = 2..5), while pass 1 (+2.6 %) and the 255-register
  // D >= 6 gradient passes (+0.4 to +2 %) lose more to its latency (profiles/r01_sym_variants.txt)
  const double kf = KF_I2F ? __int2double_rn(k) : y - EXP_SHIFT;
  const double r = fma(kf, -EXP_C, ac);
  int2 T;
  if constexpr (STRIDE == 1) {
#ifdef HK_ABLATE_TABMASK   // diagnostics only (wrong results): every lane reads one entry,
    T = tab[k & g_ablate_tabmask];   // a broadcast -- the kernel timed without bank conflicts
#else
    T = tab[k & (EXP_TABLE - 1)];
#endif
  } else {
    // interleaved copies: byte offset ((k mod 256) * STRIDE + copy) * 8, the copy's part
    // (lane_off, 0..STRIDE-1 times 8) or-ed in: one shift + one LOP3, uniform table base
    constexpr int SH = 3 + (STRIDE == 2 ? 1 : STRIDE == 4 ? 2 : 4);   // log2(8 * STRIDE)
    T = *reinterpret_cast<const int2*>(reinterpret_cast<const char*>(tab) +
                                       (((k << SH) & ((EXP_TABLE - 1) << SH)) | lane_off));
  }
  const double q = EXP_DEGREE == 2 ? fma(EXP_C2, r, 1.0) : fma(fma(EXP_C3, r, EXP_C2), r, 1.0);
  const double p = q * r;                                      // e^r - 1
  const double Tm = __hiloint2double(T.y + k * (1 << EXP_BIAS_SHIFT), T.x);   // 2^(j/256) 2^m
  return fma(Tm, p, Tm);
}

// The same exp as a product e^a = Tm * P, P = 1 + r (1 + r (c2 + c3 r)) = e^r (one rounding
// more than fexp's Tm + Tm (e^r - 1): still within ~1 ulp), for callers that only accumulate
// e^a: each sum += e^a becomes one fma(Tm, P, sum), so the exp's final multiply disappears
// into the accumulations (the unordered-pair kernels: one FP64 instruction less per term in
// pass 1, one per pair in pass 2).  A caller masks a term by zeroing Tm (P is
// finite for every finite a).
template <int STRIDE = 1, bool KF_I2F = false>
__device__ __forceinline__ void fexp_tp(double a, const int2* __restrict__ tab, int lane_off,
                                        double& Tm, double& P) {
  static_assert(STRIDE == 1 || STRIDE == 2 || STRIDE == 4 || STRIDE == 16, "interleaved copies");
  static_assert(EXP_DEGREE == 3, "the product form follows the degree-3 polynomial");
  const unsigned ahi = min((unsigned)__double2hiint(a), EXP_AMIN_HI);
  const double ac = __hiloint2double((int)ahi, __double2loint(a));
  const double y = fma(ac, EXP_K, EXP_SHIFT);
  const int k = __double2loint(y);
  const double kf = KF_I2F ? __int2double_rn(k) : y - EXP_SHIFT;
  const double r = fma(kf, -EXP_C, ac);
  int2 T;
  if constexpr (STRIDE == 1) {
#ifdef HK_ABLATE_TABMASK
    T = tab[k & g_ablate_tabmask];
#else
    T = tab[k & (EXP_TABLE - 1)];
#endif
  } else {
    constexpr int SH = 3 + (STRIDE == 2 ? 1 : STRIDE == 4 ? 2 : 4);
    T = *reinterpret_cast<const int2*>(reinterpret_cast<const char*>(tab) +
                                       (((k << SH) & ((EXP_TABLE - 1) << SH)) | lane_off));
  }
  P = fma(fma(fma(EXP_C3, r, EXP_C2), r, 1.0), r, 1.0);
  Tm = __hiloint2double(T.y + k * (1 << EXP_BIAS_SHIFT), T.x);
}

// --------------------------------------------------------------- programmatic dependent launch
// The evaluation's kernels after the first (PAIRS: pass 1 -> finalize 1 -> pass 2 -> finalize
// 2) are launched with programmatic stream serialization (hawkes_launch.cuh launch_pdl): each
// lets its dependent grid launch at its start (pdl_trigger), and the dependent runs whatever
// reads no earlier kernel's output (exp-table copy into shared memory, barrier init) before
// pdl_wait, which returns once every prerequisite grid has completed and its memory is
// visible.  Both are no-ops in a kernel launched without the attribute.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// --------------------------------------------------------------- TMA / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// two bulk copies completing on one barrier (one arrive with the summed byte count)
__device__ __forceinline__ void tma_load_1d_x2(void* dst0, const void* src0, uint32_t bytes0, void* dst1,
                                               const void* src1, uint32_t bytes1, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes0 + bytes1)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst0)),
      "l"(src0), "r"(bytes0), "r"(smem_u32(bar))
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst1)),
      "l"(src1), "r"(bytes1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------- pair bodies
enum { KIND_EARLIER = 0, KIND_LATER = 1, KIND_MIXED = 2 };

template <int D>
struct RowState {
  double x[D];
  double t;
  int g;
};

// Pass 1 (rate pass + row-local gradient part) for one (i, j) pair.
//  KIND_EARLIER: every j in the tile is strictly earlier than every row -> mu and xi.
//  KIND_LATER:   every j strictly later -> mu only (xi_ij = 0).
//  KIND_MIXED:   per-pair indicators from the tie-group ids g (g_j == g_i <=> t_j == t_i,
//                g_j < g_i <=> t_j < t_i).
template <int D, int KIND>
__device__ __forceinline__ void pair_pass1(const double* __restrict__ rj, int gj,
                                           const RowState<D>& row, double& M, double& X,
                                           double (&G)[D], const PassConst& c,
                                           const int2* __restrict__ tab) {
  double dx[D];
  double r2;
#pragma unroll
  for (int d = 0; d < D; ++d) dx[d] = rj[d] - row.x[d];
  r2 = dx[0] * dx[0];
#pragma unroll
  for (int d = 1; d < D; ++d) r2 = fma(dx[d], dx[d], r2);
  const double dt = row.t - rj[D];
  const double ab = fma(c.kx, r2, fma(c.kt * dt, dt, c.lnc_b));
  double eb = fexp(ab, tab);
  if (KIND == KIND_MIXED) eb = (gj == row.g) ? 0.0 : eb;
  if (KIND == KIND_LATER) {
    M += eb;
#pragma unroll
    for (int d = 0; d < D; ++d) G[d] = fma(eb, dx[d], G[d]);
  } else {
    const double as = fma(c.ks, r2, fma(-c.omega, dt, c.lnc_s));
    double es = fexp(as, tab);
    if (KIND == KIND_MIXED) es = (gj < row.g) ? es : 0.0;
    M += eb;
    X += es;
    const double cc = eb + es;
#pragma unroll
    for (int d = 0; d < D; ++d) G[d] = fma(cc, dx[d], G[d]);
  }
}

// Pass 2 (gradient pass, terms weighted by rho'_j) for one (i, j) pair.
//  KIND_EARLIER: xi_ji = 0 -> rho_j mu_ij only.   KIND_LATER: rho_j (mu_ij + xi_ji).
template <int D, int KIND>
__device__ __forceinline__ void pair_pass2(const double* __restrict__ rj, int gj,
                                           const RowState<D>& row, double (&G)[D],
                                           const PassConst& c, const int2* __restrict__ tab) {
  double dx[D];
  double r2;
#pragma unroll
  for (int d = 0; d < D; ++d) dx[d] = rj[d] - row.x[d];
  r2 = dx[0] * dx[0];
#pragma unroll
  for (int d = 1; d < D; ++d) r2 = fma(dx[d], dx[d], r2);
  const double dt = row.t - rj[D];
  const double rho = rj[D + 1];
  const double ab = fma(c.kx, r2, fma(c.kt * dt, dt, c.lnc_b));
  double eb = fexp(ab, tab);
  if (KIND == KIND_MIXED) eb = (gj == row.g) ? 0.0 : eb;
  double cc;
  if (KIND == KIND_EARLIER) {
    cc = rho * eb;
  } else {
    // xi_ji: t_j > t_i, exponent k_s r^2 - omega (t_j - t_i) = k_s r^2 + omega dt
    const double as = fma(c.ks, r2, fma(c.omega, dt, c.lnc_s));
    double es = fexp(as, tab);
    if (KIND == KIND_MIXED) es = (gj > row.g) ? es : 0.0;
    cc = rho * (eb + es);
  }
#pragma unroll
  for (int d = 0; d < D; ++d) G[d] = fma(cc, dx[d], G[d]);
}

// ------------------------------------------------------------- persistent kernel
struct PassArgs {
  const double* rec;     // Npad x REC
  const int* gid;        // Npad tie-group ids (first index with the same time)
  const int2* items;     // (row tile, chunk)
  int* counter;          // work counter, zeroed before launch
  double* part;          // [chunks][Npad][K]
  const int2* tab;       // EXP_TABLE-entry exp table in global memory
  long long npad;
  int N;
  int n_items;
  int chunk;             // events per j chunk (multiple of TILE_J)
  PassConst c;          // by value: DFMA constant-bank operands
};

template <int D, int PASS, int R>
__global__ void __launch_bounds__(THREADS, D <= 4 ? 4 : 3) pass_kernel(PassArgs a) {
  using L = Layout<D>;
  constexpr int REC = L::REC;
  constexpr int RT = THREADS * R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stage = reinterpret_cast<double*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + STAGES * TILE_J * REC * sizeof(double));
  int2* tab = reinterpret_cast<int2*>(bars + STAGES);
  __shared__ int s_item;

  const int tid = threadIdx.x;
  for (int q = tid; q < EXP_TABLE; q += THREADS) tab[q] = a.tab[q];
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t parity = 0;  // bit s = parity to wait for on stage s
  const PassConst c = a.c;
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

    RowState<D> row[R];
    double M[R], X[R], G[R][D];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = min(row0 + tid + r * THREADS, N - 1);
      const double* ri = a.rec + (long long)i * REC;
#pragma unroll
      for (int d = 0; d < D; ++d) row[r].x[d] = ri[d];
      row[r].t = ri[D];
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
                    (uint32_t)(cnt * REC * sizeof(double)), &bars[s]);
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
      const double* st = stage + s * TILE_J * REC;
      const int kind = (gj_last < g_first) ? KIND_EARLIER
                                           : ((gj_first > g_last) ? KIND_LATER : KIND_MIXED);
      if (kind == KIND_EARLIER) {
#pragma unroll 2
        for (int jj = 0; jj < cnt; ++jj) {
          const double* rj = st + jj * REC;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (PASS == 1)
              pair_pass1<D, KIND_EARLIER>(rj, 0, row[r], M[r], X[r], G[r], c, tab);
            else
              pair_pass2<D, KIND_EARLIER>(rj, 0, row[r], G[r], c, tab);
          }
        }
      } else if (kind == KIND_LATER) {
#pragma unroll 2
        for (int jj = 0; jj < cnt; ++jj) {
          const double* rj = st + jj * REC;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (PASS == 1)
              pair_pass1<D, KIND_LATER>(rj, 0, row[r], M[r], X[r], G[r], c, tab);
            else
              pair_pass2<D, KIND_LATER>(rj, 0, row[r], G[r], c, tab);
          }
        }
      } else {
        for (int jj = 0; jj < cnt; ++jj) {
          const double* rj = st + jj * REC;
          const int gj = a.gid[jt + jj];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if (PASS == 1)
              pair_pass1<D, KIND_MIXED>(rj, gj, row[r], M[r], X[r], G[r], c, tab);
            else
              pair_pass2<D, KIND_MIXED>(rj, gj, row[r], G[r], c, tab);
          }
        }
      }
      __syncthreads();  // every lane is done with stage s
      if (tid == 0 && tl + STAGES < ntiles) {
        const int jn = j0 + (tl + STAGES) * TILE_J;
        const int cn = min(TILE_J, j1 - jn);
        tma_load_1d(stage + s * TILE_J * REC, a.rec + (long long)jn * REC,
                    (uint32_t)(cn * REC * sizeof(double)), &bars[s]);
      }
    }

    // partial sums of this item
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = row0 + tid + r * THREADS;
      if (i < N) {
        if (PASS == 1) {
          double* o = a.part + ((long long)w.y * a.npad + i) * L::K1;
          o[0] = M[r];
          o[1] = X[r];
#pragma unroll
          for (int d = 0; d < D; ++d) o[2 + d] = G[r][d];
        } else {
          double* o = a.part + ((long long)w.y * a.npad + i) * L::K2;
#pragma unroll
          for (int d = 0; d < D; ++d) o[d] = G[r][d];
        }
      }
    }
  }
}

}  // namespace hk
