// hawkes_mh.cuh -- on-device block Metropolis-Hastings over coarsened locations.
//
// The DC and Alaska samplers update the latent locations with "a Metropolis-Hastings
// kernel with block-wise updates over sets of individual location variables":
//   * square regions (Eq. locsPrior1, |x_nd - c_nd| < s_n): per dimension a normal
//     proposal N(x_nd, (scale s_n)^2) truncated to the region ("truncated normal
//     proposals"), drawn by inverting the CDF; Hastings ratio prod_d Z_d(x) / Z_d(x*) with
//     Z_d the truncation mass;
//   * disc regions (Eq. locsPrior2, |x_n - c_n| < r_n, D = 2): x* uniform on the
//     intersection of disc(c_n, r_n) and disc(x_n, eps r_n), eps = scale (Eq. circleKernel),
//     by rejection; Hastings ratio A(x)/A(x*) with A the closed-form lens area.
// Per block, four launches (captured once as a CUDA graph and replayed per block):
// k_mh_propose (one CTA: proposals, proposal-slot map, Hastings sum in a fixed order),
// k_move_delta_rows (the O(kN) Delta ell work of hawkes_moves.cuh), k_move_terms_final
// (the per-event terms; its last CTA sums them and takes the Metropolis decision with a
// counter-based uniform), and k_move_commit gated on that decision.  No host round trip.
//
// Random numbers: Philox-4x32-10 (hawkes_ops.cuh) with counter (it_lo, it_hi, b, tag), key
// (seed_lo, seed_hi), b the block index within the sweep; proposal draws of slot q use
// tag = 0x80000000 | q << 12 | a, the accept uniform tag = 0xC0000000.
#pragma once
#include "hawkes_moves.cuh"
#include "hawkes_ops.cuh"

namespace hk {

constexpr unsigned MH_TAG = 0x80000000u, MH_ACCEPT_TAG = 0xC0000000u;
constexpr int MH_MAX_ATTEMPTS = 4096;
enum { REGION_SQUARE = 1, REGION_DISC = 2 };

__device__ __forceinline__ double2 mh_uniforms(uint2 key, unsigned long long it, unsigned b, unsigned tag) {
  const uint4 w = philox10(make_uint4((unsigned)it, (unsigned)(it >> 32), b, tag), key);
  return make_double2(u53(w.x, w.y), u53(w.z, w.w));
}

// The proposal arithmetic uses explicit round-to-nearest operations (no FMA contraction):
// it is inlined into more than one kernel (the launch-based and the cooperative sweep),
// and contraction choices that differ between inlining sites would make the two paths'
// proposals differ in the last bit.  (The oracle evaluates these formulas unfused too.)
#define MUL __dmul_rn
#define ADD __dadd_rn
#define SUB __dsub_rn

// N(x, s^2) mass of (lo, hi): 1 - Q((hi - x)/s) - Phi((lo - x)/s), Q = upper tail
__device__ __forceinline__ double trunc_mass(double x, double lo, double hi, double s) {
  const double r2 = 0.70710678118654752440;
  return SUB(SUB(1.0, MUL(0.5, erfc(MUL(SUB(hi, x) / s, r2)))),
             MUL(0.5, erfc(MUL(-(SUB(lo, x) / s), r2))));
}

// area of disc(0, R) cap disc(d e_1, rho)
__device__ __forceinline__ double lens(double R, double rho, double d) {
  const double pi = 3.14159265358979323846;
  if (d >= ADD(R, rho)) return 0.0;
  if (ADD(d, rho) <= R) return MUL(MUL(pi, rho), rho);
  if (ADD(d, R) <= rho) return MUL(MUL(pi, R), R);
  const double dd = MUL(d, d), rr = MUL(rho, rho), RR = MUL(R, R);
  const double t1 = MUL(rr, acos(SUB(ADD(dd, rr), RR) / MUL(MUL(2.0, d), rho)));
  const double t2 = MUL(RR, acos(SUB(ADD(dd, RR), rr) / MUL(MUL(2.0, d), R)));
  const double k = MUL(0.5, sqrt(MUL(MUL(MUL(ADD(SUB(rho, d), R), SUB(ADD(d, rho), R)), ADD(SUB(d, rho), R)),
                                     ADD(ADD(d, rho), R))));
  return SUB(ADD(t1, t2), k);
}

// one CTA of 256 threads; slot q < k proposes for event n = blocks[b*k + q]
// One event's proposal (slot q of block b) and its log Hastings term.
template <int D>
__device__ __forceinline__ double mh_propose_one(int n, int q, int b, uint2 key, unsigned long long it,
                                                 double scale, int kind, const double* __restrict__ xcur,
                                                 const double* __restrict__ centre,
                                                 const double* __restrict__ size, double (&y)[D]) {
  double x[D], c[D];
  double logh = 0.0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    x[d] = xcur[(long long)n * D + d];
    c[d] = centre[(long long)n * D + d];
  }
  const double sz = size[n];
  if (kind == REGION_SQUARE) {
    const double s = MUL(scale, sz);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double2 uu = mh_uniforms(key, it, (unsigned)b, MH_TAG | ((unsigned)q << 12) | (unsigned)(d / 2));
      const double u = (d & 1) ? uu.y : uu.x;
      const double lo = SUB(c[d], sz), hi = ADD(c[d], sz);
      const double Z0 = trunc_mass(x[d], lo, hi, s);
      const double p = ADD(MUL(0.5, erfc(MUL(-(SUB(lo, x[d]) / s), 0.70710678118654752440))), MUL(u, Z0));
      const double z = normcdfinv(p);
      y[d] = fmin(fmax(ADD(x[d], MUL(s, z)), lo), hi);
      logh = ADD(logh, SUB(log(Z0), log(trunc_mass(y[d], lo, hi, s))));
    }
  } else if constexpr (D >= 2) {   // REGION_DISC (the API admits it for D == 2 only)
    const double r = sz, rho = MUL(scale, sz);
#pragma unroll
    for (int d = 0; d < D; ++d) y[d] = x[d];
    for (int a = 0; a < MH_MAX_ATTEMPTS; ++a) {
      const double2 uu = mh_uniforms(key, it, (unsigned)b, MH_TAG | ((unsigned)q << 12) | (unsigned)a);
      const double rad = MUL(rho, sqrt(uu.x));
      double sn, cs;
      sincospi(MUL(2.0, uu.y), &sn, &cs);
      const double y0 = ADD(x[0], MUL(rad, cs)), y1 = ADD(x[1], MUL(rad, sn));
      const double e0 = SUB(y0, c[0]), e1 = SUB(y1, c[1]);
      if (ADD(MUL(e0, e0), MUL(e1, e1)) < MUL(r, r)) {
        y[0] = y0;
        y[1] = y1;
        logh = SUB(log(lens(r, rho, hypot(SUB(x[0], c[0]), SUB(x[1], c[1])))), log(lens(r, rho, hypot(e0, e1))));
        break;
      }
    }
  }
  return logh;
}

// The block index, key, iteration and scale come from st (device-resident), so the same
// launch -- and a CUDA graph of the whole block step -- serves every block of a sweep.  The
// previous block's proposal slots are cleared first (its commit has run).
template <int D>
__global__ void __launch_bounds__(256) k_mh_propose(const int* __restrict__ blocks, int k,
                                                    const double* __restrict__ xcur,
                                                    const double* __restrict__ centre,
                                                    const double* __restrict__ size, int kind,
                                                    int* __restrict__ move_idx,
                                                    double* __restrict__ move_x,
                                                    int* __restrict__ slot_of, EvalStatus* st) {
  __shared__ double sh[256];
  const int q = threadIdx.x;
  const int b = st->mh_block;
  const int prevk = st->mh_prevk;
  const uint2 key = make_uint2(st->mh_key_lo, st->mh_key_hi);
  const unsigned long long it = st->mh_it;
  const double scale = st->mh_scale;
  if (q < prevk) slot_of[move_idx[q]] = -1;
  __syncthreads();
  double logh = 0.0;
  if (q < k) {
    const int n = blocks[(long long)b * k + q];
    move_idx[q] = n;
    slot_of[n] = q;
    double y[D];
    logh = mh_propose_one<D>(n, q, b, key, it, scale, kind, xcur, centre, size, y);
#pragma unroll
    for (int d = 0; d < D; ++d) move_x[q * D + d] = y[d];
  }
  logh = cta_sum256(logh, sh);
  if (q == 0) {
    st->mh_hastings = logh;
    st->mh_cur = b;
    st->mh_prevk = k;
  }
}

#undef MUL
#undef ADD
#undef SUB

}  // namespace hk
