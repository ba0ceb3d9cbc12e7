// hawkes_plan.h -- host-side work decomposition (pure functions of N, W and rank):
// chunk lengths of the two decompositions, the zig-zag row-tile deal of ROWS and the
// greedy deal of PAIRS' chunk pairs.  Included by hawkes_api.cu only.
#pragma once
#include <math.h>
#include <cmath>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "hawkes_kernels.cuh"

namespace hk {

int chunk_of(long long N) {
  // j chunk: a function of N only (never of W), so per-row sums are W-independent
  long long c = (N + 63) / 64;
  c = ((c + TILE_J - 1) / TILE_J) * TILE_J;
  c = std::max<long long>(4 * TILE_J, std::min<long long>(8192, c));
  return (int)c;
}

// PAIRS chunk: a multiple of the sym kernel's 128-event tile, ~N/(138 sqrt(W)) so that the
// C(C+1)/2 chunk pairs give every rank >= ~16 work items per CTA slot (tail < ~5 %) while
// the [C+1][Npad][K] partial arrays stay ~C*N*48 bytes; 128 for small N (latency: small
// catalogs still fill the GPU).  PAIRS sums are not bitwise W-independent anyway (the
// per-event partials meet in an allreduce), so the chunk may depend on W.
int chunk_pairs_of(long long N, int W) {
  if (const char* e = getenv("HAWKES_PAIRS_CHUNK")) {   // diagnostics: A/B of the chunk size
    const long long c = atoll(e) / TILE_J * TILE_J;
    if (c >= TILE_J) return (int)c;
  }
  const double C = 138.0 * sqrt((double)std::max(1, W));
  long long c = (long long)llround((double)N / C / TILE_J) * TILE_J;   // nearest multiple
  // one-tile chunks make every item a single 128 x 128 tile pair, whose fixed cost (row
  // tile load, 4-warp row reduction, partial writes) shows: where 256-event chunks still
  // leave >= 64 sqrt(W) chunks (>= ~4.7 items per CTA slot) take them (N = 20k: -2 %,
  // profiles/r01_chunk_sweep.txt)
  if (c <= TILE_J && (double)N / (2 * TILE_J) >= 64.0 * sqrt((double)std::max(1, W))) c = 2 * TILE_J;
  return (int)std::max<long long>(TILE_J, c);
}

// Chunk pairs (a <= b) dealt to ranks by greedy longest-processing-time on their cost.
std::vector<int> pair_owners(long long N, int chunk, int W) {
  const int C = (int)((N + chunk - 1) / chunk);
  struct It { double cost; int a, b; };
  std::vector<It> items;
  for (int a = 0; a < C; ++a)
    for (int b = a; b < C; ++b) {
      const double na = (double)std::min<long long>(chunk, N - (long long)a * chunk);
      const double nb = (double)std::min<long long>(chunk, N - (long long)b * chunk);
      items.push_back({a == b ? 0.5 * na * na : na * nb, a, b});
    }
  std::stable_sort(items.begin(), items.end(), [](const It& x, const It& y) { return x.cost > y.cost; });
  std::vector<double> load(W, 0.0);
  std::vector<int> own((size_t)C * C, -1);
  for (const It& it : items) {
    int r = 0;
    for (int q = 1; q < W; ++q)
      if (load[q] < load[r]) r = q;
    load[r] += it.cost;
    own[(size_t)it.a * C + it.b] = r;
  }
  return own;
}

// Pieces (hawkes_kernels_sym.cuh PairItem s0 / s1).  When a rank's n items fill less than
// one round of the G resident CTA slots of the gradient pass (N = 2000: 136 items, one per
// SM: each CTA runs latency-bound, its 4 warps alone on an SM), every item runs as k pieces
// of 32 / k skewed steps, k the largest of 8, 4, 2 with k n <= G, each piece with its own row
// and column slot blocks, so k CTAs share an item's tile pair (N = 2000: 136 x 4 pieces;
// measured 56.5 -> 51.8 us per l + grad call, N = 500: 54 -> 40 us,
// profiles/r02_latency_pieces.jsonl).  Above one round, whole items: splitting the
// tail of a multi-round plan measured slower (N = 5000, 820 items on 592 slots: +3 %), since
// an item's fixed cost (row and column tile loads, the row reduction) does not split.
inline int choose_pieces(int n, int G) {
  if (const char* e = getenv("HAWKES_PIECES")) {   // diagnostics: 0 / 1 = whole items, 2/4/8
    const int k = atoi(e);
    if (k >= 0) return (k == 2 || k == 4 || k == 8) ? k : 1;
  }
  if (G <= 0 || n <= 0) return 1;
  for (int k : {8, 4, 2})
    if ((long long)k * n <= G) return k;
  return 1;
}

// PAIRS work items and compact slot layout of every rank (hawkes_kernels_sym.cuh PairItem):
// rank r's chunk pairs, heaviest first (dynamic scheduling takes them in this order); for every
// chunk c the ascending slot ids r's items write for c's events (row role of (c, b): b;
// column role of (a, c), a < c: a; of (c, c): C), one block of `chunk` events per slot id,
// chunk after chunk.  The ranks in `mine` (this process) are laid out one after another in one
// array of slot_events events; the others' offsets start at 0 (not allocated here).  At W = 1
// every chunk has C + 1 slots in slot-id order, the order the finalize sums them in.
struct PairsLayout {
  std::vector<std::vector<PairItem>> items;
  std::vector<int> pieces;   // k per rank (1: whole items)
  std::vector<std::vector<long long>> coff;
  std::vector<std::vector<int>> cn;
  long long slot_events = 0;
};

// G > 0: the gradient pass's resident CTA slots, for the pieces above (0: whole items only;
// the host-side plan calls, which know no device)
inline PairsLayout pairs_layout(long long N, int chunk, int W, const std::vector<int>& mine, int G = 0) {
  const int C = (int)((N + chunk - 1) / chunk);
  const std::vector<int> own = pair_owners(N, chunk, W);
  PairsLayout L;
  L.items.assign(W, {});
  L.coff.assign(W, {});
  L.cn.assign(W, {});
  L.pieces.assign(W, 1);
  long long base = 0;
  for (int r = 0; r < W; ++r) {
    const bool is_mine = std::find(mine.begin(), mine.end(), r) != mine.end();
    std::vector<std::pair<double, int2>> items;   // (pair count, (a, b)); heaviest first
    for (int a = 0; a < C; ++a)
      for (int b = a; b < C; ++b) {
        if (own[(size_t)a * C + b] != r) continue;
        const double na = (double)std::min<long long>(chunk, N - (long long)a * chunk);
        const double nb = (double)std::min<long long>(chunk, N - (long long)b * chunk);
        items.push_back({a == b ? 0.5 * na * na : na * nb, make_int2(a, b)});
      }
    std::stable_sort(items.begin(), items.end(),
                     [](const std::pair<double, int2>& x, const std::pair<double, int2>& y) {
                       return x.first > y.first;
                     });
    const int kp = choose_pieces((int)items.size(), G);
    L.pieces[r] = kp;
    auto pieces_of = [&](int) { return kp; };
    // slot ids: piece q of item (a, b) -- row role b + q (C + 1), column role a (C for a
    // diagonal item) + q (C + 1); a whole item is piece 0
    std::vector<std::vector<int>> ids(C);
    for (int i = 0; i < (int)items.size(); ++i) {
      const int a = items[i].second.x, b = items[i].second.y;
      for (int q = 0; q < pieces_of(i); ++q) {
        ids[a].push_back(b + q * (C + 1));
        ids[b].push_back((a == b ? C : a) + q * (C + 1));
      }
    }
    L.coff[r].assign(C, 0);
    L.cn[r].assign(C, 0);
    long long off = is_mine ? base : 0;
    for (int c = 0; c < C; ++c) {
      std::sort(ids[c].begin(), ids[c].end());
      L.coff[r][c] = off;
      L.cn[r][c] = (int)ids[c].size();
      off += (long long)ids[c].size() * chunk;
    }
    auto block = [&](int c, int id) {
      const auto it = std::lower_bound(ids[c].begin(), ids[c].end(), id);
      return L.coff[r][c] + (long long)(it - ids[c].begin()) * chunk;
    };
    for (int i = 0; i < (int)items.size(); ++i) {
      const int a = items[i].second.x, b = items[i].second.y;
      const int k = pieces_of(i);
      for (int q = 0; q < k; ++q)
        L.items[r].push_back(PairItem{a, b, block(a, b + q * (C + 1)),
                                      block(b, (a == b ? C : a) + q * (C + 1)), 32 * q / k,
                                      32 * (q + 1) / k});
    }
    if (is_mine) base = off;
  }
  L.slot_events = base;
  return L;
}

int owner_of_tile(int k, int W) {
  const int pos = k % (2 * W);
  return pos < W ? pos : 2 * W - 1 - pos;
}

}  // namespace hk

// ------------------------------------------------------------- spatial walk order (NEXT-2)
// The PAIRS kernels walk the events in time order by default: chunk pairs and tiles are
// time ranges, which makes the temporal culling exact and cheap.  Where the catalog's
// spatial extent is many bandwidths wide (the DC shape: 16 km across, a 3.7 km
// background cutoff), a spatial walk order instead makes tiles compact in space, so whole
// tile pairs and chunk pairs fall outside every kernel's reach and are skipped by their
// bounding boxes.  The order sorts the locations quantised on their bounding box: D = 2 by
// the Hilbert curve index (16 bits per dimension; its tiles are more compact than the Z-order
// ones: 15 % fewer live tile pairs at the DC shape, N = 5000), other D by the Morton (Z-order)
// key (64 / D bits per dimension); ties broken by index.
namespace hk {

// Hilbert index of (x, y) on a 2^bits grid (the classic rotate-and-flip walk)
inline unsigned long long hilbert_d(unsigned long long x, unsigned long long y, int bits) {
  unsigned long long d = 0;
  for (unsigned long long s = 1ULL << (bits - 1); s > 0; s >>= 1) {
    const unsigned long long rx = (x & s) ? 1 : 0, ry = (y & s) ? 1 : 0;
    d += s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = s - 1 - x;
        y = s - 1 - y;
      }
      std::swap(x, y);
    }
  }
  return d;
}

inline std::vector<int> morton_order(const double* x, int N, int D) {
  const int bits = D == 2 ? 16 : std::min(21, 64 / D);
  std::vector<double> lo(D, INFINITY), hi(D, -INFINITY);
  for (int i = 0; i < N; ++i)
    for (int d = 0; d < D; ++d) {
      lo[d] = std::min(lo[d], x[(size_t)i * D + d]);
      hi[d] = std::max(hi[d], x[(size_t)i * D + d]);
    }
  const double scale = (double)((1ULL << bits) - 1);
  std::vector<std::pair<unsigned long long, int>> key(N);
  for (int i = 0; i < N; ++i) {
    unsigned long long k = 0, qd[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int d = 0; d < D; ++d) {
      const double w = hi[d] > lo[d] ? (x[(size_t)i * D + d] - lo[d]) / (hi[d] - lo[d]) : 0.0;
      qd[d] = (unsigned long long)std::llround(std::min(1.0, std::max(0.0, w)) * scale);
      for (int b = 0; b < bits; ++b) k |= ((qd[d] >> b) & 1ULL) << (b * D + d);
    }
    if (D == 2) k = hilbert_d(qd[0], qd[1], bits);
    key[i] = {k, i};
  }
  std::sort(key.begin(), key.end());
  std::vector<int> perm(N);
  for (int i = 0; i < N; ++i) perm[i] = key[i].second;
  return perm;
}

// Work estimate of a walk order: over the unordered tile pairs (128-event tiles of the order,
// diagonal pairs at half weight), the number of pair terms (background, self-excitation)
// whose bound from the two tiles' boxes can exceed the exp's clamp.  spatial_boxes = false
// mirrors the time-order kernel, which bounds by the time gap alone.  Large N: a strided
// sample of the tile pairs (the estimate only chooses between two orders).
inline double walk_cost(const double* x, const double* t, const int* order, int N, int D,
                        const PassConst& c, bool spatial_boxes) {
  const int nt = (N + TILE_J - 1) / TILE_J;
  std::vector<double> box((size_t)nt * (2 * D + 2));
  for (int k = 0; k < nt; ++k) {
    double* b = &box[(size_t)k * (2 * D + 2)];
    for (int d = 0; d <= D; ++d) {
      b[d < D ? d : 2 * D] = INFINITY;
      b[d < D ? D + d : 2 * D + 1] = -INFINITY;
    }
    for (int p = k * TILE_J; p < std::min(N, (k + 1) * TILE_J); ++p) {
      const int i = order ? order[p] : p;
      for (int d = 0; d < D; ++d) {
        b[d] = std::min(b[d], x[(size_t)i * D + d]);
        b[D + d] = std::max(b[D + d], x[(size_t)i * D + d]);
      }
      b[2 * D] = std::min(b[2 * D], t[i]);
      b[2 * D + 1] = std::max(b[2 * D + 1], t[i]);
    }
  }
  const long long pairs = (long long)nt * (nt + 1) / 2;
  const long long stride = std::max<long long>(1, pairs / 4000000);
  double cost = 0.0;
  long long q = 0;
  for (int a = 0; a < nt; ++a)
    for (int b = a; b < nt; ++b, ++q) {
      if (q % stride) continue;
      const double* A = &box[(size_t)a * (2 * D + 2)];
      const double* B = &box[(size_t)b * (2 * D + 2)];
      double r2 = 0.0;
      if (spatial_boxes)
        for (int d = 0; d < D; ++d) {
          const double g = std::max(0.0, std::max(B[d] - A[D + d], A[d] - B[D + d]));
          r2 += g * g;
        }
      const double dt = std::max(0.0, std::max(B[2 * D] - A[2 * D + 1], A[2 * D] - B[2 * D + 1]));
      const double w = a == b ? 0.5 : 1.0;
      if (c.kx * r2 + c.kt * dt * dt + c.lnc_b > CULL_EXPONENT) cost += w;
      if (c.ks * r2 - c.omega * dt + c.lnc_s > CULL_EXPONENT) cost += w;
    }
  return cost * (double)stride;
}

}  // namespace hk
