// hawkes_plan.h -- host-side work decomposition (pure functions of N, W and rank):
// chunk lengths of the two decompositions, the zig-zag row-tile deal of ROWS and the
// greedy deal of PAIRS' chunk pairs.  Included by hawkes_api.cu only.
#pragma once
#include <math.h>
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

int owner_of_tile(int k, int W) {
  const int pos = k % (2 * W);
  return pos < W ? pos : 2 * W - 1 - pos;
}

}  // namespace hk
