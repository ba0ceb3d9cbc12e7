/* examples/c_api_demo.c -- the C ABI (include/hawkes.h) from plain C, no Python or torch:
 * a seeded synthetic catalog on the unit square, ell (Eq. 1) and the location
 * gradient (App. A) from host buffers, then one HMC leapfrog trajectory.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_2010_02994_b200 -lhawkes_b200 \
 *       -Wl,-rpath,$PWD/paper_2010_02994_b200 -lm -o /tmp/c_api_demo
 *   /tmp/c_api_demo [N]
 *
 * Exit status 0 with "ok" lines on a B200; without a usable device hawkes_create returns
 * HAWKES_ERR_CUDA, which the demo reports (exit 3) -- there is no CPU fallback. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "hawkes.h"

static uint64_t rng_state = 20102994u;
static double urand(void) {   /* xorshift64*: inputs only, no part of the method */
  rng_state ^= rng_state >> 12;
  rng_state ^= rng_state << 25;
  rng_state ^= rng_state >> 27;
  return (double)((rng_state * 2685821657736338717ull) >> 11) * 0x1.0p-53;
}

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 2000;
  const int32_t D = 2;
  printf("hawkes ABI version %d\n", hawkes_abi_version());
  double* x = malloc(sizeof(double) * N * D);
  double* t = malloc(sizeof(double) * N);
  double* g = malloc(sizeof(double) * N * D);
  double* p = calloc(N * D, sizeof(double));
  for (int64_t n = 0; n < N; ++n) {
    x[n * D] = urand();
    x[n * D + 1] = urand();
    t[n] = (double)n / (double)N;   /* sorted, distinct */
  }
  hawkes_ctx* ctx = NULL;
  int rc = hawkes_create(N, D, NULL, &ctx);
  if (rc != HAWKES_OK) {
    printf("hawkes_create: status %d (%s)\n", rc, rc == HAWKES_ERR_CUDA ? "no usable sm_100 device" : "error");
    return rc == HAWKES_ERR_CUDA ? 3 : 1;
  }
  const hawkes_params th = {0.6, 0.1, 0.1, 0.4, 20.0, 0.03};   /* (mu0, tau_x, tau_t, theta, omega, h) */
  double ell = 0.0, ell2 = 0.0, kin = 0.0;
  if ((rc = hawkes_set_times(ctx, t, HAWKES_MEM_HOST)) || (rc = hawkes_set_locations(ctx, x, HAWKES_MEM_HOST)) ||
      (rc = hawkes_set_params(ctx, &th)) || (rc = hawkes_loglik(ctx, &ell)) ||
      (rc = hawkes_grad_locations(ctx, g, HAWKES_MEM_HOST, &ell2))) {
    printf("error %d: %s\n", rc, hawkes_last_error(ctx));
    return 1;
  }
  /* translation invariance: the gradient sums to ~0 over the events */
  double s0 = 0.0, s1 = 0.0, a = 0.0;
  for (int64_t n = 0; n < N; ++n) {
    s0 += g[n * D];
    s1 += g[n * D + 1];
    a += fabs(g[n * D]) + fabs(g[n * D + 1]);
  }
  printf("ok: N=%lld ell=%.10f (loglik %.10f) |sum g|/sum|g| = %.2e\n", (long long)N, ell2, ell,
         (fabs(s0) + fabs(s1)) / a);
  for (int64_t k = 0; k < N * D; ++k) p[k] = urand() - 0.5;
  if ((rc = hawkes_leapfrog(ctx, x, p, HAWKES_MEM_HOST, 1e-5, 10, NULL, NULL, NULL, &ell, &kin))) {
    printf("leapfrog error %d: %s\n", rc, hawkes_last_error(ctx));
    return 1;
  }
  printf("ok: leapfrog 10 steps: ell_end=%.10f kinetic_end=%.6f\n", ell, kin);
  hawkes_destroy(ctx);
  free(x);
  free(t);
  free(g);
  free(p);
  return (ell == ell && fabs(s0) + fabs(s1) <= 1e-9 * a) ? 0 : 1;
}
