/* Per-call latency of hawkes_grad_at from C (no Python): N events of the unit-square
 * generator's shape (uniform x, sorted t), device buffers, host sync on ell every call.
 *   gcc -O2 -I include tools/c_grad_at_latency.c -L paper_2010_02994_b200 -lhawkes_b200 \
 *       -Wl,-rpath,$PWD/paper_2010_02994_b200 -L<cudart dir> -lcudart -lm -o /tmp/lat && /tmp/lat 5000
 * Prints one JSON line: {"N": ..., "us_per_call": ...}. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include "hawkes.h"

extern int cudaMalloc(void** p, size_t n);
extern int cudaMemcpy(void* d, const void* s, size_t n, int kind);

static double now(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 5000;
  const int reps = argc > 2 ? atoi(argv[2]) : 1000;
  const int32_t D = 2;
  double* x = malloc(sizeof(double) * N * D);
  double* t = malloc(sizeof(double) * N);
  uint64_t s = 12345;
  for (int64_t k = 0; k < N * D; ++k) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    x[k] = (double)(s >> 11) * 0x1.0p-53;
  }
  for (int64_t n = 0; n < N; ++n) t[n] = (double)n / (double)N;
  hawkes_ctx* ctx = NULL;
  if (hawkes_create(N, D, NULL, &ctx) != HAWKES_OK) return 3;
  const hawkes_params th = {0.6, 0.1, 0.1, 0.4, 20.0, 0.03};
  double *xd = NULL, *gd = NULL, ell = 0.0;
  cudaMalloc((void**)&xd, sizeof(double) * N * D);
  cudaMalloc((void**)&gd, sizeof(double) * N * D);
  cudaMemcpy(xd, x, sizeof(double) * N * D, 1 /* cudaMemcpyHostToDevice */);
  if (hawkes_set_times(ctx, t, HAWKES_MEM_HOST) || hawkes_set_params(ctx, &th)) return 1;
  for (int k = 0; k < 20; ++k)
    if (hawkes_grad_at(ctx, xd, gd, &ell)) return 1;
  const double t0 = now();
  for (int k = 0; k < reps; ++k) hawkes_grad_at(ctx, xd, gd, &ell);
  const double dt = (now() - t0) / reps;
  printf("{\"N\": %lld, \"us_per_call\": %.3f, \"ell\": %.10f}\n", (long long)N, dt * 1e6, ell);
  hawkes_destroy(ctx);
  return 0;
}
