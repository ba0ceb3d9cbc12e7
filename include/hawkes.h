/*
 * hawkes.h -- C ABI of the B200 (sm_100a) Hawkes log-likelihood + location-gradient library.
 *
 * The library evaluates, for a time-sorted catalog of N events (x_n in R^D, t_n >= 0)
 * and parameters Theta = (mu0, tau_x, tau_t, theta, omega, h):
 *
 *   lambda_n = sum_{n'} mu_{nn'} + xi_{nn'}                                  Eq. 1
 *     mu_{nn'} = mu0/(tau_x^D tau_t) phi_D((x_n-x_n')/tau_x) phi((t_n-t_n')/tau_t) I[t_n != t_n']
 *                                                                            P:L80-83
 *     xi_{nn'} = theta omega/h^D e^{-omega (t_n - t_n')} phi_D((x_n-x_n')/h) I[t_n' < t_n]
 *                                                                            P:L76-79
 *   Lambda_n = mu0 (Phi((t_N-t_n)/tau_t) - Phi(-t_n/tau_t)) - theta (e^{-omega (t_N-t_n)} - 1)
 *                                                                            P:L92-93
 *   ell      = sum_n log lambda_n - Lambda_n                                 Eq. 1
 *   d ell / d x_n = sum_{n'} (mu_{nn'}/lambda_n + mu_{n'n}/lambda_{n'}) (x_{n'}-x_n)/tau_x^2
 *                         + (xi_{nn'}/lambda_n + xi_{n'n}/lambda_{n'}) (x_{n'}-x_n)/h^2
 *                                                                            App. A
 * (phi_D = D-variate standard normal density; the gradient's sigma_x is the paper's h;
 * see DESIGN.md "Readings").  One gradient evaluation is the two-pass computation of
 * Alg. 1/2: a rate pass producing lambda_n, then a gradient pass through
 * 1/lambda.  Around it, the samplers that call it run on the device too: the HMC leapfrog
 * (hawkes_leapfrog) and a whole HMC transition with Philox momenta and the Metropolis
 * decision (hawkes_hmc_step) over X; block Metropolis-Hastings moves in O(kN)
 * (hawkes_propose_move / hawkes_accept_move) and the paper's coarsened-location sampler as
 * an on-device sweep (hawkes_set_regions / hawkes_mh_sweep); and the flu
 * model's Bayesian MDS density (hawkes_set_bmds).
 *
 * Conventions (all functions):
 *  - Every function returns a hawkes_status; no C++ exception crosses this boundary.
 *    On failure hawkes_last_error(ctx) holds a one-line message.  A CUDA or NCCL error
 *    is sticky: the context becomes unusable (every later call returns the same status).
 *  - The context owns all device memory.  set_* functions COPY the caller's arrays; the
 *    caller keeps ownership of every pointer it passes.  Outputs go to caller buffers.
 *  - hawkes_mem says where a caller pointer lives: HAWKES_MEM_HOST (pageable or pinned
 *    host memory) or HAWKES_MEM_DEVICE (device memory on opts.device).
 *  - Work is stream-ordered on opts.cuda_stream (NULL = legacy default stream).
 *    Functions that return a host scalar or write host memory synchronise that stream.
 *  - A context is not re-entrant; distinct contexts are independent.
 *  - Arrays are row-major: x is N*D doubles (x[n*D + d]), gradients likewise.
 *  - The library needs an sm_100 device; it fails with HAWKES_ERR_CUDA otherwise.
 */
#ifndef HAWKES_B200_H
#define HAWKES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HAWKES_ABI_VERSION 4   /* 3: HMC transition, coarsening regions + MH sweep, get_locations; 4: hawkes_grad_at */

typedef struct hawkes_ctx hawkes_ctx; /* opaque; owns all device memory */

typedef enum {
  HAWKES_OK = 0,
  HAWKES_ERR_ARG = -1,            /* null pointer, bad size, bad enum                        */
  HAWKES_ERR_DIM = -2,            /* unsupported D (supported: 1..HAWKES_MAX_D)             */
  HAWKES_ERR_UNSORTED = -3,       /* times not non-decreasing                                */
  HAWKES_ERR_NONFINITE = -4,      /* NaN/Inf, negative time, or |value| > 1e100 in inputs    */
  HAWKES_ERR_PARAM = -5,          /* Theta not finite / not positive / outside exp range     */
  HAWKES_ERR_STATE = -6,          /* a required set_* call is missing                        */
  HAWKES_ERR_GRAD_UNDEFINED = -7, /* some lambda_n = 0 (ell = -inf): gradient undefined      */
  HAWKES_ERR_CUDA = -8,           /* CUDA runtime failure (sticky)                           */
  HAWKES_ERR_NCCL = -9,           /* NCCL failure or NCCL unavailable (sticky)               */
  HAWKES_ERR_OOM = -10            /* device allocation failed                                */
} hawkes_status;

#define HAWKES_MAX_D 8

typedef enum {
  HAWKES_FP64 = 0, /* fp64 pair arithmetic and sums (reference precision, reading R13)     */
  HAWKES_FP32 = 1  /* fp32 pair arithmetic, fp32 in-tile sums promoted to fp64 per tile    */
} hawkes_precision;

typedef enum { HAWKES_MEM_HOST = 0, HAWKES_MEM_DEVICE = 1 } hawkes_mem;

/* Work decomposition of the two O(N^2) passes (both compute the same quantities):
 *  ROWS  -- ordered pairs: every row i sums over all j (3 exps per ordered pair over both
 *           passes); W > 1 shards row tiles and allgathers (1/lambda, ell_n) between the
 *           passes; results are bitwise identical for every W.
 *  PAIRS -- unordered pairs: chunk pairs (a < b) evaluate each pair's two exps once and
 *           feed both events (2 exps per ordered pair over both
 *           passes); W > 1 shards chunk pairs and allgathers per-event partial sums,
 *           added in rank order; results are bitwise reproducible for a fixed W.  Every D
 *           (1..8).
 *  AUTO  -- PAIRS (about 2x ROWS at N ~ 5k, ahead or level at 20k for every D). */
typedef enum { HAWKES_ALGO_AUTO = 0, HAWKES_ALGO_ROWS = 1, HAWKES_ALGO_PAIRS = 2 } hawkes_algorithm;

/* Walk order of the PAIRS fp64 kernels (hawkes_set_ordering):
 *  TIME  -- events in time order: chunk pairs and tiles are time ranges (exact temporal
 *           culling of tile pairs whose time gap puts both terms below the exp's clamp).
 *  SPACE -- events in a Morton (Z-order) permutation of their locations, fixed when chosen:
 *           tiles are compact in space and tile pairs / chunk pairs whose bounding boxes (in
 *           space and time) put both terms below the clamp are skipped -- the same exact
 *           culling rule, which pays on catalogs many bandwidths wide (the DC shape).
 *  AUTO  -- SPACE when a box-based work estimate of both orders (hawkes_plan.h walk_cost) is
 *           > 10 % lower for it, decided at the first evaluation after hawkes_set_times /
 *           hawkes_set_ordering from the locations and Theta of that evaluation (kept
 *           through later set_locations / set_params: the choice affects speed and summation
 *           order, never which terms are summed).  ROWS and D > 4 walk in time order; fp32
 *           contexts take the spatial walk too (their bounds against the fp32 flush). */
typedef enum { HAWKES_ORDER_AUTO = 0, HAWKES_ORDER_TIME = 1, HAWKES_ORDER_SPACE = 2 } hawkes_ordering;

typedef struct {
  int32_t device;            /* CUDA device ordinal                                           */
  void* cuda_stream;         /* cudaStream_t to run on; NULL = default stream                  */
  int32_t precision;         /* hawkes_precision                                              */
  int32_t rank, world;       /* row sharding: this process's rank and the number of ranks     */
  const void* nccl_unique_id;/* world > 1: pointer to a 128-byte ncclUniqueId that every rank
                                received from rank 0; the library builds its own communicator.
                                With world == 1 a non-NULL id builds a one-rank communicator
                                and runs the sharded path with its real NCCL collectives on
                                this GPU (single-GPU test of the multi-GPU plumbing; no
                                CUDA graphs); cannot be combined with emulate_world > 1     */
  int32_t emulate_world;     /* world == 1 only: > 1 runs that many logical row shards one
                                after another on this GPU, exchanging through device memory
                                (exercises the sharded path without more GPUs); 0/1 = off      */
  int32_t algorithm;         /* hawkes_algorithm                                              */
} hawkes_opts;

/* Theta in the paper's order.  sigma_x is the paper's h (Eq. 1 / App. A).
 * Requirements: tau_x, tau_t, omega, sigma_x finite and > 0; mu0, theta finite and >= 0
 * (the paper's priors keep them > 0; 0 is allowed for the special cases theta = 0 /
 * mu0 = 0); the folded kernel constants must stay inside the fp64 exp range
 * (|log(mu0/(tau_x^(D+2) tau_t))|, |log(theta omega/h^(D+2))| < 600), else HAWKES_ERR_PARAM.
 * The prior orderings 1/omega < tau_t and h < tau_x are NOT enforced. */
typedef struct {
  double mu0, tau_x, tau_t, theta, omega, sigma_x;
} hawkes_params;

/* Fill opts with defaults: device 0, default stream, FP64, rank 0 of 1, no emulation,
 * HAWKES_ALGO_AUTO. */
int hawkes_default_opts(hawkes_opts* opts);

/* Create a context for N >= 1 events in D dimensions (1 <= D <= HAWKES_MAX_D).
 * opts may be NULL (defaults).  With world > 1 every rank must call this with identical
 * N, D and opts (except rank); it is collective (NCCL communicator creation).
 * Errors: HAWKES_ERR_ARG, HAWKES_ERR_DIM, HAWKES_ERR_CUDA, HAWKES_ERR_NCCL, HAWKES_ERR_OOM. */
int hawkes_create(int64_t N, int32_t D, const hawkes_opts* opts, hawkes_ctx** out);

/* Release all device memory and the communicator.  NULL is a no-op. */
int hawkes_destroy(hawkes_ctx* ctx);

/* Event times t[0..N): finite, >= 0 (the integration window starts at 0), and
 * non-decreasing (the catalog order of P:L84, t_N = last).  Copied.  Synchronous.
 * Errors: HAWKES_ERR_ARG, HAWKES_ERR_NONFINITE, HAWKES_ERR_UNSORTED. */
int hawkes_set_times(hawkes_ctx* ctx, const double* t, int32_t mem);

/* Locations x[0..N*D) row-major.  Copied.  Host input is validated immediately
 * (HAWKES_ERR_NONFINITE); device input is validated on the device and reported by the
 * next hawkes_loglik / hawkes_grad_locations / hawkes_get_rates call. */
int hawkes_set_locations(hawkes_ctx* ctx, const double* x, int32_t mem);

/* Parameters; see hawkes_params.  Errors: HAWKES_ERR_ARG, HAWKES_ERR_PARAM. */
int hawkes_set_params(hawkes_ctx* ctx, const hawkes_params* p);

/* ell (Eq. 1) into *out_loglik (host).  -INFINITY with HAWKES_OK when some lambda_n = 0
 * (a distinguished value, reading R11).  Needs all three set_* calls (HAWKES_ERR_STATE).
 * With world > 1 every rank gets the same value. */
int hawkes_loglik(hawkes_ctx* ctx, double* out_loglik);

/* d ell / d x (App. A) for all N events into out_grad (N*D, row-major, host or device per
 * mem; with world > 1 every rank receives the full N*D array); ell into *out_loglik when
 * non-NULL.  A preceding hawkes_loglik with unchanged x and Theta is reused.
 * Errors: as hawkes_loglik, plus HAWKES_ERR_GRAD_UNDEFINED when ell = -inf. */
int hawkes_grad_locations(hawkes_ctx* ctx, double* out_grad, int32_t mem, double* out_loglik);

/* ell and d ell / d x (Eq. 1, App. A: P:L96-101) at new locations in one call: the
 * same results as hawkes_set_locations(ctx, x, HAWKES_MEM_DEVICE) followed by
 * hawkes_grad_locations(ctx, out_grad, HAWKES_MEM_DEVICE, out_loglik), bit for bit.  x
 * (N*D, row-major) and out_grad (N*D) are DEVICE arrays; x is read (and copied) by the call's
 * first kernel, so the caller may overwrite it once the call has returned.  The small-catalog
 * path (the paper's N ~ 3-5k evaluated millions of times): once the constants have
 * been used for two evaluations (W = 1, the unordered-pair algorithm, timing off) the packing,
 * both passes and both finalizes run as ONE CUDA-graph launch whose first and last nodes take
 * x and out_grad (no separate packing launch, no gradient copy); otherwise the two calls above
 * are made.  Errors: as hawkes_set_locations (device input) and hawkes_grad_locations;
 * HAWKES_ERR_STATE without set_times and set_params. */
int hawkes_grad_at(hawkes_ctx* ctx, const double* x, double* out_grad, double* out_loglik);

/* HMC leapfrog over X (potential U = -ell): starting from (x, p), n_steps steps
 *   p += (step/2) grad ell(x);  x += step * Minv * p;  [reflect into [box_lo, box_hi]];
 *   p += (step/2) grad ell(x)
 * x and p (N*D each, host or device per mem) are read and overwritten with the end state.
 * inv_mass_diag (N*D, same memory kind) may be NULL (identity mass).  box_lo/box_hi
 * (N*D, same memory kind) may both be NULL (no box); when given, a coordinate leaving the
 * box is reflected back (x <- 2 bound - x) and its momentum negated.  On return
 * *out_loglik_end = ell(x_end) and *out_kinetic_end = 1/2 sum Minv p^2 (host doubles,
 * each nullable).  The caller does the Metropolis accept/reject.
 * Errors: as hawkes_grad_locations (HAWKES_ERR_GRAD_UNDEFINED aborts the trajectory). */
int hawkes_leapfrog(hawkes_ctx* ctx, double* x, double* p, int32_t mem, double step,
                    int32_t n_steps, const double* inv_mass_diag, const double* box_lo,
                    const double* box_hi, double* out_loglik_end, double* out_kinetic_end);

/* One HMC transition over X (Neal 2011, "MCMC using Hamiltonian dynamics") from the
 * context's current locations x0, every random number drawn on the device:
 *   p0 = Minv^{-1/2} z, z_e ~ N(0,1) for element e (row-major N*D) = Box-Muller of the two
 *       53-bit uniforms u1 = words (0,1), u2 = words (2,3) of the Philox-4x32-10 block
 *       (Salmon et al. 2011) with counter (it_lo, it_hi, e/2, 0) and key (seed_lo, seed_hi):
 *       z_{2q} = sqrt(-2 log u1) cos(2 pi u2), z_{2q+1} = sqrt(-2 log u1) sin(2 pi u2),
 *       u = ((w_a >> 5) 2^26 + (w_b >> 6) + 1/2) / 2^53;
 *   (x1, p1) = hawkes_leapfrog's trajectory (n_steps, step, inv_mass_diag, box) from (x0, p0);
 *   accept iff log u < log alpha = H(x0, p0) - H(x1, p1), H = U + 1/2 sum Minv p^2 with U the
 *       potential of hawkes_set_potential, u from the block with counter
 *       (it_lo, it_hi, 0xffffffff, 1), words (0,1).
 * A trajectory that leaves the support (ell = -inf) or diverges (|x| > 1e100, NaN) has
 * log alpha = -inf and is rejected (not an error).  The chain's state becomes x1 (accepted;
 * its rates and gradient stay cached, so the next step's first gradient is free) or stays
 * x0.  The random stream depends on (seed, iteration) only: the same transition for any
 * world size.  inv_mass_diag (> 0), box_lo, box_hi: as hawkes_leapfrog, host or device per
 * mem, nullable.  x_out (nullable, N*D per mem) receives the new state; *out_accepted
 * (0/1) and *out_log_alpha are host, nullable.  One host synchronisation per call.
 * Errors: HAWKES_ERR_ARG, HAWKES_ERR_STATE, HAWKES_ERR_GRAD_UNDEFINED (ell(x0) = -inf). */
int hawkes_hmc_step(hawkes_ctx* ctx, uint64_t seed, uint64_t iteration, double step,
                    int32_t n_steps, const double* inv_mass_diag, const double* box_lo,
                    const double* box_hi, int32_t mem, double* x_out, int32_t* out_accepted,
                    double* out_log_alpha);

/* The context's current locations (N*D row-major, host or device per mem): those of the
 * last set_locations, leapfrog, accepted move / HMC transition / MH sweep.
 * Errors: HAWKES_ERR_ARG, HAWKES_ERR_STATE (no locations). */
int hawkes_get_locations(hawkes_ctx* ctx, double* out_x, int32_t mem);

/* Per-event quantities of the last evaluation (computing it if needed): lambda_n,
 * mu_n = sum_n' mu_nn', xi_n = sum_n' xi_nn' and Lambda_n; each pointer nullable, length N,
 * host or device per mem.  Full length on every rank. */
int hawkes_get_rates(hawkes_ctx* ctx, double* lambda, double* mu, double* xi, double* Lambda,
                     int32_t mem);

/* The pair-kernel precision this context evaluates with now (*out: hawkes_precision).
 * An HAWKES_FP32 context reports HAWKES_FP64 after its range guard tripped (DESIGN.md
 * reading R23): when some event's rate Lambda' falls within 2^24 N flush quanta of the fp32
 * flush threshold (terms ex2.approx.ftz sets to 0 could then carry more than 2^-24 of it),
 * the call that saw it is redone by the fp64 kernels -- hawkes_loglik,
 * hawkes_grad_locations, hawkes_get_rates, hawkes_leapfrog and hawkes_hmc_step return the
 * fp64 result; block moves and MH sweeps check the guard before using fresh rates -- and
 * the context stays on fp64 until the next hawkes_set_times / hawkes_set_params.
 * Errors: HAWKES_ERR_ARG. */
int hawkes_precision_in_use(const hawkes_ctx* ctx, int32_t* out);

/* Walk order (hawkes_ordering) of the PAIRS fp64 kernels; takes effect at the next
 * evaluation (the permutation is built then from its locations).  hawkes_ordering_in_use
 * writes the order the last evaluation used (HAWKES_ORDER_TIME or _SPACE) and, when
 * out_cost is non-NULL, the decision's two work estimates (time, space; 0 if not estimated).
 * Errors: HAWKES_ERR_ARG. */
int hawkes_set_ordering(hawkes_ctx* ctx, int32_t mode);
int hawkes_ordering_in_use(const hawkes_ctx* ctx, int32_t* out, double* out_cost);

/* Bayesian MDS: the flu application's second O(N^2)
 * term.  hawkes_set_bmds copies the N*N row-major dissimilarity matrix Y (host or device per
 * mem; only the lower triangle y[n*N + n'], n > n', is read, as in Eq. bmdsLikelihood) and
 * sigma > 0 (the paper's mdsSD).  Every y_{nn'} (n > n') must be finite and > 0 (the
 * truncated-normal support), else HAWKES_ERR_NONFINITE (host input: now; device input: at
 * the next evaluation).  The context then holds 8 N^2 bytes of device memory for Y plus
 * 8 (ceil(N/32) + 1) N (D + 1) bytes of per-block partial sums (the unordered-pair kernel).
 * hawkes_bmds_logdensity writes
 *   log p(Y | X) = sum_{n > n'} [-1/2 log(2 pi sigma^2) - (y - delta)^2/(2 sigma^2)
 *                                - log Phi(delta/sigma)],   delta = |x_n - x_n'|
 * (Eq. bmdsLikelihood with the normal constant kept) to *out_logp and, when out_grad is
 * non-NULL, its gradient in x (N*D, host or device per mem) at the context's current
 * locations.  A coincident pair (delta = 0) contributes no gradient (reading R25).
 * Errors: HAWKES_ERR_ARG, HAWKES_ERR_PARAM (sigma), HAWKES_ERR_STATE (no Y / no x). */
int hawkes_set_bmds(hawkes_ctx* ctx, const double* Y, int32_t mem, double sigma);
int hawkes_bmds_logdensity(hawkes_ctx* ctx, double* out_grad, int32_t mem, double* out_logp);

/* Which log densities hawkes_leapfrog's potential U = -(sum) includes: a bit mask of
 * HAWKES_POTENTIAL_HAWKES (ell, the default) and HAWKES_POTENTIAL_BMDS (log p(Y | X));
 * both = the flu model's HMC over X.  out_loglik_end then reports the sum. */
typedef enum { HAWKES_POTENTIAL_HAWKES = 1, HAWKES_POTENTIAL_BMDS = 2 } hawkes_potential;
int hawkes_set_potential(hawkes_ctx* ctx, int32_t flags);

/* Block Metropolis-Hastings over locations.
 * hawkes_propose_move returns in *out_delta = ell(X') - ell(X) for X' = X with the k events
 * idx[0..k) (host array, distinct, 1 <= k <= 256) moved to new_x (k*D row-major, host or
 * device per mem).  Lambda_n does not depend on x, so only the lambda_n change: the cost is
 * O(k N) given the rates of the current state, which are computed on demand (one full
 * evaluation) and then kept up to date by hawkes_accept_move.  The proposal stays pending
 * until hawkes_accept_move commits it (the context's locations and cached rates become
 * those of X'), or until another proposal, set_* or leapfrog call discards it.  IEEE
 * semantics: -inf when some lambda_n' = 0.  Accepted moves update the cached rates
 * incrementally; a hawkes_loglik / hawkes_grad_locations call recomputes everything.
 * Errors: HAWKES_ERR_ARG, HAWKES_ERR_NONFINITE, HAWKES_ERR_STATE. */
int hawkes_propose_move(hawkes_ctx* ctx, int32_t k, const int32_t* idx, const double* new_x,
                        int32_t mem, double* out_delta);
int hawkes_accept_move(hawkes_ctx* ctx);

/* Coarsening regions: the uniform location priors of the DC and Alaska models, which the
 * block MH sweep samples under.  kind HAWKES_REGION_SQUARE: |x_nd - centre_nd| < size_n for
 * every d (Eq. locsPrior1, size = the 50 m half-width); HAWKES_REGION_DISC:
 * |x_n - centre_n|_2 < size_n (Eq. locsPrior2, size = r_n; D = 2 only, else
 * HAWKES_ERR_DIM).  centre (N*D row-major) and size (N) are copied (host or device per
 * mem).  The context's locations should lie inside their regions (prior support).
 * Errors: HAWKES_ERR_ARG, HAWKES_ERR_DIM, HAWKES_ERR_NONFINITE (size <= 0 or non-finite). */
typedef enum { HAWKES_REGION_SQUARE = 1, HAWKES_REGION_DISC = 2 } hawkes_region;
int hawkes_set_regions(hawkes_ctx* ctx, int32_t kind, const double* centre, const double* size,
                       int32_t mem);

/* On-device block Metropolis-Hastings sweep over locations: n_blocks
 * sequential updates; block b moves the k distinct events blocks[b*k .. b*k+k) (host
 * int32, 1 <= k <= 256) jointly:
 *   square regions: x*_nd = x_nd + s z, z ~ N(0,1) truncated to the region by inverting its
 *     CDF, s = scale * size_n; log Hastings sum_d log Z_d(x) - log Z_d(x*), Z_d = the
 *     N(x_nd, s^2) mass of the region's interval ("truncated normal proposals");
 *   disc regions: x* uniform on disc(centre_n, r_n) cap disc(x_n, scale r_n) (Eq.
 *     circleKernel, eps = scale) by rejection (at most 4096 attempts, else x* = x); log
 *     Hastings log A(x) - log A(x*), A the closed-form lens area;
 *   log alpha = [ell(X') - ell(X)] + sum of the block's log Hastings terms (the uniform priors
 *     cancel), ell(X') - ell(X) by the O(kN) update of hawkes_propose_move;
 *   accept iff log u < log alpha; an accepted block updates the locations and cached rates.
 * Random numbers: Philox-4x32-10 (as hawkes_hmc_step) with counter (it_lo, it_hi, b, tag),
 * key (seed_lo, seed_hi): slot q's draws use tag 0x80000000 | q << 12 | a (a = dimension pair
 * for squares, attempt for discs), the accept uniform tag 0xC0000000; each block gives two
 * 53-bit uniforms (words 0,1 and 2,3).  The whole sweep runs on the device with one host
 * synchronisation at the end.  out_accepted (n_blocks int32), out_log_alpha (n_blocks
 * double), out_n_accepted: host, nullable.
 * Errors: HAWKES_ERR_ARG, HAWKES_ERR_STATE (no regions / set_* missing). */
int hawkes_mh_sweep(hawkes_ctx* ctx, int32_t n_blocks, int32_t k, const int32_t* blocks,
                    double scale, uint64_t seed, uint64_t iteration, int32_t* out_accepted,
                    double* out_log_alpha, int32_t* out_n_accepted);

/* Kernel timing (CUDA events on the context stream around each launch of the two O(N^2)
 * pass kernels).  enable != 0 starts accumulating from zero.  hawkes_get_kernel_times
 * synchronises and returns the summed milliseconds and launch counts since enabling;
 * any pointer may be NULL. */
int hawkes_enable_timing(hawkes_ctx* ctx, int32_t enable);
int hawkes_get_kernel_times(hawkes_ctx* ctx, double* rate_ms, int64_t* rate_launches,
                            double* grad_ms, int64_t* grad_launches, int64_t* total_launches);

/* Rank 0 of a multi-process run calls this to obtain the 128-byte ncclUniqueId that every
 * rank then passes as opts.nccl_unique_id (the caller distributes it, e.g. with a
 * torch.distributed broadcast).  out must hold 128 bytes.  Errors: HAWKES_ERR_NCCL. */
int hawkes_nccl_unique_id(void* out);

/* Row-sharding plan (host only; no device needed): the row tiles rank `rank` of `world`
 * owns for N events, dealt zig-zag (tile k of each group of 2*world goes to rank k or
 * 2*world-1-k) to balance the causal self-excitation work; the j-chunk length, which
 * depends on N only, so every row's summation order is the same for any world.
 * tiles_out (nullable) receives *n_tiles tile indices; a tile is rows
 * [k*rows_per_tile, min(N, (k+1)*rows_per_tile)).  Pass tiles_out = NULL to query
 * *n_tiles first.  Errors: HAWKES_ERR_ARG. */
int hawkes_plan(int64_t N, int32_t world, int32_t rank, int32_t* tiles_out, int32_t* n_tiles,
                int32_t* rows_per_tile, int32_t* chunk);

/* Work plan of HAWKES_ALGO_PAIRS (host only): the chunk length (a function of N only) and
 * the chunk pairs (a, b), a <= b, that rank `rank` of `world` evaluates (a == b: the pairs
 * inside chunk a).  items_out (nullable) receives 2 * *n_items int32 (a, b).  Chunk pairs
 * are dealt to ranks by greedy longest-processing-time on their pair counts.
 * Errors: HAWKES_ERR_ARG. */
int hawkes_plan_pairs(int64_t N, int32_t world, int32_t rank, int32_t* items_out,
                      int32_t* n_items, int32_t* chunk);

/* Spatial walk order of the PAIRS kernels (host only, the logic hawkes_ordering AUTO uses):
 * perm_out (nullable, N) receives the walk (Hilbert order of the locations for D = 2, Morton
 * for other D), cost_out (nullable, 2) the work estimates of the time and the spatial walk
 * (live (tile pair, term) counts from the tiles' bounding boxes under Theta; AUTO takes the
 * spatial walk when cost_out[1] < 0.9 cost_out[0]).  x: N*D row-major, t: N non-decreasing.
 * Errors: HAWKES_ERR_ARG. */
int hawkes_plan_walk(const double* x, const double* t, int64_t N, int32_t D, const hawkes_params* p,
                     int32_t* perm_out, double* cost_out);

/* Partial-slot footprint of HAWKES_ALGO_PAIRS on one rank (host only): the events of the
 * compact, item-indexed slot blocks rank `rank` of `world` allocates (one block of chunk
 * events per (chunk, slot id) its chunk pairs write; device memory = slot_events * 8 *
 * (2 + K2) bytes), and in *max_events (nullable) the largest over all ranks.  At world = 1
 * it is (C + 1) C chunk; the ranks together hold the same blocks, so each holds ~1/world.
 * Errors: HAWKES_ERR_ARG. */
int hawkes_plan_slots(int64_t N, int32_t world, int32_t rank, int64_t* slot_events, int64_t* max_events);

/* Work items of HAWKES_ALGO_PAIRS on one rank as the device launches them (host only): the
 * chunk pairs of hawkes_plan_pairs in the kernels' order (heaviest first), each as one item
 * or, when the rank's n items fill less than one round of `resident` CTA slots (the gradient
 * pass's resident grid; 0 = whole items), as k pieces over the skewed-step ranges
 * [32q/k, 32(q+1)/k) (k the largest of 8, 4, 2 with k n <= resident), every piece with its own
 * row and column slot blocks (DESIGN.md §5 "Small N").  items_out (nullable; n_items x 6 int64,
 * row-major): a, b, row-block event offset, column-block event offset, s0, s1 into this
 * rank's slot array of *slot_events events; *pieces receives k (1: whole items).  Call with
 * items_out = NULL for the count.  Errors: HAWKES_ERR_ARG. */
int hawkes_plan_items(int64_t N, int32_t world, int32_t rank, int32_t resident, int64_t* items_out,
                      int32_t* n_items, int32_t* pieces, int64_t* slot_events);

/* Diagnostics (not part of the numerical contract; used by the tests and bench.py):
 * hawkes_diag_exp evaluates the kernels' fast exp on n device doubles; hawkes_diag_fp64_peak
 * measures the device's dependent-DFMA throughput in FP64 lane-ops per second. */
int hawkes_diag_exp(const double* a_dev, double* out_dev, int64_t n);
/* the standard normals z_0..z_{n-1} hawkes_hmc_step draws for (seed, iteration), into n
 * device doubles (tests pin the device Philox stream against the oracle's) */
int hawkes_diag_normals(uint64_t seed, uint64_t iteration, double* out_dev, int64_t n);
int hawkes_diag_fp64_peak(double* ops_per_s);
/* FP64 operand-pattern probe (mode 0: DFMA reg,imm,imm; 1: DFMA with 3 register operands;
 * 2: DADD; 3: DMUL; 4: the kernels' fast exp; 5: DFMA reg,reg,imm) at warps_per_sm resident
 * warps: chain-steps per second over the device (x1 op each; the exp is 9 FP64 ops). */
int hawkes_diag_fp64_mode(int32_t mode, int32_t warps_per_sm, double* iters_per_s);

/* One-line description of the last failure on ctx (or of the last failed create when
 * ctx is NULL).  The string is owned by the library. */
const char* hawkes_last_error(const hawkes_ctx* ctx);

/* HAWKES_ABI_VERSION. */
int hawkes_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HAWKES_B200_H */
