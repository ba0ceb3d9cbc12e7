/*
 * hawkes_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU evaluation of the spatiotemporal Hawkes
 * log-likelihood of Holbrook, Ji & Suchard (arXiv 2010.02994) and of its
 * gradient with respect to event locations.  It exists to check the CUDA path
 * (paper_2010_02994_b200/csrc) and to be timed as the CPU baseline.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  It shares no source, header, constant or
 * helper with the CUDA path, and the CUDA path never calls it.
 *
 * Citations are to /root/reference/PAPER.md as P:L<line>.
 *
 *   mu_{nn'}  = mu0/(tau_x^D tau_t) phi_D((x_n-x_n')/tau_x) phi((t_n-t_n')/tau_t) I[t_n != t_n']
 *               -- background kernel smoother, Sec. 2.1, and Eq. 1
 *   xi_{nn'}  = theta*omega/h^D exp(-omega (t_n-t_n')) phi_D((x_n-x_n')/h) I[t_n' < t_n]
 *               -- triggering function, Sec. 2.1, and Eq. 1
 *   lambda_n  = sum_{n'=1..N} (mu_{nn'} + xi_{nn'})                       -- Eq. 1; App. A
 *   Lambda_n  = mu0 (Phi((t_N-t_n)/tau_t) - Phi(-t_n/tau_t))
 *               - theta (exp(-omega (t_N-t_n)) - 1)                        -- P:L92-93
 *   ell       = sum_n (log lambda_n - Lambda_n)                            -- Eq. 1
 *   d ell/d x_n = sum_{n'} [(mu_{nn'}/lambda_n + mu_{n'n}/lambda_{n'}) (x_n'-x_n)/tau_x^2
 *                          + (xi_{nn'}/lambda_n + xi_{n'n}/lambda_{n'}) (x_n'-x_n)/h^2]
 *               -- App. A display, with the paper's sigma_x read as h
 *                  (reading R2).
 *
 * phi_D is the D-variate standard normal density (2 pi)^(-D/2) exp(-|u|^2/2)
 * (reading R1), phi = phi_1, Phi the standard normal CDF.
 *
 * Arithmetic: IEEE double, glibc exp/log/erfc, every pair term evaluated
 * literally and separately, row sums by Neumaier compensated summation,
 * rows in parallel with OpenMP (rows are independent, so the result does not
 * depend on the thread count).  Build with -O2 -ffp-contract=off, no
 * -ffast-math (oracle/__init__.py does this).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define ORACLE_OK 0
#define ORACLE_ERR_ARG (-1)
#define ORACLE_ERR_UNSORTED (-3)

typedef struct {
  double mu0, tau_x, tau_t, theta, omega, h; /* Theta in the paper's order */
} oracle_params;

/* ---- compensated summation (Neumaier) ---------------------------------- */
typedef struct { double s, c; } nsum;

static void nsum_add(nsum* a, double v) {
  double t = a->s + v;
  if (fabs(a->s) >= fabs(v))
    a->c += (a->s - t) + v;
  else
    a->c += (v - t) + a->s;
  a->s = t;
}
static double nsum_get(const nsum* a) { return a->s + a->c; }

/* ---- densities ---------------------------------------------------------- */
static const double ORACLE_PI = 3.14159265358979323846264338327950288;

/* standard normal density phi(z) */
static double phi1(double z) { return exp(-0.5 * z * z) / sqrt(2.0 * ORACLE_PI); }

/* D-variate standard normal density phi_D(u), u = (a - b)/s componentwise */
static double phiD_scaled(const double* a, const double* b, int D, double s) {
  double q = 0.0;
  for (int d = 0; d < D; ++d) {
    double u = (a[d] - b[d]) / s;
    q += u * u;
  }
  return exp(-0.5 * q) / pow(2.0 * ORACLE_PI, 0.5 * D);
}

/* standard normal CDF */
static double Phi(double z) { return 0.5 * erfc(-z / sqrt(2.0)); }

/* ---- pair terms, P:L98-99 ----------------------------------------------- */
double oracle_mu_pair(int D, const double* x, const double* t, long n, long m,
                      const oracle_params* p) {
  if (t[n] == t[m]) return 0.0; /* I[t_n != t_n'] */
  return p->mu0 / (pow(p->tau_x, D) * p->tau_t) *
         phiD_scaled(x + n * D, x + m * D, D, p->tau_x) *
         phi1((t[n] - t[m]) / p->tau_t);
}

double oracle_xi_pair(int D, const double* x, const double* t, long n, long m,
                      const oracle_params* p) {
  if (!(t[m] < t[n])) return 0.0; /* I[t_n' < t_n] */
  return p->theta * p->omega / pow(p->h, D) * exp(-p->omega * (t[n] - t[m])) *
         phiD_scaled(x + n * D, x + m * D, D, p->h);
}

static int check_sorted(long N, const double* t) {
  for (long n = 1; n < N; ++n)
    if (t[n] < t[n - 1]) return ORACLE_ERR_UNSORTED;
  return ORACLE_OK;
}

/* ---- rates: lambda_n, and its two parts, for rows [row0, row1) ---------- */
int oracle_rates(long N, int D, const double* x, const double* t, const oracle_params* p,
                 long row0, long row1, double* lambda, double* mu_out, double* xi_out) {
  if (N < 0 || D < 1 || row0 < 0 || row1 > N || row0 > row1) return ORACLE_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 8)
  for (long n = row0; n < row1; ++n) {
    nsum lam = {0, 0}, mus = {0, 0}, xis = {0, 0};
    for (long m = 0; m < N; ++m) { /* n' = n included: zero by both indicators */
      double mu = oracle_mu_pair(D, x, t, n, m, p);
      double xi = oracle_xi_pair(D, x, t, n, m, p);
      nsum_add(&mus, mu);
      nsum_add(&xis, xi);
      nsum_add(&lam, mu);
      nsum_add(&lam, xi);
    }
    if (lambda) lambda[n] = nsum_get(&lam);
    if (mu_out) mu_out[n] = nsum_get(&mus);
    if (xi_out) xi_out[n] = nsum_get(&xis);
  }
  return ORACLE_OK;
}

/* ---- Lambda_n, P:L92-93 (t_N = last time of the sorted catalog) --------- */
int oracle_Lambda(long N, const double* t, const oracle_params* p, double* Lambda) {
  if (N < 1) return ORACLE_ERR_ARG;
  if (check_sorted(N, t)) return ORACLE_ERR_UNSORTED;
  double tN = t[N - 1];
  for (long n = 0; n < N; ++n)
    Lambda[n] = p->mu0 * (Phi((tN - t[n]) / p->tau_t) - Phi(-t[n] / p->tau_t)) -
                p->theta * (exp(-p->omega * (tN - t[n])) - 1.0);
  return ORACLE_OK;
}

/* ---- ell, Eq. 1 ----------------------------------------------------------
 * lambda_out / Lambda_out (length N, nullable) receive lambda_n and Lambda_n.
 * ell = -inf when some lambda_n = 0 (log 0).                               */
int oracle_loglik(long N, int D, const double* x, const double* t, const oracle_params* p,
                  double* ell, double* lambda_out, double* Lambda_out) {
  if (N < 1 || D < 1) return ORACLE_ERR_ARG;
  if (check_sorted(N, t)) return ORACLE_ERR_UNSORTED;
  double* lam = lambda_out ? lambda_out : (double*)malloc(sizeof(double) * N);
  double* Lam = Lambda_out ? Lambda_out : (double*)malloc(sizeof(double) * N);
  oracle_rates(N, D, x, t, p, 0, N, lam, NULL, NULL);
  oracle_Lambda(N, t, p, Lam);
  nsum acc = {0, 0};
  int zero = 0;
  for (long n = 0; n < N; ++n) {
    if (lam[n] == 0.0) zero = 1;
    nsum_add(&acc, log(lam[n]) - Lam[n]);
  }
  *ell = zero ? -INFINITY : nsum_get(&acc);
  if (!lambda_out) free(lam);
  if (!Lambda_out) free(Lam);
  return ORACLE_OK;
}

/* ---- gradient, App. A, rows [row0, row1) ---------------------------
 * lambda: all N rates (from oracle_rates).  grad, scale: N*D row-major,
 * written for rows in range.  scale[n,d] = sum_{n'} |c_{nn'} (x_{n'd}-x_{nd})|,
 * the conditioning scale of component (n,d) used by the parity tolerance. */
int oracle_grad(long N, int D, const double* x, const double* t, const oracle_params* p,
                const double* lambda, long row0, long row1, double* grad, double* scale) {
  if (N < 0 || D < 1 || row0 < 0 || row1 > N || row0 > row1) return ORACLE_ERR_ARG;
  const double tx2 = p->tau_x * p->tau_x, h2 = p->h * p->h;
#pragma omp parallel for schedule(dynamic, 8)
  for (long n = row0; n < row1; ++n) {
    nsum g[16];
    nsum s[16];
    for (int d = 0; d < D; ++d) { g[d].s = g[d].c = 0; s[d].s = s[d].c = 0; }
    for (long m = 0; m < N; ++m) {
      double mu_nm = oracle_mu_pair(D, x, t, n, m, p);
      double mu_mn = oracle_mu_pair(D, x, t, m, n, p);
      double xi_nm = oracle_xi_pair(D, x, t, n, m, p);
      double xi_mn = oracle_xi_pair(D, x, t, m, n, p);
      double cb = mu_nm / lambda[n] + mu_mn / lambda[m];
      double cs = xi_nm / lambda[n] + xi_mn / lambda[m];
      for (int d = 0; d < D; ++d) {
        double dx = x[m * D + d] - x[n * D + d];
        double term = cb * (dx / tx2) + cs * (dx / h2);
        nsum_add(&g[d], term);
        nsum_add(&s[d], fabs(cb * (dx / tx2)) + fabs(cs * (dx / h2)));
      }
    }
    for (int d = 0; d < D; ++d) {
      grad[n * D + d] = nsum_get(&g[d]);
      if (scale) scale[n * D + d] = nsum_get(&s[d]);
    }
  }
  return ORACLE_OK;
}

/* ---- complex-step form of ell (x = x_re + i x_im; t, Theta real) ----------
 * ell is analytic in x (|u|^2 = sum u_d^2, no abs; indicators depend on t
 * only), so d ell/d x . V = Im ell(X + i eps V) / eps for tiny eps.         */
static double complex phiD_scaled_c(const double* are, const double* aim, const double* bre,
                                    const double* bim, int D, double s) {
  double complex q = 0.0;
  for (int d = 0; d < D; ++d) {
    double complex u = ((are[d] - bre[d]) + I * (aim[d] - bim[d])) / s;
    q += u * u;
  }
  return cexp(-0.5 * q) / pow(2.0 * ORACLE_PI, 0.5 * D);
}

int oracle_loglik_complex(long N, int D, const double* x_re, const double* x_im,
                          const double* t, const oracle_params* p, double* ell_re,
                          double* ell_im) {
  if (N < 1 || D < 1 || D > 16) return ORACLE_ERR_ARG;
  if (check_sorted(N, t)) return ORACLE_ERR_UNSORTED;
  double* Lam = (double*)malloc(sizeof(double) * N);
  double* lre = (double*)malloc(sizeof(double) * N);
  double* lim = (double*)malloc(sizeof(double) * N);
  oracle_Lambda(N, t, p, Lam);
#pragma omp parallel for schedule(dynamic, 8)
  for (long n = 0; n < N; ++n) {
    double complex lam = 0.0;
    for (long m = 0; m < N; ++m) {
      if (t[n] != t[m])
        lam += p->mu0 / (pow(p->tau_x, D) * p->tau_t) *
               phiD_scaled_c(x_re + n * D, x_im + n * D, x_re + m * D, x_im + m * D, D, p->tau_x) *
               phi1((t[n] - t[m]) / p->tau_t);
      if (t[m] < t[n])
        lam += p->theta * p->omega / pow(p->h, D) * exp(-p->omega * (t[n] - t[m])) *
               phiD_scaled_c(x_re + n * D, x_im + n * D, x_re + m * D, x_im + m * D, D, p->h);
    }
    double complex l = clog(lam);
    lre[n] = creal(l) - Lam[n];
    lim[n] = cimag(l);
  }
  nsum a = {0, 0}, b = {0, 0};
  for (long n = 0; n < N; ++n) { nsum_add(&a, lre[n]); nsum_add(&b, lim[n]); }
  *ell_re = nsum_get(&a);
  *ell_im = nsum_get(&b);
  free(Lam); free(lre); free(lim);
  return ORACLE_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---- BMDS (Eq. bmdsLikelihood) -------------------------------
 * Observed dissimilarities y_{nn'} ~ N(delta_{nn'}, sigma^2) I[y > 0], n > n',
 * delta_{nn'} = |x_n - x_n'|_2.  The log density of Y given X is
 *   log p = sum_{n > n'} [ -1/2 log(2 pi sigma^2) - (y - delta)^2/(2 sigma^2)
 *                          - log Phi(delta/sigma) ]
 * i.e. Eq. bmdsLikelihood (which writes it up to the 2 pi factor) with the
 * normal density's constant kept.  Y is N*N row-major; only n > n' is read.
 * Gradient (derived here by hand, parity checked against finite differences and a
 * 40-digit brute force in the tests):
 *   d log p / d x_n = - sum_{n' != n} dr/d delta * (x_n - x_n')/delta,
 *   dr/d delta = -(y - delta)/sigma^2 + phi(delta/sigma) / (sigma Phi(delta/sigma)),
 * with y = y_{max(n,n') min(n,n')}; a coincident pair (delta = 0) contributes 0.       */
double oracle_bmds_pair(double y, double delta, double sigma) {
  double z = delta / sigma;
  return 0.5 * log(2.0 * ORACLE_PI * sigma * sigma) +
         (y - delta) * (y - delta) / (2.0 * sigma * sigma) + log(Phi(z));
}

int oracle_bmds(long N, int D, const double* x, const double* Y, double sigma, double* logp,
                double* grad, double* scale) {
  if (N < 1 || D < 1 || !(sigma > 0)) return ORACLE_ERR_ARG;
  double* rows = (double*)malloc(sizeof(double) * N);
#pragma omp parallel for schedule(dynamic, 8)
  for (long n = 0; n < N; ++n) {
    nsum lp = {0, 0};
    nsum g[16], sc[16];
    for (int d = 0; d < D; ++d) g[d].s = g[d].c = sc[d].s = sc[d].c = 0;
    for (long m = 0; m < N; ++m) {
      if (m == n) continue;
      double r2 = 0.0;
      for (int d = 0; d < D; ++d) {
        double u = x[n * D + d] - x[m * D + d];
        r2 += u * u;
      }
      double delta = sqrt(r2);
      double y = n > m ? Y[n * N + m] : Y[m * N + n];
      if (m < n) nsum_add(&lp, -oracle_bmds_pair(y, delta, sigma)); /* each pair once */
      if (grad && delta > 0.0) {
        double z = delta / sigma;
        double drdd = -(y - delta) / (sigma * sigma) + phi1(z) / (sigma * Phi(z));
        for (int d = 0; d < D; ++d) {
          double term = -drdd * (x[n * D + d] - x[m * D + d]) / delta;
          nsum_add(&g[d], term);
          nsum_add(&sc[d], fabs(term));
        }
      }
    }
    rows[n] = nsum_get(&lp);
    for (int d = 0; d < D; ++d) {
      if (grad) grad[n * D + d] = nsum_get(&g[d]);
      if (scale) scale[n * D + d] = nsum_get(&sc[d]);
    }
  }
  nsum tot = {0, 0};
  for (long n = 0; n < N; ++n) nsum_add(&tot, rows[n]);
  *logp = nsum_get(&tot);
  free(rows);
  return ORACLE_OK;
}

/* ---- HMC transition (Neal 2011) with counter-based random numbers ----------
 * Philox-4x32-10 (Salmon et al. 2011, "Parallel random numbers: as easy as 1, 2, 3"):
 * 10 rounds of (L, R) <- (mulhi(R0,M0) ^ k0 ^ R1, lo(R0 M0), ...) with the Weyl key
 * schedule.  The HMC step draws, for momentum element e (row-major N*D) and iteration it,
 * one block with counter (it_lo, it_hi, e/2, 0) and key (seed_lo, seed_hi); two 53-bit
 * uniforms from its four words, and Box-Muller gives the normals of elements 2q, 2q+1.
 * The accept uniform uses counter (it_lo, it_hi, 0xffffffff, 1).                      */
static void philox_round(uint32_t* c, const uint32_t* k) {
  const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
  const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
  const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  const uint32_t n0 = hi1 ^ c[1] ^ k[0];
  const uint32_t n2 = hi0 ^ c[3] ^ k[1];
  c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
}

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int r = 0; r < 10; ++r) {
    philox_round(c, k);
    k[0] += 0x9E3779B9u;
    k[1] += 0xBB67AE85u;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

static double u53(uint32_t a, uint32_t b) {   /* (0, 1), 53 bits */
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6) + 0.5) / 9007199254740992.0;
}

void oracle_hmc_normals(uint64_t seed, uint64_t it, long n, double* z) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  for (long q = 0; 2 * q < n; ++q) {
    const uint32_t ctr[4] = {(uint32_t)it, (uint32_t)(it >> 32), (uint32_t)q, 0u};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    const double u1 = u53(w[0], w[1]), u2 = u53(w[2], w[3]);
    const double rad = sqrt(-2.0 * log(u1)), ang = 2.0 * ORACLE_PI * u2;
    z[2 * q] = rad * cos(ang);
    if (2 * q + 1 < n) z[2 * q + 1] = rad * sin(ang);
  }
}

double oracle_hmc_uniform(uint64_t seed, uint64_t it) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const uint32_t ctr[4] = {(uint32_t)it, (uint32_t)(it >> 32), 0xffffffffu, 1u};
  uint32_t w[4];
  oracle_philox4x32_10(ctr, key, w);
  return u53(w[0], w[1]);
}
