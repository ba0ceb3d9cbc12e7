"""Pins of the CPU oracle against things other than itself (no GPU needed).

Each test names the passage of PAPER.md (P:L<line>) it checks and what would
fail if the oracle had a plausible mistake:

  closed forms at N=2 (hand-derived)       -> wrong normalisation, indicator, sign, sigma_x reading
  N=3 structure of App. A                  -> transposed operand / wrong lambda in the cross term
  40-digit brute force + mp.diff gradient  -> rounding / summation / indexing, App. A vs d ell/dx
  complex step, finite differences         -> App. A gradient vs Eq. 1
  quadrature of the intensity              -> Lambda_n closed form and phi_D normalisation
  sklearn leave-one-out KDE (theta = 0)    -> background smoother of P:L82
  invariances, ties, N=1, t_n = t_N        -> indicators, dependence on differences only
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
import synth
from tests import mp_brute

pytestmark = pytest.mark.filterwarnings("ignore::DeprecationWarning")


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


def _mp_eval(expr):
    with mp.workdps(40):
        env = {"exp": mp.exp, "pi": mp.pi, "Phi": mp.ncdf}
        return eval(expr.replace("1/", "mp.mpf(1)/"), {"mp": mp, **env})


# ---------------------------------------------------------------- closed forms
def test_p1_closed_form_n2(golden_dir):
    """P1: N=2 closed forms (Eq. 1, Lambda P:L92-93, App. A)."""
    g = _load(golden_dir, "p1_n2.json")
    x, t, th = np.array(g["x"]), np.array(g["t"]), g["theta"]
    cf = g["closed_form"]
    lam1, lam2 = float(_mp_eval(cf["lambda_1"])), float(_mp_eval(cf["lambda_2"]))
    Lam1, Lam2 = float(_mp_eval(cf["Lambda_1"])), float(_mp_eval(cf["Lambda_2"]))
    ell_ref = math.log(lam1) + math.log(lam2) - Lam1 - Lam2
    xi21 = math.exp(-1.5) / (2 * math.pi)
    c = (1 + lam1 / lam2) / 4 + xi21 / lam2

    ell, lam, Lam = oracle.loglik(x, t, th)
    np.testing.assert_allclose(lam, [lam1, lam2], rtol=2e-15)
    np.testing.assert_allclose(Lam, [Lam1, Lam2], rtol=2e-15)
    assert ell == pytest.approx(ell_ref, rel=2e-15)
    gr, _ = oracle.grad(x, t, th)
    np.testing.assert_allclose(gr, [[c, 0.0], [-c, 0.0]], rtol=2e-15, atol=1e-300)
    # the decomposition into mu and xi
    _, mu, xi = oracle.rates(x, t, th)
    np.testing.assert_allclose(mu, [lam1, lam1], rtol=2e-15)
    np.testing.assert_allclose(xi, [0.0, xi21], rtol=2e-15, atol=0)


def test_p2_structure_n3(golden_dir):
    """P2: App. A's c_nn' is symmetric, so g_2y = g_3x = c_23 and columns sum to 0."""
    g = _load(golden_dir, "p2_n3.json")
    x, t, th = np.array(g["x"]), np.array(g["t"]), g["theta"]
    gr, _ = oracle.grad(x, t, th)
    assert gr[1, 1] == pytest.approx(gr[2, 0], rel=1e-14)
    np.testing.assert_allclose(gr.sum(axis=0), 0.0, atol=1e-14 * np.abs(gr).sum())
    ref = mp_brute.evaluate(g["x"], g["t"], th)
    np.testing.assert_allclose(gr, np.array([[float(v) for v in r] for r in ref["grad"]]), rtol=1e-13)


# --------------------------------------------------------------- brute force
@pytest.mark.parametrize("N,D,seed", [(4, 2, 0), (7, 2, 1), (6, 3, 2), (8, 1, 3)])
def test_brute_force_40_digits(N, D, seed):
    """P3: oracle vs a 40-digit mpmath evaluation; the gradient reference is mp.diff of ell."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(0, 1, size=(N, D))
    t = np.sort(rng.uniform(0, 1, size=N))
    th = (0.7, 0.4, 0.3, 0.5, 3.0, 0.2)
    ref = mp_brute.evaluate(x.tolist(), t.tolist(), th)
    ell, lam, Lam = oracle.loglik(x, t, th)
    np.testing.assert_allclose(lam, [float(v) for v in ref["lam"]], rtol=1e-14)
    np.testing.assert_allclose(Lam, [float(v) for v in ref["Lam"]], rtol=1e-14, atol=1e-16)
    assert ell == pytest.approx(float(ref["ell"]), rel=1e-13)
    gr, S = oracle.grad(x, t, th)
    gref = np.array([[float(v) for v in r] for r in ref["grad"]])
    assert np.all(np.abs(gr - gref) <= 1e-13 * np.maximum(np.abs(gref), S))


# --------------------------------------------------------- derivative checks
def test_complex_step_directional():
    """P4: <g, V> = Im ell(X + i eps V)/eps (ell analytic in X) at N=60."""
    c = synth.unit_square(60, config=11)
    V = np.random.default_rng(5).normal(size=c.x.shape)
    eps = 1e-30
    _, im = oracle.loglik_complex(c.x, eps * V, c.t, c.theta)
    gr, S = oracle.grad(c.x, c.t, c.theta)
    lhs = float(np.sum(gr * V))
    assert abs(lhs - im / eps) <= 1e-12 * float(np.sum(np.abs(S * V)))


def test_complex_step_components():
    """P4 per component: d ell/d x_nd = Im ell(X + i eps e_nd)/eps for sampled (n,d)."""
    c = synth.unit_square(30, config=12)
    gr, S = oracle.grad(c.x, c.t, c.theta)
    eps = 1e-30
    for n, d in [(0, 0), (7, 1), (15, 0), (29, 1)]:
        E = np.zeros_like(c.x)
        E[n, d] = eps
        _, im = oracle.loglik_complex(c.x, E, c.t, c.theta)
        assert abs(gr[n, d] - im / eps) <= 1e-12 * max(abs(gr[n, d]), S[n, d])


def test_finite_differences_spec():
    """P5: central differences, step 1e-5, relative error < 1e-5."""
    for seed in range(5):
        c = synth.unit_square(20, config=13, replicate=seed)
        gr, S = oracle.grad(c.x, c.t, c.theta)
        h = 1e-5
        for n in range(c.N):
            for d in range(c.D):
                xp, xm = c.x.copy(), c.x.copy()
                xp[n, d] += h
                xm[n, d] -= h
                fd = (oracle.loglik(xp, c.t, c.theta)[0] - oracle.loglik(xm, c.t, c.theta)[0]) / (2 * h)
                assert abs(fd - gr[n, d]) <= 1e-5 * max(abs(gr[n, d]), 1e-3 * S[n, d])


# ------------------------------------------------------------ Lambda / phi_D
def test_Lambda_matches_quadrature_of_intensity():
    """P6: Lambda_n = int_0^{t_N} of the spatially integrated intensity
    contributed by event n: mu0 phi((t-t_n)/tau_t)/tau_t + theta omega e^{-omega(t-t_n)} I[t>t_n]."""
    from scipy import integrate
    c = synth.unit_square(25, config=14)
    for th in [c.theta, (1.3, 0.2, 0.05, 0.8, 7.0, 0.1)]:
        mu0, _, tt, tht, om, _ = th
        Lam = oracle.Lambda(c.t, th)
        tN = c.t[-1]
        for n in range(c.N):
            bg, _ = integrate.quad(lambda s: mu0 * math.exp(-0.5 * ((s - c.t[n]) / tt) ** 2)
                                   / (tt * math.sqrt(2 * math.pi)), 0, tN, epsabs=0, epsrel=1e-13,
                                   points=[c.t[n]], limit=200)
            se, _ = integrate.quad(lambda s: tht * om * math.exp(-om * (s - c.t[n])), c.t[n], tN,
                                   epsabs=0, epsrel=1e-13, limit=200) if c.t[n] < tN else (0.0, 0)
            assert Lam[n] == pytest.approx(bg + se, rel=1e-11, abs=1e-14)


def test_pair_terms_integrate_to_their_weights():
    """phi_D normalisation (reading R1): integrating mu_nm over x_n in R^2 leaves
    mu0 phi(dt/tau_t)/tau_t, and xi_nm leaves theta omega e^{-omega dt}; these are the
    integrands whose time integrals give Lambda_n."""
    from scipy import integrate
    th = (0.9, 0.3, 0.4, 0.6, 2.5, 0.2)
    t = np.array([0.1, 0.7])
    dt = t[1] - t[0]

    def f(kind, a, b):
        x = np.array([[0.3, -0.2], [0.3 + a, -0.2 + b]])
        return oracle.mu_pair(x, t, th, 1, 0) if kind == "mu" else oracle.xi_pair(x, t, th, 1, 0)

    L = 12.0
    mu_int, _ = integrate.dblquad(lambda b, a: f("mu", a, b), -L * th[1], L * th[1],
                                  -L * th[1], L * th[1], epsabs=0, epsrel=1e-10)
    xi_int, _ = integrate.dblquad(lambda b, a: f("xi", a, b), -L * th[5], L * th[5],
                                  -L * th[5], L * th[5], epsabs=0, epsrel=1e-10)
    assert mu_int == pytest.approx(th[0] * math.exp(-0.5 * (dt / th[2]) ** 2)
                                   / (th[2] * math.sqrt(2 * math.pi)), rel=1e-9)
    assert xi_int == pytest.approx(th[3] * th[4] * math.exp(-th[4] * dt), rel=1e-9)


# -------------------------------------------------------------- KDE (theta=0)
def test_theta_zero_is_leave_one_out_kde():
    """P8: with theta = 0, lambda_n is mu0 times the leave-one-out Gaussian product-kernel
    space-time KDE (the smoother of P:L82), evaluated here by scikit-learn."""
    from sklearn.neighbors import KernelDensity
    c = synth.unit_square(200, config=15)
    th = (0.8, 0.12, 0.07, 0.0, 20.0, 0.03)
    lam, _, _ = oracle.rates(c.x, c.t, th)
    z = np.column_stack([c.x / th[1], c.t / th[2]])
    kde = KernelDensity(kernel="gaussian", bandwidth=1.0, rtol=0.0, atol=0.0).fit(z)
    dens = np.exp(kde.score_samples(z)) * c.N          # sum_m phi_3(z_n - z_m), self included
    self_term = (2 * math.pi) ** -1.5
    ref = th[0] * (dens - self_term) / (th[1] ** 2 * th[2])
    np.testing.assert_allclose(lam, ref, rtol=1e-9)


# ------------------------------------------------------------------ invariants
def test_invariances_translation_rotation_scaling():
    """P7: ell depends on X only through differences and norms."""
    c = synth.unit_square(80, config=16)
    ell, _, _ = oracle.loglik(c.x, c.t, c.theta)
    g, S = oracle.grad(c.x, c.t, c.theta)
    # (i) sum of gradients vanishes (c_nn' symmetric, App. A)
    assert np.all(np.abs(g.sum(axis=0)) <= 1e-13 * S.sum(axis=0))
    # (ii) translation
    ell2, _, _ = oracle.loglik(c.x + np.array([3.7, -11.2]), c.t, c.theta)
    assert ell2 == pytest.approx(ell, rel=1e-12)
    # (iii) rotation
    a = 0.7
    R = np.array([[math.cos(a), -math.sin(a)], [math.sin(a), math.cos(a)]])
    xr = c.x @ R.T
    ell3, _, _ = oracle.loglik(xr, c.t, c.theta)
    assert ell3 == pytest.approx(ell, rel=1e-12)
    g3, _ = oracle.grad(xr, c.t, c.theta)
    assert np.all(np.abs(g3 - g @ R.T) <= 1e-11 * (S + np.abs(g)).max())
    # (iv) scaling covariance: ell(aX; a tau_x, a h) = ell(X) - N D ln a, g -> g/a
    s = 3.5
    th = list(c.theta)
    th[1] *= s
    th[5] *= s
    ell4, _, _ = oracle.loglik(s * c.x, c.t, th)
    assert ell4 == pytest.approx(ell - c.N * c.D * math.log(s), rel=1e-12)
    g4, _ = oracle.grad(s * c.x, c.t, th)
    np.testing.assert_allclose(g4, g / s, rtol=1e-10, atol=1e-12 * np.abs(g).max())
    # (v) time shift leaves every lambda_n unchanged
    _, lam, _ = oracle.loglik(c.x, c.t, c.theta)
    _, lam5, _ = oracle.loglik(c.x, c.t + 0.25, c.theta)
    np.testing.assert_allclose(lam5, lam, rtol=1e-12)


def test_decomposition_sum_of_pairs():
    """P9: sum_n lambda_n = sum_{n,n'} (mu_nn' + xi_nn')."""
    c = synth.unit_square(40, config=17)
    lam, _, _ = oracle.rates(c.x, c.t, c.theta)
    tot = math.fsum(oracle.mu_pair(c.x, c.t, c.theta, n, m) + oracle.xi_pair(c.x, c.t, c.theta, n, m)
                    for n in range(c.N) for m in range(c.N))
    assert lam.sum() == pytest.approx(tot, rel=1e-12)


# --------------------------------------------------------- special / edge cases
def test_single_event_is_minus_infinity():
    """N=1: both indicators vanish, lambda_1 = 0 -> ell = -inf."""
    ell, lam, _ = oracle.loglik(np.array([[0.2, 0.3]]), np.array([0.5]), synth.THETA_UNIT)
    assert lam[0] == 0.0 and ell == -math.inf


def test_ties_contribute_nothing():
    """Equal-time pairs contribute to neither mu nor xi (reading R8)."""
    c = synth.with_ties(60, 7)
    for n in range(c.N):
        for m in range(c.N):
            if c.t[n] == c.t[m]:
                assert oracle.mu_pair(c.x, c.t, c.theta, n, m) == 0.0
                assert oracle.xi_pair(c.x, c.t, c.theta, n, m) == 0.0
    # all events at one time: every lambda is 0
    ell, lam, _ = oracle.loglik(c.x, np.full(c.N, 0.5), c.theta)
    assert np.all(lam == 0.0) and ell == -math.inf
    # a tied pair far from everything else has zero gradient on the pair's axis
    x = np.array([[0.0, 0.0], [0.01, 0.0], [5.0, 5.0]])
    t = np.array([0.2, 0.2, 0.3])
    g, _ = oracle.grad(x, t, (1.0, 1.0, 1.0, 1.0, 1.0, 1.0))
    assert np.all(np.isfinite(g))
    mu01 = oracle.mu_pair(x, t, (1.0, 1.0, 1.0, 1.0, 1.0, 1.0), 0, 1)
    assert mu01 == 0.0


def test_last_event_has_no_self_excitation_integral():
    """t_n = t_N: the exponential term of Lambda_n is -theta(e^0 - 1) = 0."""
    th = (0.0, 1.0, 1.0, 2.0, 3.0, 1.0)   # mu0 = 0 isolates the self-excitation term
    Lam = oracle.Lambda(np.array([0.1, 0.4, 0.9]), th)
    assert Lam[-1] == 0.0
    assert Lam[0] == pytest.approx(2.0 * (1 - math.exp(-3.0 * 0.8)), rel=1e-15)


def test_unsorted_times_rejected():
    with pytest.raises(ValueError):
        oracle.loglik(np.zeros((3, 2)), np.array([0.3, 0.1, 0.2]), synth.THETA_UNIT)


# ------------------------------------------------------------------- BMDS oracle
def test_bmds_two_points_is_a_truncated_normal():
    """N=2: the BMDS density of Eq. bmdsLikelihood is the density of one
    N(delta, sigma^2) variate truncated to y > 0 (scipy.stats.truncnorm)."""
    from scipy.stats import truncnorm
    x = np.array([[0.3, -0.2, 1.1], [1.0, 0.4, 0.2]])
    delta = float(np.linalg.norm(x[0] - x[1]))
    for y, s in [(1.1, 0.3), (0.2, 0.9), (4.0, 2.0)]:
        Y = np.array([[0.0, y], [y, 0.0]])
        lp, _ = oracle.bmds(x, Y, s)
        ref = truncnorm.logpdf(y, a=-delta / s, b=np.inf, loc=delta, scale=s)
        assert lp == pytest.approx(ref, rel=1e-13)


@pytest.mark.parametrize("N,D", [(4, 2), (5, 6)])
def test_bmds_brute_force_40_digits(N, D):
    """mpmath transcription of Eq. bmdsLikelihood; its gradient by mp.diff (so the hand-
    derived gradient in the oracle is pinned to the density)."""
    rng = np.random.default_rng(N + D)
    x = rng.normal(size=(N, D))
    Y = synth.bmds_dissimilarities(x, 0.4, seed=N)
    s = 0.4
    with mp.workdps(40):
        def logp(X):
            tot = mp.mpf(0)
            for n in range(N):
                for m in range(n):
                    d = mp.sqrt(sum((X[n][k] - X[m][k]) ** 2 for k in range(D)))
                    tot += -mp.log(2 * mp.pi * s * s) / 2 - (mp.mpf(Y[n, m]) - d) ** 2 / (2 * s * s) \
                        - mp.log(mp.ncdf(d / s))
            return tot
        X = [[mp.mpf(v) for v in row] for row in x]
        ref = logp(X)
        gref = []
        for n in range(N):
            for k in range(D):
                def f(v, n=n, k=k):
                    Xv = [list(r) for r in X]
                    Xv[n][k] = v
                    return logp(Xv)
                gref.append(float(mp.diff(f, X[n][k])))
    lp, g, S = oracle.bmds(x, Y, s, with_scale=True)
    assert lp == pytest.approx(float(ref), rel=1e-13)
    np.testing.assert_allclose(g.reshape(-1), gref, rtol=0, atol=1e-12 * S.max())


def test_bmds_gradient_invariances_and_differences():
    c, Y, s = synth.flu_shaped(60, 3)
    lp, g, S = oracle.bmds(c.x, Y, s, with_scale=True)
    assert np.all(np.abs(g.sum(axis=0)) <= 1e-12 * S.sum(axis=0))
    shifted, _ = oracle.bmds(c.x + 5.0, Y, s)
    assert shifted == pytest.approx(lp, rel=1e-12)
    h = 1e-6
    for n, d in [(0, 0), (17, 2), (59, 1)]:
        xp, xm = c.x.copy(), c.x.copy()
        xp[n, d] += h
        xm[n, d] -= h
        fd = (oracle.bmds(xp, Y, s, with_grad=False)[0] - oracle.bmds(xm, Y, s, with_grad=False)[0]) / (2 * h)
        assert abs(fd - g[n, d]) <= 1e-6 * max(abs(g[n, d]), S[n, d])


# ---- HMC transition (Neal 2011) and its counter-based random numbers

def test_philox_known_answers(golden_dir):
    """Philox-4x32-10 against the published Random123 known-answer vectors."""
    with open(os.path.join(golden_dir, "philox4x32_10_kat.json")) as f:
        kat = json.load(f)
    for v in kat["vectors"]:
        ctr = [int(w, 16) for w in v["ctr"]]
        key = [int(w, 16) for w in v["key"]]
        assert oracle.philox4x32_10(ctr, key) == [int(w, 16) for w in v["out"]]


def test_hmc_normals_are_standard_normal():
    """Box-Muller of the Philox uniforms: Kolmogorov-Smirnov against N(0,1), moments, and
    no correlation between the two normals of a block or between iterations/seeds."""
    from scipy import stats
    n = 200_001
    z = oracle.hmc_normals(5, 3, n)
    assert stats.kstest(z, "norm").pvalue > 1e-3
    assert abs(z.mean()) < 5 / math.sqrt(n)
    assert abs(z.var() - 1) < 5 * math.sqrt(2 / n)
    assert abs(np.mean(z ** 4) - 3) < 0.1          # kurtosis of the normal
    m = (n - 1) // 2
    assert abs(np.corrcoef(z[0:2 * m:2], z[1:2 * m:2])[0, 1]) < 5 / math.sqrt(m)
    z2 = oracle.hmc_normals(5, 4, n)
    z3 = oracle.hmc_normals(6, 3, n)
    assert abs(np.corrcoef(z, z2)[0, 1]) < 5 / math.sqrt(n)
    assert abs(np.corrcoef(z, z3)[0, 1]) < 5 / math.sqrt(n)
    # prefix property: element e's draw does not depend on the length requested
    assert np.array_equal(oracle.hmc_normals(5, 3, 101), z[:101])
    # the uniform is (0,1) and varies with the iteration
    u = np.array([oracle.hmc_uniform(5, it) for it in range(2000)])
    assert u.min() > 0 and u.max() < 1 and stats.kstest(u, "uniform").pvalue > 1e-3


def test_hmc_step_energy_error_is_second_order():
    """log alpha = H0 - H1 of the leapfrog is O(step^2) (Neal 2011 sec. 5.2): halving the
    step divides it by ~4.  A sign error in H (U - K instead of U + K) or a potential of the
    wrong sign leaves an O(1) term and fails this."""
    c = synth.config("C1", 200)
    las = []
    for step in (2e-4, 1e-4, 5e-5):
        _, _, la = oracle.hmc_step(c.x, c.t, c.theta, 3, 0, step, int(round(4e-4 / step)))
        las.append(abs(la))
    assert 3.0 < las[0] / las[1] < 5.0 and 3.0 < las[1] / las[2] < 5.0


def test_hmc_step_zero_steps_accepts_and_keeps_x():
    """No trajectory: H1 = H0, log alpha = 0 and log u < 0 always accepts."""
    c = synth.config("C1", 100)
    x1, acc, la = oracle.hmc_step(c.x, c.t, c.theta, 9, 1, 1e-3, 0)
    assert acc and la == 0.0 and np.array_equal(x1, c.x)


def test_hmc_step_reversible():
    """The transition's proposal is an involution: from (x1, -p1) the same leapfrog returns
    to (x0, -p0), so a Metropolis step with H alone is valid (Neal 2011 sec. 3.2)."""
    c = synth.config("C1", 150)
    z = oracle.hmc_normals(4, 2, c.x.size).reshape(c.x.shape)
    x1, p1, _, _ = oracle.leapfrog(c.x, z, c.t, c.theta, 2e-3, 6)
    x2, p2, _, _ = oracle.leapfrog(x1, -p1, c.t, c.theta, 2e-3, 6)
    assert np.allclose(x2, c.x, atol=1e-10) and np.allclose(-p2, z, atol=1e-8)


# ---- leapfrog / HMC branches with a diagonal mass and a reflecting box (reading R15:
# diagonal M, optional reflecting box).  These pin the oracle's mass and box arithmetic against
# properties they must have, not against a retyped formula: a reflection that is not an
# involution breaks reversibility; M instead of M^-1 in the drift breaks the scaling
# equivalence; p0 = z sqrt(Minv) instead of z / sqrt(Minv) breaks the momentum covariance.

def _mass_box_case(N=120, seed=7):
    c = synth.config("C1", N)
    rng = np.random.default_rng(seed)
    minv = rng.uniform(0.25, 4.0, size=c.x.shape)          # non-identity diagonal M^-1
    half = 0.004                                            # box of +-half around x0
    return c, minv, c.x - half, c.x + half


def _reflections(x0, p0, c, minv, lo, hi, step, L):
    """Count the components whose momentum sign flips in the trajectory (proof the box was hit)."""
    x, p = x0.copy(), p0.copy()
    flips = 0
    for _ in range(L):
        x1, p1, _, _ = oracle.leapfrog(x, p, c.t, c.theta, step, 1, inv_mass=minv, box_lo=lo, box_hi=hi)
        flips += int(np.sum(np.sign(p1) != np.sign(p + 0.5 * step * oracle.grad(x, c.t, c.theta)[0])))
        x, p = x1, p1
    return flips


def test_leapfrog_box_and_mass_reversible():
    """Leapfrog with a reflecting box and a diagonal mass is an involution up to the momentum
    sign: (x1, -p1) integrates back to (x0, -p0).  The box is hit (momenta flip) on the way,
    and every state stays inside it."""
    c, minv, lo, hi = _mass_box_case()
    z = oracle.hmc_normals(11, 0, c.x.size).reshape(c.x.shape)
    p0 = z / np.sqrt(minv)
    step, L = 2e-3, 8
    assert _reflections(c.x, p0, c, minv, lo, hi, step, L) > 20
    x1, p1, _, _ = oracle.leapfrog(c.x, p0, c.t, c.theta, step, L, inv_mass=minv, box_lo=lo, box_hi=hi)
    assert np.all(x1 >= lo) and np.all(x1 <= hi)
    assert not np.allclose(x1, c.x, atol=1e-6)
    x2, p2, _, _ = oracle.leapfrog(x1, -p1, c.t, c.theta, step, L, inv_mass=minv, box_lo=lo, box_hi=hi)
    assert np.allclose(x2, c.x, rtol=0, atol=1e-11)
    assert np.allclose(-p2, p0, rtol=1e-9, atol=1e-9 * np.abs(p0).max())


def test_leapfrog_mass_energy_error_is_second_order():
    """With a non-identity diagonal mass, H = -ell + 1/2 sum Minv p^2 is conserved to O(step^2):
    halving the step divides the energy error by ~4 (a kinetic energy of the wrong form,
    e.g. 1/2 sum p^2 / Minv, leaves an O(step) or O(1) error)."""
    c, minv, _, _ = _mass_box_case(N=150, seed=3)
    z = oracle.hmc_normals(2, 5, c.x.size).reshape(c.x.shape)
    p0 = z / np.sqrt(minv)
    H0 = -oracle.loglik(c.x, c.t, c.theta)[0] + 0.5 * float(np.sum(minv * p0 * p0))
    errs = []
    for step in (1e-4, 5e-5, 2.5e-5):
        _, _, ell, kin = oracle.leapfrog(c.x, p0, c.t, c.theta, step, int(round(4e-4 / step)),
                                         inv_mass=minv)
        errs.append(abs(-ell + kin - H0))
    assert 3.0 < errs[0] / errs[1] < 5.0 and 3.0 < errs[1] / errs[2] < 5.0


def test_leapfrog_scaling_equivalence_with_mass_and_box():
    """Coordinates scaled by a (x -> a x, tau_x -> a tau_x, h -> a h, box -> a box,
    M^-1 -> a^2 M^-1, p -> p / a): ell changes by -N D ln a (pin P7(iv)), the gradient by 1/a,
    so the leapfrog must give exactly a times the trajectory and 1/a times the momenta, with
    the same kinetic energy.  Pins that the drift multiplies by M^-1 (not M) and that the
    reflection is applied to the scaled box."""
    c, minv, lo, hi = _mass_box_case(N=100, seed=5)
    z = oracle.hmc_normals(8, 1, c.x.size).reshape(c.x.shape)
    p0 = z / np.sqrt(minv)
    step, L, a = 2e-3, 6, 8.0          # power of two: the scaling is exact in fp64
    mu0, tx, tt, th, om, h = c.theta
    theta_a = (mu0, a * tx, tt, th, om, a * h)
    x1, p1, ell1, k1 = oracle.leapfrog(c.x, p0, c.t, c.theta, step, L, inv_mass=minv, box_lo=lo, box_hi=hi)
    xa, pa, ella, ka = oracle.leapfrog(a * c.x, p0 / a, c.t, theta_a, step, L, inv_mass=a * a * minv,
                                       box_lo=a * lo, box_hi=a * hi)
    assert np.allclose(xa, a * x1, rtol=0, atol=1e-12 * a)
    assert np.allclose(pa, p1 / a, rtol=1e-10, atol=1e-10 * np.abs(p1).max() / a)
    assert ka == pytest.approx(k1, rel=1e-10)
    assert ella == pytest.approx(ell1 - c.N * c.D * math.log(a), rel=1e-12)


def test_hmc_step_momenta_have_covariance_M():
    """hmc_step draws p0 ~ N(0, M) (p0 = z / sqrt(Minv)).  With a zero potential (hawkes=False,
    no BMDS) one leapfrog step is x1 = x0 + step Minv p0 exactly and H is conserved (always
    accepted), so (x1 - x0) / (step sqrt(Minv)) must be standard normal per component: KS and
    variance against N(0, 1) with Minv spanning 1/16..16 (p0 = z sqrt(Minv) would give
    variances Minv^2 and fail)."""
    from scipy import stats
    N, D = 4000, 3
    rng = np.random.default_rng(1)
    x0 = rng.uniform(0, 1, size=(N, D))
    minv = np.exp(rng.uniform(np.log(1 / 16), np.log(16), size=(N, D)))
    t = np.sort(rng.uniform(0, 1, N))
    step = 1e-3
    x1, acc, la = oracle.hmc_step(x0, t, (0.6, 0.1, 0.1, 0.4, 20.0, 0.03), 21, 4, step, 1,
                                  inv_mass=minv, hawkes=False)
    assert acc and abs(la) < 1e-9
    w = ((x1 - x0) / (step * np.sqrt(minv))).ravel()
    assert stats.kstest(w, "norm").pvalue > 1e-3
    assert abs(w.var() - 1.0) < 5 * math.sqrt(2.0 / w.size)
    # and the scale really depends on Minv: the raw displacements' variance tracks Minv
    hi, lo = minv.ravel() > 4, minv.ravel() < 0.25
    dx = ((x1 - x0) / step).ravel()
    assert dx[hi].var() / dx[lo].var() > 16


# ---- block MH over coarsened locations (Eq. circleKernel)

def test_lens_area_closed_forms_and_monte_carlo():
    """Two unit circles one radius apart: 2 pi/3 - sqrt(3)/2 (textbook); containment and
    disjoint limits; continuity at the branch points; 2e6-point Monte Carlo elsewhere."""
    la = oracle.lens_area
    assert la(1.0, 1.0, 1.0) == pytest.approx(2 * math.pi / 3 - math.sqrt(3) / 2, rel=1e-14)
    assert la(2.0, 0.5, 1.0) == pytest.approx(math.pi * 0.25, rel=1e-15)
    assert la(0.5, 2.0, 1.0) == pytest.approx(math.pi * 0.25, rel=1e-15)
    assert la(1.0, 1.0, 2.0) == 0.0
    for R, rho in ((1.0, 0.3), (1.0, 1.7)):
        dc = abs(R - rho)
        assert la(R, rho, dc * (1 + 1e-9)) == pytest.approx(math.pi * min(R, rho) ** 2, rel=1e-4)
        assert la(R, rho, (R + rho) * (1 - 1e-12)) < 1e-10
    rng = np.random.default_rng(0)
    for R, rho, d in ((1.0, 0.6, 0.8), (1.0, 1.0, 0.4), (2.0, 1.1, 1.9), (1.0, 1.5, 0.9)):
        n = 2_000_000
        p = rng.uniform(-rho, rho, size=(n, 2))
        inside_small = np.sum(p * p, axis=1) < rho * rho
        inside_big = (p[:, 0] + d) ** 2 + p[:, 1] ** 2 < R * R     # big disc centred at (-d, 0)
        frac = np.mean(inside_small & inside_big)
        se = math.sqrt(frac * (1 - frac) / n)
        assert abs(la(R, rho, d) - 4 * rho * rho * frac) < 5 * 4 * rho * rho * se


def test_truncated_normal_proposal_distribution():
    """Square proposals (Eq. locsPrior1 region) follow N(x, s^2) truncated to the box:
    Kolmogorov-Smirnov against scipy.stats.truncnorm, per dimension."""
    from scipy import stats
    x, c, h, scale = np.array([30.0, -45.0]), np.array([0.0, 0.0]), 50.0, 0.8
    s = scale * h
    draws = np.array([oracle.mh_propose("square", x, c, h, scale, 5, 1, b, 3)[0] for b in range(6000)])
    for d in range(2):
        a, b = (c[d] - h - x[d]) / s, (c[d] + h - x[d]) / s
        assert stats.kstest(draws[:, d], stats.truncnorm(a, b, loc=x[d], scale=s).cdf).pvalue > 1e-3
    assert np.all(np.abs(draws - c) <= h)


def test_disc_proposal_is_uniform_on_the_lens():
    """Disc proposals (Eq. circleKernel) are uniform on disc(c, r) cap disc(x, r eps):
    two-sample KS per coordinate against an independent numpy rejection sampler."""
    from scipy import stats
    c, r, eps = np.array([0.0, 0.0]), 1.0, 0.9
    x = np.array([0.7, 0.2])
    draws = np.array([oracle.mh_propose("disc", x, c, r, eps, 9, 2, b, 0)[0] for b in range(6000)])
    assert np.all(np.sum((draws - c) ** 2, axis=1) < r * r)
    assert np.all(np.sum((draws - x) ** 2, axis=1) < (r * eps) ** 2)
    rng = np.random.default_rng(1)
    p = x + rng.uniform(-r * eps, r * eps, size=(60000, 2))
    keep = (np.sum((p - x) ** 2, axis=1) < (r * eps) ** 2) & (np.sum((p - c) ** 2, axis=1) < r * r)
    ref = p[keep]
    for d in range(2):
        assert stats.ks_2samp(draws[:, d], ref[:, d]).pvalue > 1e-3


def _mh_chain_r2(kind, size, scale, T):
    """One event of a 3-event catalog moved by the block MH kernel T times; returns the chain's
    E|x - c|^2 with its batch-means standard error and the exact value by grid quadrature."""
    t = np.array([0.0, 0.5, 0.7])
    theta = (0.5, 0.6, 1.0, 0.5, 2.0, 0.4)
    x0 = np.array([[0.8, 0.3], [0.0, 0.0], [-0.5, 0.9]])
    centre, sz = np.zeros((3, 2)), np.full(3, size)
    r2 = np.empty(T)
    x = x0.copy()
    for it in range(T):
        x, _, _ = oracle.mh_sweep(x, t, theta, kind, centre, sz, [[1]], scale, 17, it)
        r2[it] = x[1, 0] ** 2 + x[1, 1] ** 2
    bm = r2.reshape(40, -1).mean(axis=1)
    se = bm.std(ddof=1) / math.sqrt(len(bm))
    G = 160
    g = (np.arange(G) + 0.5) / G * 2 * size - size
    w = np.zeros((G, G))
    for i in range(G):
        for j in range(G):
            if kind == "disc" and g[i] ** 2 + g[j] ** 2 >= size ** 2:
                continue
            xp = x0.copy()
            xp[1] = (g[i], g[j])
            w[i, j] = math.exp(oracle.loglik(xp, t, theta)[0])
    G2 = g[:, None] ** 2 + g[None, :] ** 2
    return r2.mean(), se, float(np.sum(w * G2) / np.sum(w))


@pytest.mark.parametrize("kind,scale", [("square", 1.0), ("disc", 1.0)])
def test_block_mh_targets_the_posterior(kind, scale):
    """Stationarity: the chain's E|x_n - c|^2 matches the exact posterior of one event
    (likelihood x uniform region prior, grid quadrature).  The proposals here are strongly
    asymmetric near the region edge, so dropping or inverting the Hastings term shifts this
    moment by 9-15 standard errors (0.044 for the square, 0.055 for the disc at eps = 1)."""
    m, se, exact = _mh_chain_r2(kind, 1.0, scale, 16000)
    assert abs(m - exact) < max(4 * se, 0.004), (m, se, exact)
