"""40-digit brute-force evaluation of Eq. 1 and the App. A gradient (mpmath).

An independent transcription used only to pin the oracle's floating-point
evaluation on tiny catalogs (N <= 10): it checks rounding, summation and
indexing, not the reading of the formulas (the closed-form, quadrature,
finite-difference, complex-step and KDE pins in test_oracle_pins.py do that).
The gradient here is NOT the App. A formula: it is the derivative of ell
computed by mpmath's numerical differentiation (mp.diff) at 40 digits, so it
pins the App. A formula itself as well.
"""
import mpmath as mp


def _terms(x, t, theta, D):
    mu0, tx, tt, th, om, h = [mp.mpf(v) for v in theta]
    N = len(t)
    two_pi = 2 * mp.pi

    def lam(n, X):
        s = mp.mpf(0)
        for m in range(N):
            r2_b = sum(((X[n][d] - X[m][d]) / tx) ** 2 for d in range(D))
            r2_s = sum(((X[n][d] - X[m][d]) / h) ** 2 for d in range(D))
            if t[n] != t[m]:
                dtt = (mp.mpf(t[n]) - mp.mpf(t[m])) / tt
                s += mu0 / (tx ** D * tt) * mp.exp(-r2_b / 2) / two_pi ** (mp.mpf(D) / 2) \
                    * mp.exp(-dtt ** 2 / 2) / mp.sqrt(two_pi)
            if t[m] < t[n]:
                s += th * om / h ** D * mp.exp(-om * (mp.mpf(t[n]) - mp.mpf(t[m]))) \
                    * mp.exp(-r2_s / 2) / two_pi ** (mp.mpf(D) / 2)
        return s

    tN = mp.mpf(max(t))
    Phi = lambda z: mp.ncdf(z)
    Lam = [mu0 * (Phi((tN - mp.mpf(tn)) / tt) - Phi(-mp.mpf(tn) / tt))
           - th * (mp.exp(-om * (tN - mp.mpf(tn))) - 1) for tn in t]
    return lam, Lam


def evaluate(x, t, theta, dps=40, with_grad=True):
    """Returns dict(lam, Lam, ell, grad) as mpf values."""
    with mp.workdps(dps):
        N = len(t)
        D = len(x[0])
        X = [[mp.mpf(v) for v in row] for row in x]
        lam, Lam = _terms(x, t, theta, D)
        lams = [lam(n, X) for n in range(N)]

        def ell_of(Xv):
            return sum(mp.log(lam(n, Xv)) - Lam[n] for n in range(N))

        ell = sum(mp.log(l) - L for l, L in zip(lams, Lam))
        out = {"lam": lams, "Lam": Lam, "ell": ell}
        if with_grad:
            g = []
            for n in range(N):
                row = []
                for d in range(D):
                    def f(v, n=n, d=d):
                        Xv = [list(r) for r in X]
                        Xv[n][d] = v
                        return ell_of(Xv)
                    row.append(mp.diff(f, X[n][d]))
                g.append(row)
            out["grad"] = g
        return out
