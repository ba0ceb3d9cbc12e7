"""CPU oracle for the Hawkes log-likelihood and location gradient -- TEST INFRASTRUCTURE ONLY.

Plain fp64 C (``hawkes_oracle.c``) behind ctypes, plus a literal leapfrog
integrator in numpy.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import this
package.  The CUDA product path (``paper_2010_02994_b200``) never imports it and
shares no code with it.

Every function cites /root/reference/PAPER.md as P:L<line>; the formulas are
restated in the header of ``hawkes_oracle.c``.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hawkes_oracle.c")
_LIB = os.path.join(_HERE, "_build", "liboracle.so")

ORACLE_OK = 0


class _Params(ctypes.Structure):
    # Theta = (mu0, tau_x, tau_t, theta, omega, h)
    _fields_ = [(n, ctypes.c_double) for n in ("mu0", "tau_x", "tau_t", "theta", "omega", "h")]


def build(force: bool = False) -> str:
    """Compile the oracle with strict IEEE flags (-O2 -ffp-contract=off, OpenMP)."""
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-std=c11", _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        pp = ctypes.POINTER(_Params)
        L, I = ctypes.c_long, ctypes.c_int
        lib.oracle_rates.argtypes = [L, I, dp, dp, pp, L, L, dp, dp, dp]
        lib.oracle_Lambda.argtypes = [L, dp, pp, dp]
        lib.oracle_loglik.argtypes = [L, I, dp, dp, pp, dp, dp, dp]
        lib.oracle_grad.argtypes = [L, I, dp, dp, pp, dp, L, L, dp, dp]
        lib.oracle_loglik_complex.argtypes = [L, I, dp, dp, dp, pp, dp, dp]
        lib.oracle_mu_pair.argtypes = [I, dp, dp, L, L, pp]
        lib.oracle_mu_pair.restype = ctypes.c_double
        lib.oracle_xi_pair.argtypes = [I, dp, dp, L, L, pp]
        lib.oracle_xi_pair.restype = ctypes.c_double
        lib.oracle_num_threads.restype = ctypes.c_int
        lib.oracle_bmds.argtypes = [L, I, dp, dp, ctypes.c_double, dp, dp, dp]
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib.oracle_philox4x32_10.argtypes = [u32p, u32p, u32p]
        lib.oracle_hmc_normals.argtypes = [ctypes.c_uint64, ctypes.c_uint64, L, dp]
        lib.oracle_hmc_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.oracle_hmc_uniform.restype = ctypes.c_double
        lib.oracle_bmds_pair.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double]
        lib.oracle_bmds_pair.restype = ctypes.c_double
        _lib = lib
    return _lib


def _dptr(a: Optional[np.ndarray]):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _prep(x, t):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    t = np.ascontiguousarray(t, dtype=np.float64)
    assert x.shape[0] == t.shape[0], "x and t disagree on N"
    return x, t


def _params(theta: Sequence[float]) -> _Params:
    return _Params(*[float(v) for v in theta])


def _check(rc: int, what: str):
    if rc != ORACLE_OK:
        raise ValueError(f"oracle {what} failed with status {rc}")


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def mu_pair(x, t, theta, n: int, m: int) -> float:
    """mu_{nm}, P:L98 (background term of lambda_nm)."""
    x, t = _prep(x, t)
    p = _params(theta)
    return _load().oracle_mu_pair(x.shape[1], _dptr(x), _dptr(t), n, m, ctypes.byref(p))


def xi_pair(x, t, theta, n: int, m: int) -> float:
    """xi_{nm}, P:L99 (self-excitation term of lambda_nm)."""
    x, t = _prep(x, t)
    p = _params(theta)
    return _load().oracle_xi_pair(x.shape[1], _dptr(x), _dptr(t), n, m, ctypes.byref(p))


def rates(x, t, theta, rows: Optional[slice] = None):
    """lambda_n, mu_n = sum_n' mu_nn', xi_n = sum_n' xi_nn' for rows (Eq. 1).

    Returns arrays of length N; rows outside ``rows`` are NaN."""
    x, t = _prep(x, t)
    N, D = x.shape
    r0, r1 = (0, N) if rows is None else (rows.start or 0, N if rows.stop is None else rows.stop)
    lam = np.full(N, np.nan)
    mu = np.full(N, np.nan)
    xi = np.full(N, np.nan)
    p = _params(theta)
    _check(_load().oracle_rates(N, D, _dptr(x), _dptr(t), ctypes.byref(p), r0, r1,
                                _dptr(lam), _dptr(mu), _dptr(xi)), "rates")
    return lam, mu, xi


def Lambda(t, theta) -> np.ndarray:
    """Lambda_n."""
    t = np.ascontiguousarray(t, dtype=np.float64)
    out = np.empty_like(t)
    p = _params(theta)
    _check(_load().oracle_Lambda(t.shape[0], _dptr(t), ctypes.byref(p), _dptr(out)), "Lambda")
    return out


def loglik(x, t, theta):
    """(ell, lambda, Lambda) -- Eq. 1.  ell = -inf if any lambda_n = 0."""
    x, t = _prep(x, t)
    N, D = x.shape
    lam = np.empty(N)
    Lam = np.empty(N)
    ll = ctypes.c_double()
    p = _params(theta)
    _check(_load().oracle_loglik(N, D, _dptr(x), _dptr(t), ctypes.byref(p), ctypes.byref(ll),
                                 _dptr(lam), _dptr(Lam)), "loglik")
    return ll.value, lam, Lam


def grad(x, t, theta, lam: Optional[np.ndarray] = None, rows: Optional[slice] = None):
    """(grad N x D, scale N x D) -- App. A.

    ``lam`` defaults to the oracle's own rates; ``scale[n,d]`` is
    sum_n' |c_nn' (x_n'd - x_nd)|, the conditioning scale of g[n,d].
    Raises if some lambda_n = 0 (gradient undefined)."""
    x, t = _prep(x, t)
    N, D = x.shape
    if lam is None:
        lam, _, _ = rates(x, t, theta)
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    if np.any(lam == 0.0):
        raise ValueError("gradient undefined: some lambda_n = 0 (ell = -inf)")
    r0, r1 = (0, N) if rows is None else (rows.start or 0, N if rows.stop is None else rows.stop)
    g = np.full((N, D), np.nan)
    s = np.full((N, D), np.nan)
    p = _params(theta)
    _check(_load().oracle_grad(N, D, _dptr(x), _dptr(t), ctypes.byref(p), _dptr(lam), r0, r1,
                               _dptr(g), _dptr(s)), "grad")
    return g, s


def loglik_complex(x_re, x_im, t, theta):
    """Complex-step ell(X_re + i X_im): returns (Re ell, Im ell)."""
    x_re, t = _prep(x_re, t)
    x_im = np.ascontiguousarray(x_im, dtype=np.float64).reshape(x_re.shape)
    N, D = x_re.shape
    a, b = ctypes.c_double(), ctypes.c_double()
    p = _params(theta)
    _check(_load().oracle_loglik_complex(N, D, _dptr(x_re), _dptr(x_im), _dptr(t),
                                         ctypes.byref(p), ctypes.byref(a), ctypes.byref(b)),
           "loglik_complex")
    return a.value, b.value


def leapfrog(x, p, t, theta, step: float, n_steps: int, inv_mass=None, box_lo=None, box_hi=None,
             bmds_data=None, hawkes: bool = True):
    """Leapfrog trajectory of HMC over locations (Neal 2011, cited there).

    Potential U(X) = -ell(X) [- log p(Y | X) with bmds_data = (Y, sigma): the flu model's
    joint density; hawkes=False drops ell].  Each step: p += (step/2) grad ell; x += step M^-1 p
    (reflecting off [box_lo, box_hi] componentwise when given, negating p);
    p += (step/2) grad ell.  Returns (x, p, ell_end, kinetic_end) with
    kinetic = 1/2 sum p^2 M^-1."""
    x = np.array(x, dtype=np.float64, copy=True)
    p = np.array(p, dtype=np.float64, copy=True)
    minv = np.ones_like(x) if inv_mass is None else np.asarray(inv_mass, dtype=np.float64)

    def grad(xx):
        gg = np.zeros_like(xx)
        if hawkes:
            gg = gg + globals()["grad"](xx, t, theta)[0]
        if bmds_data is not None:
            gg = gg + bmds(xx, bmds_data[0], bmds_data[1])[1]
        return gg

    g = grad(x)
    for _ in range(n_steps):
        p = p + 0.5 * step * g
        x = x + step * minv * p
        if box_lo is not None:
            lo = np.asarray(box_lo, dtype=np.float64)
            hi = np.asarray(box_hi, dtype=np.float64)
            for _r in range(64):  # reflect until inside (bounded)
                below = x < lo
                above = x > hi
                if not (below.any() or above.any()):
                    break
                x = np.where(below, 2 * lo - x, x)
                x = np.where(above, 2 * hi - x, x)
                p = np.where(below | above, -p, p)
        g = grad(x)
        p = p + 0.5 * step * g
    ell = loglik(x, t, theta)[0] if hawkes else 0.0
    if bmds_data is not None:
        ell += bmds(x, bmds_data[0], bmds_data[1], with_grad=False)[0]
    kin = 0.5 * float(np.sum(p * p * minv))
    return x, p, ell, kin


def bmds(x, Y, sigma: float, with_grad: bool = True, with_scale: bool = False):
    """BMDS log density of the dissimilarities Y given locations x (Eq. bmdsLikelihood,
    P:L158-184, normal constant kept) and its gradient in x.  Returns (logp, grad or None)
    or, with_scale, (logp, grad, scale) with scale[n,d] = sum_n' |term_{nn'd}|."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    Y = np.ascontiguousarray(Y, dtype=np.float64)
    N, D = x.shape
    assert Y.shape == (N, N)
    lp = ctypes.c_double()
    g = np.empty((N, D)) if (with_grad or with_scale) else None
    sc = np.empty((N, D)) if with_scale else None
    _check(_load().oracle_bmds(N, D, _dptr(x), _dptr(Y), float(sigma), ctypes.byref(lp), _dptr(g),
                               _dptr(sc)), "bmds")
    return (lp.value, g, sc) if with_scale else (lp.value, g)


def bmds_pair(y: float, delta: float, sigma: float) -> float:
    """r_{nn'} of Eq. bmdsLikelihood plus the normal constant 1/2 log(2 pi sigma^2)."""
    return _load().oracle_bmds_pair(float(y), float(delta), float(sigma))


def philox4x32_10(ctr, key):
    """Philox-4x32-10 block (Salmon et al. 2011) of counter ctr (4 x uint32), key (2 x uint32)."""
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    _load().oracle_philox4x32_10(c, k, o)
    return list(o)


def hmc_normals(seed: int, it: int, n: int) -> np.ndarray:
    """The HMC step's standard normals for iteration it (hawkes_hmc_step's stream)."""
    z = np.empty(n)
    _load().oracle_hmc_normals(seed, it, n, _dptr(z))
    return z


def hmc_uniform(seed: int, it: int) -> float:
    return _load().oracle_hmc_uniform(seed, it)


def hmc_step(x, t, theta, seed: int, it: int, step: float, n_steps: int, inv_mass=None,
             box_lo=None, box_hi=None, bmds_data=None, hawkes: bool = True):
    """One HMC transition (Neal 2011): p = z / sqrt(Minv) with z from the Philox
    stream, leapfrog, accept iff log u < H0 - H1, H = -logpost + 1/2 sum Minv p^2.
    Returns (x_next, accepted, log_alpha)."""
    x = np.asarray(x, dtype=np.float64)
    minv = np.ones_like(x) if inv_mass is None else np.asarray(inv_mass, dtype=np.float64)
    p0 = hmc_normals(seed, it, x.size).reshape(x.shape) / np.sqrt(minv)
    lp0 = (loglik(x, t, theta)[0] if hawkes else 0.0) + \
        (bmds(x, bmds_data[0], bmds_data[1], with_grad=False)[0] if bmds_data is not None else 0.0)
    H0 = -lp0 + 0.5 * float(np.sum(minv * p0 * p0))
    with np.errstate(all="ignore"):
        x1, p1, lp1, k1 = leapfrog(x, p0, t, theta, step, n_steps, inv_mass=inv_mass,
                                   box_lo=box_lo, box_hi=box_hi, bmds_data=bmds_data,
                                   hawkes=hawkes)
    H1 = -lp1 + k1
    # a trajectory that leaves the support or diverges has H1 = +inf (rejected)
    log_alpha = H0 - H1 if (np.isfinite(H1) and np.all(np.abs(x1) <= 1e100)) else -math.inf
    acc = math.log(hmc_uniform(seed, it)) < log_alpha
    return (x1 if acc else x.copy()), acc, log_alpha


# ---- block Metropolis-Hastings over coarsened locations --------------------
# Random numbers: the Philox-4x32-10 block with counter (it_lo, it_hi, b, tag) and key
# (seed_lo, seed_hi); b = block index within the sweep.  Proposal draws for slot q use
# tag = 0x80000000 | q << 12 | a (a = attempt / dimension pair), the accept uniform uses
# tag = 0xC0000000.  Two 53-bit uniforms per block (words 0,1 and 2,3).
_MH_TAG, _MH_ACCEPT = 0x80000000, 0xC0000000
_M32 = 0xFFFFFFFF


def _u53(a: int, b: int) -> float:
    return ((a >> 5) * 67108864.0 + (b >> 6) + 0.5) / 9007199254740992.0


def mh_uniforms(seed: int, it: int, b: int, tag: int):
    w = philox4x32_10([it & _M32, (it >> 32) & _M32, b & _M32, tag & _M32],
                      [seed & _M32, (seed >> 32) & _M32])
    return _u53(w[0], w[1]), _u53(w[2], w[3])


def _Phi(z: float) -> float:
    return 0.5 * math.erfc(-z / math.sqrt(2.0))


def _trunc_mass(x: float, lo: float, hi: float, s: float) -> float:
    """Z(x) = Phi((hi - x)/s) - Phi((lo - x)/s): the N(x, s^2) mass of (lo, hi)."""
    return 1.0 - 0.5 * math.erfc((hi - x) / s / math.sqrt(2.0)) - _Phi((lo - x) / s)


def lens_area(R: float, rho: float, d: float) -> float:
    """Area of the intersection of a disc of radius R and one of radius rho whose centres are
    d apart (the 'asymmetric lens' of P:L248), by the textbook circle-circle formula."""
    if d >= R + rho:
        return 0.0
    if d + rho <= R:
        return math.pi * rho * rho
    if d + R <= rho:
        return math.pi * R * R
    a1 = rho * rho * math.acos((d * d + rho * rho - R * R) / (2.0 * d * rho))
    a2 = R * R * math.acos((d * d + R * R - rho * rho) / (2.0 * d * R))
    k = 0.5 * math.sqrt((-d + rho + R) * (d + rho - R) * (d - rho + R) * (d + rho + R))
    return a1 + a2 - k


MH_MAX_ATTEMPTS = 4096


def mh_propose(kind: str, x_n, centre_n, size_n: float, scale: float, seed: int, it: int,
               b: int, q: int):
    """Proposal for one event and its log Hastings term log q(x|x*) - log q(x*|x).
    square (Eq. locsPrior1): per dimension a N(x_d, (scale*size)^2) draw truncated to
      (c_d - size, c_d + size) by inverting the CDF: z = Phi^-1(Phi(alpha) + u Z), x* = x + s z;
      Hastings prod_d Z_d(x) / Z_d(x*) (the truncation normalisers).
    disc (Eq. circleKernel / locsPrior2): uniform on {|y - c| < r} cap {|y - x| < r eps},
      eps = scale, by rejection from the disc of radius r eps around x; Hastings A(x)/A(x*)
      with A the lens area.  After MH_MAX_ATTEMPTS failed attempts the proposal is x itself."""
    from scipy.special import ndtri   # Phi^-1 (library primitive)
    x_n = np.asarray(x_n, dtype=np.float64)
    D = x_n.size
    if kind == "square":
        s = scale * size_n
        xs = np.empty(D)
        logh = 0.0
        for d in range(D):
            u = mh_uniforms(seed, it, b, _MH_TAG | (q << 12) | (d // 2))[d % 2]
            lo, hi = centre_n[d] - size_n, centre_n[d] + size_n
            alpha = (lo - x_n[d]) / s
            Z0 = _trunc_mass(x_n[d], lo, hi, s)
            z = float(ndtri(_Phi(alpha) + u * Z0))
            xs[d] = min(max(x_n[d] + s * z, lo), hi)
            logh += math.log(Z0) - math.log(_trunc_mass(xs[d], lo, hi, s))
        return xs, logh
    if kind == "disc":
        r, rho = size_n, scale * size_n
        for a in range(MH_MAX_ATTEMPTS):
            u1, u2 = mh_uniforms(seed, it, b, _MH_TAG | (q << 12) | a)
            rad, ang = rho * math.sqrt(u1), 2.0 * math.pi * u2
            y = np.array([x_n[0] + rad * math.cos(ang), x_n[1] + rad * math.sin(ang)])
            if (y[0] - centre_n[0]) ** 2 + (y[1] - centre_n[1]) ** 2 < r * r:
                A0 = lens_area(r, rho, math.hypot(x_n[0] - centre_n[0], x_n[1] - centre_n[1]))
                A1 = lens_area(r, rho, math.hypot(y[0] - centre_n[0], y[1] - centre_n[1]))
                return y, math.log(A0) - math.log(A1)
        return x_n.copy(), 0.0
    raise ValueError(kind)


def mh_sweep(x, t, theta, kind: str, centre, size, blocks, scale: float, seed: int, it: int):
    """Sequential block MH updates: for block b (an array of k distinct events),
    propose all k jointly, log alpha = [ell(X') - ell(X)] + sum log Hastings (uniform priors
    cancel inside the regions), accept iff log u < log alpha.  Returns
    (x_final, accepted list, log_alpha list).  ell by full evaluations (Eq. 1)."""
    x = np.array(x, dtype=np.float64)
    ell = loglik(x, t, theta)[0]
    accs, las = [], []
    for b, blk in enumerate(blocks):
        xp = x.copy()
        logh = 0.0
        for q, n in enumerate(blk):
            xp[n], h = mh_propose(kind, x[n], centre[n], float(size[n]), scale, seed, it, b, q)
            logh += h
        ell1 = loglik(xp, t, theta)[0]
        la = (ell1 - ell) + logh if ell1 > -math.inf else -math.inf
        u = mh_uniforms(seed, it, b, _MH_ACCEPT)[0]
        acc = math.log(u) < la
        if acc:
            x, ell = xp, ell1
        accs.append(acc)
        las.append(la)
    return x, accs, las
