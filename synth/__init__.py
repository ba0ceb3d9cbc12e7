"""Seeded synthetic event catalogs shared by the oracle tests, the GPU tests and bench.py.

This module only *draws inputs*: it holds none of the likelihood's arithmetic
(no rates, no kernels, no gradients), so sharing it does not couple the oracle
and the CUDA path.  The recipe is a simplified
version of the cluster (branching) simulation the paper uses for its
simulation study (App. C; Zhuang et al. 2004): background events
first, then offspring at t_parent + Exp(omega) and x_parent + N(0, h^2 I),
then a sort by time.  Shapes and parameters follow SURVEY.md §8(d):

  C1  N=500,  D=2, unit square x [0,1) time           (BASELINE configs[0])
  C2  N=5k,   DC-gunfire-shaped, metres / hours, 100 m coarsening boxes
  C3  N=20k,  Alaska-wildfire-shaped, km / days, mixed coarsening radii
  C4  N=100k..1M, as C1 (the scaling sweep; bench workload at N=100k)
  C5  N=50k,  as C1 (HMC trajectories)

Random numbers come from numpy's counter-based Philox-4x32-10 generator with
seed 20102994 + 100*config + replicate.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

# Theta = (mu0, tau_x, tau_t, theta, omega, h)  -- paper order
THETA_UNIT = (0.6, 0.1, 0.1, 0.4, 20.0, 0.03)
# DC full-model posterior medians (Table; readings R20, R21)
THETA_DC = (0.89, 98.1, 1763.7, 0.11, 111.1, 61.4)
# Alaska full-model posterior medians (Table; reading R20)
THETA_AK = (0.66, 34.8, 25.9, 0.34, 0.909, 11.1)


@dataclass
class Catalog:
    x: np.ndarray          # N x D float64, row-major
    t: np.ndarray          # N float64, non-decreasing, >= 0
    theta: Tuple[float, ...]
    name: str
    seed: int
    # coarsening regions the locations were drawn in (C2: squares, C3: discs), else None
    region: Optional[str] = None        # "square" | "disc"
    centre: Optional[np.ndarray] = None  # N x D observed locations (box / disc centres)
    size: Optional[np.ndarray] = None    # N: square half-width or disc radius

    @property
    def N(self) -> int:
        return int(self.t.shape[0])

    @property
    def D(self) -> int:
        return int(self.x.shape[1])


def _rng(config: int, replicate: int) -> Tuple[np.random.Generator, int]:
    seed = 20102994 + 100 * config + replicate
    return np.random.Generator(np.random.Philox(seed)), seed


def _cluster(rng, n_total: int, n_bg: int, bg_x, bg_t, omega: float, h: float, horizon: float):
    """Background events, then offspring of uniformly drawn parents (App. C)."""
    xs = [bg_x]
    ts = [bg_t]
    have = n_bg
    X = bg_x
    T = bg_t
    while have < n_total:
        need = n_total - have
        m = max(need, 16)
        par = rng.integers(0, X.shape[0], size=m)
        ct = T[par] + rng.exponential(1.0 / omega, size=m)
        cx = X[par] + rng.normal(0.0, h, size=(m, X.shape[1]))
        keep = ct < horizon
        ct, cx = ct[keep][:need], cx[keep][:need]
        xs.append(cx)
        ts.append(ct)
        have += ct.shape[0]
        X = np.concatenate(xs)
        T = np.concatenate(ts)
    order = np.argsort(T, kind="stable")
    return np.ascontiguousarray(X[order]), np.ascontiguousarray(T[order])


def unit_square(N: int, config: int = 1, replicate: int = 0, D: int = 2,
                theta: Tuple[float, ...] = THETA_UNIT) -> Catalog:
    """C1 / C4 / C5: uniform background on [0,1]^D x [0,1), 40% offspring."""
    rng, seed = _rng(config, replicate)
    n_bg = max(1, int(round(0.6 * N)))
    bx = rng.uniform(0.0, 1.0, size=(n_bg, D))
    bt = rng.uniform(0.0, 1.0, size=n_bg)
    x, t = _cluster(rng, N, n_bg, bx, bt, theta[4], theta[5], 1.0)
    return Catalog(x, t, tuple(theta), f"unit_square_N{N}_D{D}", seed)


def dc_shaped(N: int = 5000, replicate: int = 0) -> Catalog:
    """C2: DC-gunfire-shaped.  16 x 16 km in metres (centred), 25 Gaussian hot
    spots (sd 400 m) + 20% uniform background, hours in [0, 8760), 11% offspring,
    then coarsening to 100 m boxes (Eq. locsPrior1): the catalog's
    locations are box centre + U(-50, 50)^2."""
    rng, seed = _rng(2, replicate)
    theta = THETA_DC
    n_bg = int(round(0.89 * N))
    n_uni = int(round(0.2 * n_bg))
    centres = rng.uniform(-6000.0, 6000.0, size=(25, 2))
    pick = rng.integers(0, 25, size=n_bg - n_uni)
    bx = np.concatenate([centres[pick] + rng.normal(0.0, 400.0, size=(n_bg - n_uni, 2)),
                         rng.uniform(-8000.0, 8000.0, size=(n_uni, 2))])
    bt = rng.uniform(0.0, 8760.0, size=n_bg)
    x, t = _cluster(rng, N, n_bg, bx, bt, theta[4], theta[5], 8760.0)
    box = 100.0 * np.round(x / 100.0)
    x = box + rng.uniform(-50.0, 50.0, size=x.shape)
    return Catalog(np.ascontiguousarray(x), t, theta, f"dc_shaped_N{N}", seed, "square",
                   np.ascontiguousarray(box), np.full(N, 50.0))


def alaska_shaped(N: int = 20000, replicate: int = 0) -> Catalog:
    """C3: Alaska-wildfire-shaped.  2400 x 1400 km (centred), 40 hot spots
    (sd 60 km), days in [0, 1826) with a seasonal peak per year (day ~ N(190, 25)),
    34% offspring, then coarsening radii r_n (60% at 0.01 km, 40% Pareto(0.01,
    1.06) clipped at 4.42 km) and locations uniform in disc(centre, r_n)
    (Eq. locsPrior2)."""
    rng, seed = _rng(3, replicate)
    theta = THETA_AK
    n_bg = int(round(0.66 * N))
    centres = np.column_stack([rng.uniform(-1200.0, 1200.0, 40), rng.uniform(-700.0, 700.0, 40)])
    pick = rng.integers(0, 40, size=n_bg)
    bx = centres[pick] + rng.normal(0.0, 60.0, size=(n_bg, 2))
    year = rng.integers(0, 5, size=n_bg)
    day = np.clip(rng.normal(190.0, 25.0, size=n_bg), 0.0, 364.0)
    bt = np.minimum(365.2 * year + day, 1825.999)
    x, t = _cluster(rng, N, n_bg, bx, bt, theta[4], theta[5], 1826.0)
    r = np.where(rng.uniform(size=N) < 0.6, 0.01,
                 np.minimum(0.01 * (1.0 - rng.uniform(size=N)) ** (-1.0 / 1.06), 4.42))
    ang = rng.uniform(0.0, 2 * np.pi, size=N)
    rad = r * np.sqrt(rng.uniform(size=N))
    centre = x
    x = x + np.column_stack([rad * np.cos(ang), rad * np.sin(ang)])
    return Catalog(np.ascontiguousarray(x), t, theta, f"alaska_shaped_N{N}", seed, "disc",
                   np.ascontiguousarray(centre), np.ascontiguousarray(r))


def with_ties(N: int, ndistinct: int, replicate: int = 0, D: int = 2) -> Catalog:
    """Unit-square catalog whose times are rounded onto ``ndistinct`` levels,
    so many events share a timestamp (tests the indicators of P:L82)."""
    c = unit_square(N, config=9, replicate=replicate, D=D)
    t = np.floor(c.t * ndistinct) / ndistinct
    order = np.argsort(t, kind="stable")
    return Catalog(np.ascontiguousarray(c.x[order]), np.ascontiguousarray(t[order]), c.theta,
                   f"ties_N{N}_k{ndistinct}", c.seed)


def config(name: str, N: Optional[int] = None, replicate: int = 0) -> Catalog:
    """Catalog for a BASELINE config id (C1..C5); N overrides the size."""
    name = name.upper()
    if name == "C1":
        return unit_square(N or 500, config=1, replicate=replicate)
    if name == "C2":
        return dc_shaped(N or 5000, replicate)
    if name == "C3":
        return alaska_shaped(N or 20000, replicate)
    if name == "C4":
        return unit_square(N or 100_000, config=4, replicate=replicate)
    if name == "C5":
        return unit_square(N or 50_000, config=5, replicate=replicate)
    raise KeyError(name)


def momenta(N: int, D: int, seed: int = 7) -> np.ndarray:
    """Standard normal momenta for HMC tests / benches (Philox)."""
    return np.random.Generator(np.random.Philox(seed)).normal(size=(N, D))


def bmds_dissimilarities(x: np.ndarray, sigma: float, seed: int = 0) -> np.ndarray:
    """Synthetic BMDS data for latent locations x (N x D): y_nn' ~ N(|x_n - x_n'|, sigma^2)
    truncated to y > 0 (rejection), symmetric, zero diagonal (P:L171-173 data model)."""
    rng = np.random.Generator(np.random.Philox(seed))
    N = x.shape[0]
    diff = x[:, None, :] - x[None, :, :]
    delta = np.sqrt(np.sum(diff * diff, axis=-1))
    Y = np.zeros((N, N))
    iu = np.triu_indices(N, 1)
    d = delta[iu]
    y = d + sigma * rng.normal(size=d.shape)
    bad = y <= 0
    while bad.any():
        y[bad] = d[bad] + sigma * rng.normal(size=int(bad.sum()))
        bad = y <= 0
    Y[iu] = y
    Y[(iu[1], iu[0])] = y
    return Y


def flu_shaped(N: int = 4733, D: int = 6, sigma: float = 0.3, replicate: int = 0):
    """Flu-shaped synthetic BMDS + Hawkes workload (N = 4733 cases, latent D = 6):
    latent locations from a 64-country Gaussian mixture in R^D, days over 12 years, and
    dissimilarities drawn from the BMDS data model.  Returns (Catalog, Y, sigma)."""
    rng, seed = _rng(6, replicate)
    centres = rng.normal(0.0, 3.0, size=(64, D))
    pick = rng.integers(0, 64, size=N)
    x = centres[pick] + rng.normal(0.0, 0.5, size=(N, D))
    t = np.sort(rng.uniform(0.0, 4383.0, size=N))
    theta = (0.5, 2.0, 60.0, 0.5, 0.1, 0.5)
    Y = bmds_dissimilarities(x, sigma, seed=seed)
    return Catalog(np.ascontiguousarray(x), t, theta, f"flu_shaped_N{N}_D{D}", seed), Y, sigma
