"""Shared helpers for the GPU parity tests: run the CUDA path through the C ABI and
compare with the oracle under the tolerance rule of DESIGN.md ("Parity tolerance")."""
from __future__ import annotations

import functools

import numpy as np
import torch

import oracle

# DESIGN.md "Parity tolerance" (north_star: 1e-9 fp64, 1e-4 fp32, on ell and on every
# gradient component; per-component scale floor for components that cancel)
TOL = {"fp64": (1e-9, 1e-3), "fp32": (1e-4, 1.0)}


def gpu_eval(x, t, theta, precision="fp64", emulate_world=0, with_rates=True, device=0,
             algorithm="auto", ordering="auto"):
    from paper_2010_02994_b200 import HawkesContext
    N, D = x.shape
    with HawkesContext(N, D, device=device, precision=precision, emulate_world=emulate_world,
                       algorithm=algorithm) as ctx:
        ctx.set_ordering(ordering)
        ctx.set_times(torch.from_numpy(np.ascontiguousarray(t)).cuda(device))
        ctx.set_locations(torch.from_numpy(np.ascontiguousarray(x)).cuda(device))
        ctx.set_params(theta)
        ell0 = ctx.loglik()
        rates = ctx.get_rates() if with_rates else None
        if ell0 == -np.inf:
            return ell0, None, rates
        g, ell = ctx.grad_locations()
        torch.cuda.synchronize()
        assert ell == ell0
        return ell, g.cpu().numpy(), rates


@functools.lru_cache(maxsize=64)
def _oracle_cached(key):
    x, t, theta = _REG[key]
    ell, lam, Lam = oracle.loglik(x, t, theta)
    if ell == -np.inf:
        return ell, lam, Lam, None, None
    g, S = oracle.grad(x, t, theta, lam=lam)
    return ell, lam, Lam, g, S


_REG = {}


def oracle_eval(x, t, theta):
    key = (x.tobytes(), t.tobytes(), tuple(theta))
    key = hash(key)
    _REG[key] = (x, t, tuple(theta))
    return _oracle_cached(key)


def assert_parity(ell, g, ell_ref, g_ref, S, precision="fp64", what=""):
    tol, floor = TOL[precision]
    assert abs(ell - ell_ref) <= tol * abs(ell_ref), f"{what}: ell {ell!r} vs oracle {ell_ref!r}"
    bound = tol * np.maximum(np.abs(g_ref), floor * S)
    err = np.abs(g - g_ref)
    bad = err > bound
    assert not bad.any(), (f"{what}: {int(bad.sum())} of {bad.size} gradient components out of "
                           f"tolerance; worst err/bound = {float(np.max(err / bound)):.3g}")
    return float(np.max(err / np.maximum(bound, 1e-300)))
