"""Reading R23, oracle side: where a rate's terms have exp factors in the
subnormal range, the oracle's literal unscaled evaluation (c * exp(.)) loses
precision, and the fuzz harness counts such cases apart.  These CPU tests pin the tools that
decide it: tools/mp_check_case.py's 30-digit App. A evaluation against mp.diff of ell
(tests/mp_brute.py), and a tiny catalog whose background exp factors are ~1e-315 -- the oracle's
rates drift from the 30-digit ones there, and the fuzz floor flags the case."""
from __future__ import annotations

import importlib.util
import os

import numpy as np
import pytest

import oracle
from tests import mp_brute

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tool(name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "tools", f"{name}.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_mp_truth_matches_numerical_derivative_of_ell():
    """The 30-digit App. A gradient of the check tool equals 40-digit mp.diff of Eq. 1."""
    mc = _tool("mp_check_case")
    rng = np.random.default_rng(7)
    N, D = 5, 2
    x = rng.uniform(0, 1, size=(N, D))
    t = np.sort(rng.uniform(0, 1, size=N))
    th = (0.7, 0.4, 0.3, 0.5, 3.0, 0.2)
    lam, g = mc.mp_truth(x, t, th)
    ref = mp_brute.evaluate(x.tolist(), t.tolist(), th)
    np.testing.assert_allclose(lam, [float(v) for v in ref["lam"]], rtol=1e-15)
    gref = np.array([[float(v) for v in r] for r in ref["grad"]])
    np.testing.assert_allclose(g, gref, rtol=1e-13, atol=1e-13 * np.abs(gref).max())


def _subnormal_catalog():
    """D = 8, tau_x = 0.003 (c_b ~ 1e15): three events ~0.114 apart, so each background term
    is c_b * e^-725 ~ 1e-300 with an exp factor ~1e-315 (subnormal); theta = 0 (reading R22)."""
    D = 8
    x = np.zeros((3, D))
    x[1, 0] = 0.1142
    x[2, 1] = 0.1139
    t = np.array([0.0, 0.001, 0.002])
    th = (0.7, 0.003, 0.5, 0.0, 1.0, 0.01)
    return x, t, th


def test_oracle_rates_drift_where_exp_factors_are_subnormal():
    mc = _tool("mp_check_case")
    x, t, th = _subnormal_catalog()
    lam_mp, _ = mc.mp_truth(x, t, th)
    _, lam_o, _ = oracle.loglik(x, t, th)
    assert np.all(lam_mp > 1e-305) and np.all(lam_mp < 1e-290)          # normal rates...
    rel = np.abs(lam_o - lam_mp) / lam_mp
    assert rel.max() > 1e-12                                              # ...off in the oracle
    fz = _tool("fuzz_parity")
    assert lam_o.min() < fz.oracle_subnormal_floor(th, x.shape[1], len(t))   # and flagged


@pytest.mark.parametrize("name,N", [("C1", 500), ("C4", 3000)])
def test_subnormal_floor_leaves_the_configs_alone(name, N):
    """The floor sits far below every rate of the workload configs: none is counted apart."""
    import synth
    c = synth.config(name, N=N)
    _, lam, _ = oracle.loglik(c.x, c.t, c.theta)
    assert lam.min() > 1e6 * _tool("fuzz_parity").oracle_subnormal_floor(c.theta, c.D, c.N)
