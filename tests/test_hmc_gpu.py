"""GPU parity of hawkes_hmc_step (Neal 2011): the device Philox stream, the whole
transition (momenta, leapfrog, Metropolis decision) and the chain state against the oracle's
oracle.hmc_step, which draws the same counter-based numbers with its own C Philox."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed,it,n", [(5, 3, 100_001), (2**40 + 7, 2**33 + 5, 4097), (0, 0, 1)])
def test_device_normals_match_oracle(seed, it, n):
    """Same Philox block, same Box-Muller: uniforms are exact integers / 2^53, so the normals
    differ only by the last-ulp rounding of log / sincos."""
    from paper_2010_02994_b200.hawkes import diag_normals
    z = diag_normals(seed, it, n).cpu().numpy()
    zr = oracle.hmc_normals(seed, it, n)
    assert np.max(np.abs(z - zr)) <= 1e-14 * max(1.0, np.abs(zr).max())


def _ctx(c, **kw):
    from paper_2010_02994_b200 import HawkesContext
    ctx = HawkesContext(c.N, c.D, **kw)
    ctx.set_times(c.t)
    ctx.set_locations(c.x)
    ctx.set_params(c.theta)
    return ctx


@pytest.mark.parametrize("mem", ["host", "device"])
def test_hmc_chain_matches_oracle(mem):
    """A 5-transition chain at N=300 with step sizes that give both accepts and rejects:
    the same decisions, log alpha and states as the oracle."""
    c = synth.config("C1", 300)
    steps = [2e-3, 5e-3, 1e-2, 2e-2, 4e-2]
    x_ref = c.x.copy()
    with _ctx(c) as ctx:
        decisions = []
        for it, step in enumerate(steps):
            x_ref, acc_ref, la_ref = oracle.hmc_step(x_ref, c.t, c.theta, 11, it, step, 5)
            x_out = np.empty_like(c.x) if mem == "host" else torch.empty(c.N, c.D, dtype=torch.float64, device="cuda")
            acc, la = ctx.hmc_step(11, it, step, 5, x_out=x_out)
            xg = x_out if mem == "host" else x_out.cpu().numpy()
            assert acc == acc_ref, f"iteration {it}: accepted {acc} vs oracle {acc_ref}"
            assert la == pytest.approx(la_ref, rel=1e-8, abs=1e-9)
            assert np.max(np.abs(xg - x_ref)) <= 1e-9
            decisions.append(acc)
        assert True in decisions and False in decisions
        # the context's state is the chain's: ell matches the oracle at x_ref
        assert ctx.loglik() == pytest.approx(oracle.loglik(x_ref, c.t, c.theta)[0], rel=1e-9)


def test_hmc_mass_and_box_match_oracle():
    """Diagonal inverse mass and the reflecting coarsening box inside the transition."""
    c = synth.config("C1", 250, replicate=2)
    rng = np.random.default_rng(3)
    minv = rng.uniform(0.5, 2.0, size=c.x.shape)
    lo, hi = c.x - 0.01, c.x + 0.01
    x_ref = c.x.copy()
    with _ctx(c) as ctx:
        for it in range(3):
            x_ref, acc_ref, la_ref = oracle.hmc_step(x_ref, c.t, c.theta, 21, it, 4e-3, 6, inv_mass=minv,
                                                     box_lo=lo, box_hi=hi)
            x_out = np.empty_like(c.x)
            acc, la = ctx.hmc_step(21, it, 4e-3, 6, inv_mass=minv, box_lo=lo, box_hi=hi, x_out=x_out)
            assert acc == acc_ref and la == pytest.approx(la_ref, rel=1e-8, abs=1e-9)
            assert np.max(np.abs(x_out - x_ref)) <= 1e-9
            assert np.all(x_out >= lo) and np.all(x_out <= hi)


def test_hmc_bmds_joint_potential_matches_oracle():
    """The flu model's joint potential -(ell + log p(Y | X))."""
    c, Y, s = synth.flu_shaped(200, 3)
    x_ref = c.x.copy()
    with _ctx(c) as ctx:
        ctx.set_bmds(Y, s)
        ctx.set_potential(hawkes=True, bmds=True)
        for it in range(3):
            x_ref, acc_ref, la_ref = oracle.hmc_step(x_ref, c.t, c.theta, 8, it, 2e-3, 4,
                                                     bmds_data=(Y, s))
            x_out = np.empty_like(c.x)
            acc, la = ctx.hmc_step(8, it, 2e-3, 4, x_out=x_out)
            assert acc == acc_ref and la == pytest.approx(la_ref, rel=1e-8, abs=1e-8)
            assert np.max(np.abs(x_out - x_ref)) <= 1e-9 * np.abs(x_ref).max()


def test_hmc_divergent_trajectory_is_rejected():
    """A huge step sends x off to |x| > 1e100 / NaN: rejected, log alpha = -inf, no error, and
    the chain stays at x0 with a usable context."""
    c = synth.config("C1", 200)
    ell0 = oracle.loglik(c.x, c.t, c.theta)[0]
    with _ctx(c) as ctx:
        x_out = np.empty_like(c.x)
        acc, la = ctx.hmc_step(1, 0, 1e120, 3, x_out=x_out)
        assert not acc and la == -np.inf
        assert np.array_equal(x_out, c.x)
        assert ctx.loglik() == pytest.approx(ell0, rel=1e-9)
        acc, la = ctx.hmc_step(1, 1, 2e-3, 3)
        assert np.isfinite(la)


def test_hmc_rows_world_emulation_is_bitwise_identical():
    """ROWS decomposition: the transition is the same for emulated world 1 and 3 (rows
    summed in a W-independent order; the random stream depends on (seed, it) only)."""
    c = synth.config("C1", 700)
    outs = []
    for W in (0, 3):
        with _ctx(c, emulate_world=W, algorithm="rows") as ctx:
            res = []
            for it in range(3):
                x_out = np.empty_like(c.x)
                res.append((ctx.hmc_step(4, it, 3e-3, 4, x_out=x_out), x_out))
            outs.append(res)
    for (a, xa), (b, xb) in zip(*outs):
        assert a == b and np.array_equal(xa, xb)


def test_hmc_errors():
    from paper_2010_02994_b200 import HawkesContext, HawkesError
    c = synth.config("C1", 100)
    with HawkesContext(c.N, c.D) as ctx:
        with pytest.raises(HawkesError, match="STATE"):
            ctx.hmc_step(1, 0, 1e-3, 2)        # no locations
        ctx.set_times(c.t)
        ctx.set_locations(c.x)
        ctx.set_params(c.theta)
        with pytest.raises(HawkesError, match="ARG"):
            ctx.hmc_step(1, 0, float("nan"), 2)
        with pytest.raises(HawkesError, match="ARG"):
            ctx.hmc_step(1, 0, 1e-3, 2, inv_mass=-np.ones_like(c.x))
        with pytest.raises(HawkesError, match="ARG"):
            ctx.hmc_step(1, 0, 1e-3, 2, box_lo=c.x - 1)
