"""BMDS log density and gradient (Eq. bmdsLikelihood)
on the GPU against the oracle, and the flu model's joint HMC potential."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def _ctx(c, Y, s):
    from paper_2010_02994_b200 import HawkesContext
    ctx = HawkesContext(c.N, c.D)
    ctx.set_times(c.t)
    ctx.set_locations(c.x)
    ctx.set_params(c.theta)
    ctx.set_bmds(Y, s)
    return ctx


@pytest.mark.parametrize("N,D,device_y", [(500, 6, False), (777, 2, True), (4733, 6, True), (300, 8, False)])
def test_bmds_matches_oracle(N, D, device_y):
    """Includes the flu shape itself: N = 4733 cases, latent D = 6."""
    c, Y, s = synth.flu_shaped(N, D)
    lp_ref, g_ref, S = oracle.bmds(c.x, Y, s, with_scale=True)
    with _ctx(c, torch.from_numpy(Y).cuda() if device_y else Y, s) as ctx:
        lp, g = ctx.bmds_logdensity()
        g = g.cpu().numpy()
    assert abs(lp - lp_ref) <= 1e-11 * abs(lp_ref)
    assert np.all(np.abs(g - g_ref) <= 1e-9 * np.maximum(np.abs(g_ref), 1e-3 * S))


def test_bmds_reads_the_lower_triangle():
    """Only y_{nn'} with n > n' enters (Eq. bmdsLikelihood): garbage above the diagonal
    changes nothing."""
    c, Y, s = synth.flu_shaped(200, 3)
    Yg = Y.copy()
    iu = np.triu_indices(200, 1)
    Yg[iu] = -7.0
    with _ctx(c, Y, s) as a, _ctx(c, Yg, s) as b:
        la, ga = a.bmds_logdensity()
        lb, gb = b.bmds_logdensity()
        assert la == lb and torch.equal(ga, gb)


def test_joint_potential_leapfrog_matches_oracle():
    """hawkes_leapfrog with U = -(ell + log p(Y|X)) against the oracle's literal leapfrog,
    and with U = -log p(Y|X) alone."""
    c, Y, s = synth.flu_shaped(300, 3)
    p0 = synth.momenta(c.N, c.D, seed=3)
    for hawkes in (True, False):
        xr, pr, er, kr = oracle.leapfrog(c.x, p0, c.t, c.theta, 2e-3, 10, bmds_data=(Y, s), hawkes=hawkes)
        with _ctx(c, Y, s) as ctx:
            ctx.set_potential(hawkes=hawkes, bmds=True)
            x = torch.from_numpy(c.x.copy()).cuda()
            p = torch.from_numpy(p0.copy()).cuda()
            _, _, e, k = ctx.leapfrog(x, p, 2e-3, 10)
            assert np.max(np.abs(x.cpu().numpy() - xr)) <= 1e-9 * np.abs(xr).max()
            assert e == pytest.approx(er, rel=1e-9)
            assert k == pytest.approx(kr, rel=1e-9)
            # the context's locations are the trajectory's end: BMDS at x_end
            lp, _ = ctx.bmds_logdensity(grad=False)
            assert lp == pytest.approx(oracle.bmds(xr, Y, s, with_grad=False)[0], rel=1e-10)


def test_bmds_errors():
    from paper_2010_02994_b200 import HawkesError
    c, Y, s = synth.flu_shaped(50, 2)
    with _ctx(c, Y, s) as ctx:
        with pytest.raises(HawkesError) as ei:
            ctx.set_bmds(Y, -1.0)
        assert ei.value.status == "HAWKES_ERR_PARAM"
        Yb = Y.copy()
        Yb[7, 3] = 0.0
        with pytest.raises(HawkesError) as ei:
            ctx.set_bmds(Yb, s)
        assert ei.value.status == "HAWKES_ERR_NONFINITE"
        ctx.set_bmds(torch.from_numpy(Yb).cuda(), s)       # device input: reported later
        with pytest.raises(HawkesError) as ei:
            ctx.bmds_logdensity()
        assert ei.value.status == "HAWKES_ERR_NONFINITE"
