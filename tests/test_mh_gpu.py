"""GPU parity of the on-device block Metropolis-Hastings sweep (hawkes_mh_sweep):
proposals (truncated normals in the DC squares, lens-uniform in the Alaska discs), Hastings
terms, Delta ell, the Metropolis decisions and the final state against oracle.mh_sweep, which
draws the same Philox numbers with its own generator and takes Delta ell from two full
evaluations of Eq. 1."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


def _ctx(c, **kw):
    from paper_2010_02994_b200 import HawkesContext
    ctx = HawkesContext(c.N, c.D, **kw)
    ctx.set_times(c.t)
    ctx.set_locations(c.x)
    ctx.set_params(c.theta)
    ctx.set_regions(c.region, c.centre, c.size)
    return ctx


def _blocks(N, n_blocks, k, seed):
    rng = np.random.default_rng(seed)
    return np.stack([rng.choice(N, size=k, replace=False) for _ in range(n_blocks)]).astype(np.int32)


@pytest.mark.parametrize("name,scale,k", [("C2", 0.5, 8), ("C2", 1.5, 1), ("C3", 0.7, 8),
                                          ("C3", 1.0, 32)])
def test_mh_sweep_matches_oracle(name, scale, k):
    c = synth.config(name, 400)
    blocks = _blocks(c.N, 12, k, 5)
    x_ref, acc_ref, la_ref = oracle.mh_sweep(c.x, c.t, c.theta, c.region, c.centre, c.size,
                                             blocks, scale, 77, 3)
    with _ctx(c) as ctx:
        acc, la = ctx.mh_sweep(blocks, scale, 77, 3)
        x = ctx.get_locations().cpu().numpy()
        ell = ctx.loglik()
    for b in range(len(blocks)):
        assert la[b] == pytest.approx(la_ref[b], rel=1e-7, abs=1e-7), f"block {b}"
        if abs(la_ref[b] - np.log(oracle.mh_uniforms(77, 3, b, 0xC0000000)[0])) > 1e-6:
            assert acc[b] == acc_ref[b], f"block {b}"
    assert list(acc) == list(acc_ref)
    scale_x = np.abs(c.x).max()
    assert np.max(np.abs(x - x_ref)) <= 1e-12 * scale_x
    assert ell == pytest.approx(oracle.loglik(x_ref, c.t, c.theta)[0], rel=1e-9)
    # every location stays in its region
    if c.region == "square":
        assert np.all(np.abs(x - c.centre) <= c.size[:, None])
    else:
        assert np.all(np.hypot(*(x - c.centre).T) < c.size)


def test_mh_sweeps_chain_and_mix_with_other_calls():
    """Consecutive sweeps (new iteration numbers) continue from the committed state, and a
    gradient afterwards is that of the chain's state."""
    c = synth.config("C2", 300, replicate=1)
    x_ref = c.x.copy()
    with _ctx(c) as ctx:
        for it in range(3):
            blocks = _blocks(c.N, 6, 4, it)
            x_ref, acc_ref, _ = oracle.mh_sweep(x_ref, c.t, c.theta, "square", c.centre, c.size,
                                                blocks, 0.6, 1, it)
            acc, _ = ctx.mh_sweep(blocks, 0.6, 1, it)
            assert list(acc) == list(acc_ref)
        g, ell = ctx.grad_locations()
        g_ref, _ = oracle.grad(x_ref, c.t, c.theta)
        assert np.max(np.abs(g.cpu().numpy() - g_ref)) <= 1e-9 * np.abs(g_ref).max()


def test_mh_sweep_rows_world_emulation_identical():
    """The sweep's decisions do not depend on the decomposition or the emulated world."""
    c = synth.config("C3", 500)
    blocks = _blocks(c.N, 8, 8, 2)
    res = []
    for kw in ({}, {"algorithm": "rows", "emulate_world": 3}, {"algorithm": "pairs", "emulate_world": 2}):
        with _ctx(c, **kw) as ctx:
            acc, la = ctx.mh_sweep(blocks, 0.8, 4, 0)
            res.append((acc, la, ctx.get_locations().cpu().numpy()))
    for acc, la, x in res[1:]:
        assert np.array_equal(acc, res[0][0])
        assert np.allclose(la, res[0][1], rtol=1e-9, atol=1e-9)
        assert np.allclose(x, res[0][2], rtol=0, atol=1e-12 * np.abs(x).max())


def test_mh_errors():
    from paper_2010_02994_b200 import HawkesContext, HawkesError
    c = synth.config("C2", 100)
    with HawkesContext(c.N, c.D) as ctx:
        ctx.set_times(c.t)
        ctx.set_locations(c.x)
        ctx.set_params(c.theta)
        with pytest.raises(HawkesError, match="STATE"):
            ctx.mh_sweep([[0, 1]], 0.5, 1, 0)
        ctx.set_regions("square", c.centre, c.size)
        with pytest.raises(HawkesError, match="ARG"):
            ctx.mh_sweep([[0, 0]], 0.5, 1, 0)      # repeated index
        with pytest.raises(HawkesError, match="ARG"):
            ctx.mh_sweep([[0, 100]], 0.5, 1, 0)    # out of range
        with pytest.raises(HawkesError, match="ARG"):
            ctx.mh_sweep([[0, 1]], 0.0, 1, 0)
        with pytest.raises(HawkesError, match="NONFINITE"):
            ctx.set_regions("square", c.centre, np.zeros(c.N))
    c1 = synth.config("C1", 50, )
    with HawkesContext(c1.N, 3) as ctx:
        with pytest.raises(HawkesError, match="DIM"):
            ctx.set_regions("disc", np.zeros((c1.N, 3)), np.ones(c1.N))


def test_mh_sweep_graph_replay_matches_plain_launches(monkeypatch):
    """A sweep of >= 8 blocks replays one captured block step; with HAWKES_NO_GRAPHS it runs
    plain launches.  Same kernels, same order: bitwise identical decisions and states."""
    c = synth.config("C3", 600)
    blocks = _blocks(c.N, 24, 4, 9)
    res = []
    for plain in (False, True):
        if plain:
            monkeypatch.setenv("HAWKES_NO_GRAPHS", "1")
        with _ctx(c) as ctx:
            acc, la = ctx.mh_sweep(blocks, 0.8, 6, 2)
            res.append((acc, la, ctx.get_locations().cpu().numpy()))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])


def test_mh_sweep_recaptures_on_k_and_params_change():
    """The captured step bakes in k and the folded constants: a sweep with another k, and one
    after set_params, must match the oracle with the new values."""
    c = synth.config("C2", 400, replicate=2)
    theta2 = tuple(v * f for v, f in zip(c.theta, (1.1, 0.9, 1.2, 0.8, 1.0, 1.05)))
    x_ref = c.x.copy()
    with _ctx(c) as ctx:
        b1 = _blocks(c.N, 10, 2, 1)
        x_ref, a_ref, _ = oracle.mh_sweep(x_ref, c.t, c.theta, "square", c.centre, c.size, b1, 0.5, 3, 0)
        acc, _ = ctx.mh_sweep(b1, 0.5, 3, 0)
        assert list(acc) == list(a_ref)
        b2 = _blocks(c.N, 10, 5, 2)
        x_ref, a_ref, _ = oracle.mh_sweep(x_ref, c.t, c.theta, "square", c.centre, c.size, b2, 0.5, 3, 1)
        acc, _ = ctx.mh_sweep(b2, 0.5, 3, 1)
        assert list(acc) == list(a_ref)
        ctx.set_params(theta2)
        b3 = _blocks(c.N, 10, 5, 3)
        x_ref, a_ref, la_ref = oracle.mh_sweep(x_ref, c.t, theta2, "square", c.centre, c.size, b3, 0.5, 3, 2)
        acc, la = ctx.mh_sweep(b3, 0.5, 3, 2)
        assert list(acc) == list(a_ref)
        assert np.allclose(la, la_ref, rtol=1e-7, atol=1e-7)
        assert np.max(np.abs(ctx.get_locations().cpu().numpy() - x_ref)) <= 1e-12 * np.abs(x_ref).max()


@pytest.mark.parametrize("name,k,nb", [("C2", 1, 30), ("C3", 8, 20), ("C2", 32, 6)])
def test_mh_sweep_cooperative_kernel_matches_launch_path(monkeypatch, name, k, nb):
    """The persistent cooperative sweep (HAWKES_MH_COOP=1; default for k <= 8) and the
    launch-based block step (HAWKES_MH_COOP=0) use the same arithmetic and reduction orders:
    bitwise identical decisions, log alphas, locations and rates."""
    c = synth.config(name, 900)
    blocks = _blocks(c.N, nb, k, 4)
    res = []
    for coop in (True, False):
        monkeypatch.setenv("HAWKES_MH_COOP", "1" if coop else "0")
        with _ctx(c) as ctx:
            acc, la = ctx.mh_sweep(blocks, 0.7, 12, 5)
            lam = ctx.get_rates()["lambda"]
            res.append((acc, la, ctx.get_locations().cpu().numpy(), lam))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])
    assert np.array_equal(res[0][3], res[1][3])


def test_samplers_in_fp32_contexts():
    """fp32 contexts: the sweep's Delta ell comes from fp32-accurate cached rates and the
    commits update the fp32 records too; decisions agree with the oracle wherever log u is not
    within the fp32 error of log alpha, and a later fp32 evaluation sees the chain's state.
    (A dense catalog: in sparse ones an isolated event's rate underflows fp32's range,
    reading R23, and ell is -inf there.)"""
    c0 = synth.config("C1", 500)
    centre = 0.01 * np.round(c0.x / 0.01)                 # 0.01-boxes (Eq. locsPrior1 style)
    c = synth.Catalog(c0.x, c0.t, c0.theta, "C1-boxed", c0.seed, "square", centre,
                      np.full(c0.N, 0.005))
    blocks = _blocks(c.N, 16, 2, 8)
    x_ref, acc_ref, la_ref = oracle.mh_sweep(c.x, c.t, c.theta, "square", c.centre, c.size, blocks,
                                             0.6, 5, 1)
    with _ctx(c, precision="fp32") as ctx:
        acc, la = ctx.mh_sweep(blocks, 0.6, 5, 1)
        for b in range(len(blocks)):
            lu = np.log(oracle.mh_uniforms(5, 1, b, 0xC0000000)[0])
            if abs(la_ref[b] - lu) > 1e-3:
                assert acc[b] == acc_ref[b], b
            assert la[b] == pytest.approx(la_ref[b], abs=1e-3)
        x = ctx.get_locations().cpu().numpy()
        if list(acc) == list(acc_ref):
            assert np.max(np.abs(x - x_ref)) <= 1e-12
            assert ctx.loglik() == pytest.approx(oracle.loglik(x_ref, c.t, c.theta)[0], rel=1e-5)
        acc_h, la_h = ctx.hmc_step(3, 0, 1e-3, 3)
        assert np.isfinite(la_h)


@pytest.mark.parametrize("D", [1, 3])
def test_mh_sweep_square_regions_other_dimensions(D):
    """Square regions (Eq. locsPrior1) in D = 1 and 3: truncated normals per dimension."""
    c0 = synth.unit_square(400, config=31, D=D)
    centre = 0.02 * np.round(c0.x / 0.02)
    c = synth.Catalog(c0.x, c0.t, c0.theta, f"boxed D={D}", c0.seed, "square", centre, np.full(c0.N, 0.01))
    blocks = _blocks(c.N, 10, 3, 2)
    x_ref, acc_ref, la_ref = oracle.mh_sweep(c.x, c.t, c.theta, "square", c.centre, c.size, blocks, 0.7, 4, 0)
    with _ctx(c) as ctx:
        acc, la = ctx.mh_sweep(blocks, 0.7, 4, 0)
        x = ctx.get_locations().cpu().numpy()
    assert list(acc) == list(acc_ref)
    assert np.allclose(la, la_ref, rtol=1e-7, atol=1e-7)
    assert np.max(np.abs(x - x_ref)) <= 1e-12


def test_samplers_tiny_and_degenerate_catalogs():
    """N = 2: both samplers against the oracle.  N = 1: ell = -inf (reading R11); the HMC
    transition reports GRAD_UNDEFINED, the MH sweep rejects (-inf - -inf is not a gain)."""
    from paper_2010_02994_b200 import HawkesContext, HawkesError
    x2 = np.array([[0.40, 0.50], [0.43, 0.52]])
    t2 = np.array([0.1, 0.3])
    th = (0.6, 0.1, 0.1, 0.4, 20.0, 0.03)
    xr, acc_r, la_r = oracle.hmc_step(x2, t2, th, 6, 0, 1e-3, 5)
    with HawkesContext(2, 2) as ctx:
        ctx.set_times(t2)
        ctx.set_locations(x2)
        ctx.set_params(th)
        out = np.empty_like(x2)
        acc, la = ctx.hmc_step(6, 0, 1e-3, 5, x_out=out)
        assert acc == acc_r and la == pytest.approx(la_r, rel=1e-8, abs=1e-10)
        assert np.max(np.abs(out - xr)) <= 1e-12
        ctx.set_locations(x2)
        centre = np.round(x2, 1)
        ctx.set_regions("square", centre, np.full(2, 0.05))
        x_ref, a_ref, l_ref = oracle.mh_sweep(x2, t2, th, "square", centre, np.full(2, 0.05),
                                              [[0], [1], [0, 1]][:2], 0.5, 1, 0)
        acc2, la2 = ctx.mh_sweep(np.array([[0], [1]], dtype=np.int32), 0.5, 1, 0)
        assert list(acc2) == list(a_ref) and np.allclose(la2, l_ref, rtol=1e-8, atol=1e-10)
    with HawkesContext(1, 2) as ctx:
        ctx.set_times(np.array([0.5]))
        ctx.set_locations(np.array([[0.2, 0.2]]))
        ctx.set_params(th)
        assert ctx.loglik() == -np.inf
        with pytest.raises(HawkesError, match="GRAD_UNDEFINED"):
            ctx.hmc_step(1, 0, 1e-3, 2)
        ctx.set_regions("square", np.array([[0.2, 0.2]]), np.array([0.05]))
        acc, la = ctx.mh_sweep(np.array([[0]], dtype=np.int32), 0.5, 1, 0)
        assert not acc[0] and la[0] == -np.inf
