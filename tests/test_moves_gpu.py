"""Block Metropolis-Hastings moves (hawkes_propose_move / hawkes_accept_move; P:L245,
SURVEY.md §8(f) NEXT-3) against the oracle: Delta ell = ell(X') - ell(X) = sum_n
log(lambda_n' / lambda_n) (Lambda_n has no x), computed from the oracle's own rates."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def _oracle_delta(x, x2, t, theta):
    lam, _, _ = oracle.rates(x, t, theta)
    lam2, _, _ = oracle.rates(x2, t, theta)
    with np.errstate(divide="ignore"):
        terms = np.log(lam2) - np.log(lam)
    return math.fsum(terms), float(np.sum(np.abs(terms)))


def _ctx(c, **kw):
    from paper_2010_02994_b200 import HawkesContext
    ctx = HawkesContext(c.N, c.D, **kw)
    ctx.set_times(c.t)
    ctx.set_locations(c.x)
    ctx.set_params(c.theta)
    return ctx


@pytest.mark.parametrize("name,k,scale", [("C1", 1, 0.01), ("C1", 7, 0.02), ("C1", 64, 0.01),
                                          ("C2", 1, 50.0), ("C2", 33, 50.0), ("C3", 16, 5.0)])
def test_propose_matches_oracle(name, k, scale):
    c = synth.config(name, N=3000 if name == "C3" else None)
    rng = np.random.default_rng(k)
    idx = rng.choice(c.N, size=k, replace=False).astype(np.int32)
    new = c.x[idx] + rng.uniform(-scale, scale, size=(k, c.D))
    x2 = c.x.copy()
    x2[idx] = new
    ref, S = _oracle_delta(c.x, x2, c.t, c.theta)
    with _ctx(c) as ctx:
        d = ctx.propose_move(idx, new)
        d_dev = ctx.propose_move(idx, torch.from_numpy(new).cuda())   # device input, same move
    assert d == d_dev
    assert abs(d - ref) <= 1e-9 * S + 1e-11 * k, (d, ref, S)


@pytest.mark.parametrize("algorithm,emulate", [("pairs", 0), ("rows", 0), ("pairs", 3), ("rows", 2)])
def test_accept_chain_tracks_oracle(algorithm, emulate):
    """A chain of accepted / rejected block moves: every proposal uses the incrementally
    updated rates; the accumulated ell matches the oracle at the end, and a fresh full
    evaluation agrees."""
    c = synth.config("C1", replicate=4)
    rng = np.random.default_rng(99)
    x = c.x.copy()
    ell0, _, _ = oracle.loglik(x, c.t, c.theta)
    ell_chain = ell0
    with _ctx(c, algorithm=algorithm, emulate_world=emulate) as ctx:
        for step in range(40):
            k = int(rng.integers(1, 9))
            idx = rng.choice(c.N, size=k, replace=False).astype(np.int32)
            new = x[idx] + rng.normal(0, 0.01, size=(k, c.D))
            d = ctx.propose_move(idx, new)
            if step % 8 == 0:
                x2 = x.copy()
                x2[idx] = new
                ref, S = _oracle_delta(x, x2, c.t, c.theta)
                assert abs(d - ref) <= 1e-9 * S + 1e-11 * k, (step, d, ref)
            if rng.uniform() < 0.6:
                ctx.accept_move()
                x[idx] = new
                ell_chain += d
        ell_ref, _, _ = oracle.loglik(x, c.t, c.theta)
        assert ell_chain == pytest.approx(ell_ref, rel=1e-10)
        assert ctx.loglik() == pytest.approx(ell_ref, rel=1e-9)
        g, _ = ctx.grad_locations()
        g_ref, S = oracle.grad(x, c.t, c.theta)
        assert np.all(np.abs(g.cpu().numpy() - g_ref) <= 1e-9 * np.maximum(np.abs(g_ref), 1e-3 * S))


def test_move_to_isolation_gives_minus_infinity():
    """Moving the only neighbour far away can make some lambda_n' = 0: Delta ell = -inf."""
    x = np.array([[0.0, 0.0], [0.05, 0.0]])
    t = np.array([0.1, 0.2])
    th = synth.THETA_UNIT
    from paper_2010_02994_b200 import HawkesContext
    with HawkesContext(2, 2) as ctx:
        ctx.set_times(t)
        ctx.set_locations(x)
        ctx.set_params(th)
        d = ctx.propose_move(np.array([1], dtype=np.int32), np.array([[1e4, 1e4]]))
    ell2, _, _ = oracle.loglik(np.array([[0.0, 0.0], [1e4, 1e4]]), t, th)
    assert ell2 == -math.inf and d == -math.inf


def test_move_errors():
    from paper_2010_02994_b200 import HawkesError
    c = synth.config("C1")
    with _ctx(c) as ctx:
        with pytest.raises(HawkesError) as ei:
            ctx.accept_move()
        assert ei.value.status == "HAWKES_ERR_STATE"
        for bad in ([3, 3], [-1], [c.N]):
            with pytest.raises(HawkesError) as ei:
                ctx.propose_move(np.array(bad, dtype=np.int32), np.zeros((len(bad), 2)))
            assert ei.value.status == "HAWKES_ERR_ARG"
        with pytest.raises(HawkesError) as ei:
            ctx.propose_move(np.arange(257, dtype=np.int32), np.zeros((257, 2)))
        assert ei.value.status == "HAWKES_ERR_ARG"
        with pytest.raises(HawkesError) as ei:
            ctx.propose_move(np.array([1], dtype=np.int32), np.array([[np.nan, 0.0]]))
        assert ei.value.status == "HAWKES_ERR_NONFINITE"
        # a set_* call discards the pending proposal
        ctx.propose_move(np.array([1], dtype=np.int32), c.x[[1]] + 0.001)
        ctx.set_params(c.theta)
        with pytest.raises(HawkesError) as ei:
            ctx.accept_move()
        assert ei.value.status == "HAWKES_ERR_STATE"
