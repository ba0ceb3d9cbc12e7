"""The multi-GPU plumbing on one GPU: a context created with world = 1 and an NCCL unique id
builds a real one-rank communicator and runs the sharded code path -- per-rank slot sums and
ncclAllReduce (PAIRS), row packing and ncclAllGather (ROWS), the exchanged finalize, and the
block-move row exchange -- against the oracle and the plain single-GPU path."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.gpu_helpers import assert_parity, oracle_eval

pytestmark = pytest.mark.gpu


def _eval(c, **kw):
    from paper_2010_02994_b200 import HawkesContext
    with HawkesContext(c.N, c.D, **kw) as ctx:
        ctx.set_times(c.t)
        ctx.set_locations(c.x)
        ctx.set_params(c.theta)
        ell0 = ctx.loglik()
        g, ell = ctx.grad_locations()
        assert ell == ell0
        lam = ctx.get_rates()["lambda"]
        return ell, g.cpu().numpy(), lam


@pytest.mark.parametrize("algorithm", ["pairs", "rows"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_one_rank_nccl_path_matches_oracle_and_single_gpu(algorithm, precision):
    from paper_2010_02994_b200 import nccl_unique_id
    c = synth.config("C1", 1500)
    ell_n, g_n, lam_n = _eval(c, algorithm=algorithm, precision=precision, nccl_id=nccl_unique_id())
    ell_1, g_1, lam_1 = _eval(c, algorithm=algorithm, precision=precision)
    ell_r, _, _, g_r, S = oracle_eval(c.x, c.t, c.theta)
    assert_parity(ell_n, g_n, ell_r, g_r, S, precision=precision, what=f"nccl {algorithm} {precision}")
    # same arithmetic as the plain path (only the exchange differs): agree to rounding
    tol = 1e-13 if precision == "fp64" else 1e-6
    assert abs(ell_n - ell_1) <= tol * abs(ell_1)
    assert np.max(np.abs(g_n - g_1)) <= tol * np.abs(g_1).max()
    assert np.max(np.abs(lam_n - lam_1) / lam_1) <= tol


def test_one_rank_nccl_leapfrog_and_moves():
    """The leapfrog (gradient exchange every step) and the block-move rate exchange."""
    from paper_2010_02994_b200 import HawkesContext, nccl_unique_id
    c = synth.config("C1", 800)
    p0 = synth.momenta(c.N, c.D, seed=3)
    xr, pr, ellr, kr = oracle.leapfrog(c.x, p0, c.t, c.theta, 2e-4, 5)
    for algorithm in ("pairs", "rows"):
        with HawkesContext(c.N, c.D, algorithm=algorithm, nccl_id=nccl_unique_id()) as ctx:
            ctx.set_times(c.t)
            ctx.set_params(c.theta)
            x, p = torch.from_numpy(c.x.copy()).cuda(), torch.from_numpy(p0.copy()).cuda()
            _, _, ell, kin = ctx.leapfrog(x, p, 2e-4, 5)
            assert np.max(np.abs(x.cpu().numpy() - xr)) <= 1e-9
            assert ell == pytest.approx(ellr, rel=1e-9)
            idx = np.array([3, 77, 500], dtype=np.int32)
            new = xr[idx] + 0.01
            d = ctx.propose_move(idx, new)
            x2 = xr.copy()
            x2[idx] = new
            assert d == pytest.approx(oracle.loglik(x2, c.t, c.theta)[0] - oracle.loglik(xr, c.t, c.theta)[0],
                                      rel=1e-7, abs=1e-8)


def test_nccl_id_with_emulation_rejected():
    from paper_2010_02994_b200 import HawkesContext, HawkesError, nccl_unique_id
    with pytest.raises(HawkesError, match="ARG"):
        HawkesContext(100, 2, nccl_id=nccl_unique_id(), emulate_world=2)


@pytest.mark.parametrize("algorithm", ["pairs", "rows"])
def test_one_rank_nccl_hmc_and_mh_sweep(algorithm):
    """The HMC transition (gradient exchanges every leapfrog step) and the MH sweep (exchanged
    rates for ROWS) on the sharded path with a real one-rank communicator: the same decisions
    as a plain context."""
    from paper_2010_02994_b200 import HawkesContext, nccl_unique_id
    c = synth.config("C2", 700)
    rng = np.random.default_rng(1)
    blocks = np.stack([rng.choice(c.N, size=3, replace=False) for _ in range(12)]).astype(np.int32)
    res = []
    for nccl in (True, False):
        kw = {"nccl_id": nccl_unique_id()} if nccl else {}
        with HawkesContext(c.N, c.D, algorithm=algorithm, **kw) as ctx:
            ctx.set_times(c.t)
            ctx.set_locations(c.x)
            ctx.set_params(c.theta)
            ctx.set_regions(c.region, c.centre, c.size)
            acc, la = ctx.mh_sweep(blocks, 0.5, 9, 0)
            h = [ctx.hmc_step(9, it, 20.0, 4) for it in range(3)]
            res.append((acc, la, h, ctx.get_locations().cpu().numpy()))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.allclose(res[0][1], res[1][1], rtol=1e-12, atol=1e-12)
    assert [a for a, _ in res[0][2]] == [a for a, _ in res[1][2]]
    assert np.allclose(res[0][3], res[1][3], rtol=0, atol=1e-9)


@pytest.mark.parametrize("algorithm", ["pairs", "rows"])
def test_one_rank_nccl_grad_at(algorithm):
    """hawkes_grad_at on the sharded path (no captured graph there: the two calls) equals
    set_locations + grad_locations on the same kind of context, bit for bit."""
    from paper_2010_02994_b200 import HawkesContext, nccl_unique_id
    c = synth.config("C1", 1200)
    ctxs = [HawkesContext(c.N, c.D, algorithm=algorithm, nccl_id=nccl_unique_id()) for _ in range(2)]
    rng = np.random.default_rng(3)
    try:
        for ctx in ctxs:
            ctx.set_times(c.t)
            ctx.set_params(c.theta)
        for k in range(4):
            x = torch.from_numpy(c.x + 1e-3 * rng.normal(size=c.x.shape)).cuda()
            ctxs[0].set_locations(x)
            g0, e0 = ctxs[0].grad_locations()
            g1, e1 = ctxs[1].grad_at(x)
            assert e0 == e1 and torch.equal(g0, g1), f"call {k}"
    finally:
        for ctx in ctxs:
            ctx.close()
