"""Uninitialised-memory regression: device memory (and, through the unified L1 / shared-memory
SRAM, stale shared memory) filled with NaN before the context exists must not leak into
results.  Found a masked-column hazard in the sym kernels: padding columns of a ragged tile
read stale shared memory, and 0 * NaN in a masked term stayed NaN (fixed by selecting the
padding column's values to 0)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth
from tests.gpu_helpers import assert_parity, oracle_eval

pytestmark = pytest.mark.gpu


def _poison():
    free, _ = torch.cuda.mem_get_info()
    n = int(min(free * 0.6, 40e9)) // 8
    x = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    del x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("N,D", [(777, 2), (1500, 2), (1001, 3)])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("algorithm", ["pairs", "rows"])
def test_poisoned_memory_does_not_leak(N, D, precision, algorithm):
    from paper_2010_02994_b200 import HawkesContext
    c = synth.unit_square(N, config=1, D=D)
    _poison()
    with HawkesContext(N, D, precision=precision, algorithm=algorithm) as ctx:
        ctx.set_times(c.t)
        ctx.set_locations(c.x)
        ctx.set_params(c.theta)
        g, ell = ctx.grad_locations()
        g = g.cpu().numpy()
        lam = ctx.get_rates()["lambda"]
    assert np.isfinite(ell) and np.isfinite(g).all() and np.isfinite(lam).all()
    ell_r, _, _, g_r, S = oracle_eval(c.x, c.t, c.theta)
    assert_parity(ell, g, ell_r, g_r, S, precision=precision, what=f"poisoned {precision} {algorithm}")


def test_poisoned_memory_moves_hmc_sweep_bmds():
    """The other entry points on poisoned memory: block moves, the HMC transition, the MH
    sweep and the BMDS density, against the oracle."""
    import oracle
    from paper_2010_02994_b200 import HawkesContext
    c = synth.config("C2", 700)
    _poison()
    with HawkesContext(c.N, c.D) as ctx:
        ctx.set_times(c.t)
        ctx.set_locations(c.x)
        ctx.set_params(c.theta)
        idx = np.array([5, 300, 699], dtype=np.int32)
        new = c.x[idx] + 20.0
        d = ctx.propose_move(idx, new)
        x2 = c.x.copy()
        x2[idx] = new
        ell0 = oracle.loglik(c.x, c.t, c.theta)[0]
        assert d == pytest.approx(oracle.loglik(x2, c.t, c.theta)[0] - ell0, rel=1e-7, abs=1e-7)
        ctx.set_regions("square", c.centre, c.size)
        blocks = np.arange(40, dtype=np.int32).reshape(10, 4)
        x_ref, acc_ref, _ = oracle.mh_sweep(c.x, c.t, c.theta, "square", c.centre, c.size, blocks, 0.5, 2, 0)
        acc, _ = ctx.mh_sweep(blocks, 0.5, 2, 0)
        assert list(acc) == list(acc_ref)
        x_ref, acc_ref, la_ref = oracle.hmc_step(x_ref, c.t, c.theta, 4, 0, 5.0, 3)
        acc, la = ctx.hmc_step(4, 0, 5.0, 3)
        assert acc == acc_ref and la == pytest.approx(la_ref, rel=1e-7, abs=1e-8)
    cf, Y, s = synth.flu_shaped(300, 3)
    _poison()
    with HawkesContext(cf.N, cf.D) as ctx:
        ctx.set_locations(cf.x)
        ctx.set_bmds(Y, s)
        lp, g = ctx.bmds_logdensity()
        lp_r, g_r = oracle.bmds(cf.x, Y, s)
        assert lp == pytest.approx(lp_r, rel=1e-10)
        assert np.max(np.abs(g.cpu().numpy() - g_r)) <= 1e-9 * np.abs(g_r).max()
