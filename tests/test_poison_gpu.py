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
