"""The spatial walk order of the PAIRS fp64 kernels (hawkes_plan.h,
hawkes_kernels_sym.cuh GEN): events walked in a Morton permutation of their locations, the
general-direction pair bodies (either event may be the later one), and exact culling of
tile pairs and chunk pairs by their bounding boxes in space and time.  Parity with the
oracle under the tolerance rule on every config shape, ties, D = 1..4, ragged sizes and
emulated ranks; bitwise reproducibility; the AUTO choice (space for the DC shape, time for
the unit square)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth
from tests.gpu_helpers import assert_parity, gpu_eval, oracle_eval

pytestmark = pytest.mark.gpu


def _check(c, what, **kw):
    ell, g, rates = gpu_eval(c.x, c.t, c.theta, ordering="space", **kw)
    ell_r, lam_r, Lam_r, g_r, S = oracle_eval(c.x, c.t, c.theta)
    np.testing.assert_allclose(rates["lambda"], lam_r, rtol=1e-11, err_msg=what)
    np.testing.assert_allclose(rates["Lambda"], Lam_r, rtol=1e-12, atol=1e-15, err_msg=what)
    return assert_parity(ell, g, ell_r, g_r, S, what=what)


@pytest.mark.parametrize("name,N", [("C1", 3000), ("C2", 5000), ("C2", 20000), ("C3", 6000),
                                    ("C4", 4097)])
def test_space_order_matches_oracle(name, N):
    _check(synth.config(name, N), f"space {name} N={N}")


@pytest.mark.parametrize("N", [256, 257, 383, 1003, 16_411])
def test_space_order_ragged_sizes(N):
    _check(synth.dc_shaped(N, replicate=N), f"space DC N={N}")


@pytest.mark.parametrize("N,k", [(700, 40), (2000, 300)])
def test_space_order_ties(N, k):
    """Equal times anywhere in the spatial walk: every tile pair takes the masked path."""
    _check(synth.with_ties(N, k), f"space ties N={N} k={k}")


@pytest.mark.parametrize("D", [1, 3, 4])
def test_space_order_dimensions(D):
    _check(synth.unit_square(1500, config=22, D=D), f"space D={D}")


@pytest.mark.parametrize("W", [2, 3])
def test_space_order_emulated_ranks(W):
    _check(synth.config("C2", 6000), f"space W={W}", emulate_world=W)


def test_space_order_reproducible_and_close_to_time_order():
    c = synth.config("C2", 12000)
    a = gpu_eval(c.x, c.t, c.theta, ordering="space")
    b = gpu_eval(c.x, c.t, c.theta, ordering="space")
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2]["lambda"], b[2]["lambda"])
    t = gpu_eval(c.x, c.t, c.theta, ordering="time")
    assert abs(a[0] - t[0]) <= 1e-13 * abs(t[0])
    np.testing.assert_allclose(a[2]["lambda"], t[2]["lambda"], rtol=1e-13)


def test_auto_ordering_choice_and_samplers():
    """AUTO takes the spatial walk for the DC shape (16 km across, 3.7 km cutoff) and the time
    walk for the unit square; the samplers run on the spatial walk too (HMC transition and MH
    sweep against the time walk: same decisions)."""
    from paper_2010_02994_b200 import HawkesContext
    out = {}
    for name, N in (("C2", 20000), ("C4", 20000)):
        c = synth.config(name, N)
        with HawkesContext(c.N, c.D) as ctx:
            ctx.set_times(c.t)
            ctx.set_locations(c.x)
            ctx.set_params(c.theta)
            ctx.loglik()
            out[name] = ctx.ordering_in_use
    assert out["C2"][0] == "space" and out["C4"][0] == "time", out
    c = synth.config("C2", 3000)
    res = {}
    for mode in ("space", "time"):
        with HawkesContext(c.N, c.D) as ctx:
            ctx.set_ordering(mode)
            ctx.set_times(c.t)
            ctx.set_locations(c.x)
            ctx.set_params(c.theta)
            ctx.set_regions("square", c.centre, c.size)
            blocks = np.arange(60, dtype=np.int32).reshape(30, 2)
            acc, la = ctx.mh_sweep(blocks, 0.5, 3, 0)
            acc_h, la_h = ctx.hmc_step(3, 1, 2.0, 4)
            res[mode] = (acc, la, acc_h, la_h, ctx.get_locations().cpu().numpy(), ctx.ordering_in_use[0])
    assert res["space"][5] == "space" and res["time"][5] == "time"
    assert list(res["space"][0]) == list(res["time"][0])
    np.testing.assert_allclose(res["space"][1], res["time"][1], rtol=1e-9, atol=1e-9)
    assert res["space"][2] == res["time"][2] and abs(res["space"][3] - res["time"][3]) <= 1e-8
    np.testing.assert_allclose(res["space"][4], res["time"][4], rtol=0, atol=1e-8)


@pytest.mark.parametrize("name,N", [("C2", 6000), ("C3", 6000), ("C1", 3001)])
def test_space_order_fp32(name, N):
    """The fp32 kernels on the spatial walk (hawkes_kernels_f32.cuh GEN) under the fp32 gate."""
    c = synth.config(name, N)
    ell, g, rates = gpu_eval(c.x, c.t, c.theta, precision="fp32", ordering="space")
    ell_r, lam_r, _, g_r, S = oracle_eval(c.x, c.t, c.theta)
    np.testing.assert_allclose(rates["lambda"], lam_r, rtol=1e-4)
    assert_parity(ell, g, ell_r, g_r, S, precision="fp32", what=f"space fp32 {name}")
