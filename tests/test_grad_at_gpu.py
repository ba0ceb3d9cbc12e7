"""hawkes_grad_at (include/hawkes.h): ell and the location gradient (Eq. 1, App. A; P:L96-101,
P:L385) at new device locations in one call -- after two evaluations with unchanged
constants, one CUDA-graph launch whose packing and gradient-finalize nodes take the caller's
x and out_grad pointers.  It must give the same bits as set_locations + grad_locations, follow
the caller's buffers from call to call (new pointers and new contents behind an old pointer),
report device-side validation errors, and match the oracle."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth
from tests.gpu_helpers import assert_parity, oracle_eval

pytestmark = pytest.mark.gpu


def _pair(c, **kw):
    from paper_2010_02994_b200 import HawkesContext
    N, D = c.x.shape
    ctxs = [HawkesContext(N, D, **kw) for _ in range(2)]
    t = torch.from_numpy(np.ascontiguousarray(c.t)).cuda()
    for ctx in ctxs:
        ctx.set_times(t)
        ctx.set_params(c.theta)
    return ctxs


def _states(c, n, seed=1):
    """n location arrays near c.x (small moves, as consecutive HMC states)."""
    rng = np.random.default_rng(seed)
    scale = 1e-3 * (c.x.max(axis=0) - c.x.min(axis=0))
    return [torch.from_numpy(c.x + rng.normal(size=c.x.shape) * scale).cuda() for _ in range(n)]


@pytest.mark.parametrize("name,N,kw", [
    ("C4", 5000, {}),
    ("C2", 5000, {}),                       # DC shape: AUTO takes the spatial walk
    ("C1", 1111, {"precision": "fp32"}),
    ("C3", 3001, {}),
    ("C1", 700, {"algorithm": "rows"}),     # no captured path: the two calls
    ("C1", 2000, {"emulate_world": 2}),     # no captured path (W > 1)
])
def test_grad_at_bitwise_equals_two_calls(name, N, kw):
    c = synth.config(name, N)
    ref, at = _pair(c, **kw)
    xs = _states(c, 6)
    with ref, at:
        for k, x in enumerate(xs):
            ref.set_locations(x)
            g_ref, ell_ref = ref.grad_locations()
            g_at, ell_at = at.grad_at(x)
            torch.cuda.synchronize()
            assert ell_at == ell_ref, f"call {k}"
            assert torch.equal(g_at, g_ref), f"call {k}: max diff {(g_at - g_ref).abs().max().item()}"
            # the cached state is the new one: a following ell / rates call agrees
            assert at.loglik() == ell_ref
        np.testing.assert_array_equal(at.get_rates()["lambda"], ref.get_rates()["lambda"])


@pytest.mark.parametrize("D,N,ties", [(1, 1500, 0), (3, 2100, 0), (5, 900, 0), (2, 1700, 60)])
def test_grad_at_other_dimensions_and_ties(D, N, ties):
    """Every D's captured graph (its own packing / finalize node instantiations) and a tie
    catalog (masked tile pairs): bitwise equal to the two calls."""
    c = synth.with_ties(N, ties, D=D) if ties else synth.unit_square(N, config=1, D=D)
    ref, at = _pair(c)
    xs = _states(c, 4, seed=D)
    with ref, at:
        for k, x in enumerate(xs):
            ref.set_locations(x)
            g_ref, ell_ref = ref.grad_locations()
            g_at, ell_at = at.grad_at(x)
            assert ell_at == ell_ref and torch.equal(g_at, g_ref), f"D={D} call {k}"


def test_grad_at_follows_buffer_contents_and_outputs():
    c = synth.config("C4", 3000)
    ref, at = _pair(c)
    xs = _states(c, 3)
    x = xs[0].clone()
    outs = [torch.empty_like(x) for _ in range(3)]
    with ref, at:
        for k in range(8):
            # the same x pointer with new contents, and a rotating output buffer
            x.copy_(xs[k % 3])
            out = outs[k % 3]
            out.fill_(float("nan"))
            g_at, ell_at = at.grad_at(x, out)
            assert g_at.data_ptr() == out.data_ptr()
            ref.set_locations(xs[k % 3])
            g_ref, ell_ref = ref.grad_locations()
            torch.cuda.synchronize()
            assert ell_at == ell_ref and torch.equal(out, g_ref), f"call {k}"


def test_grad_at_matches_oracle():
    c = synth.config("C2", 4000)
    (at,) = _pair(c)[:1]
    with at:
        x = torch.from_numpy(c.x).cuda()
        for _ in range(4):   # the last calls take the captured path
            g, ell = at.grad_at(x)
    ell_r, lam_r, Lam_r, g_r, S = oracle_eval(c.x, c.t, c.theta)
    assert_parity(ell, g.cpu().numpy(), ell_r, g_r, S, what="grad_at C2 N=4000")


def test_grad_at_validates_device_input():
    from paper_2010_02994_b200 import HawkesError
    c = synth.config("C4", 2000)
    (at,) = _pair(c)[:1]
    xs = _states(c, 2)
    with at:
        for x in xs + xs:
            at.grad_at(x)
        bad = xs[0].clone()
        bad[17, 1] = float("nan")
        with pytest.raises(HawkesError):
            at.grad_at(bad)
        g, ell = at.grad_at(xs[1])   # recovers
        ref, = _pair(c)[:1]
        with ref:
            ref.set_locations(xs[1])
            g_ref, ell_ref = ref.grad_locations()
        assert ell == ell_ref and torch.equal(g, g_ref)


def test_grad_at_after_params_change():
    c = synth.config("C4", 2500)
    ref, at = _pair(c)
    xs = _states(c, 4)
    theta2 = list(c.theta)
    theta2[3] *= 0.9
    with ref, at:
        for k, x in enumerate(xs * 2):
            if k == 5:   # drops the graphs; the next calls recapture
                at.set_params(theta2)
                ref.set_params(theta2)
            ref.set_locations(x)
            g_ref, ell_ref = ref.grad_locations()
            g_at, ell_at = at.grad_at(x)
            assert ell_at == ell_ref and torch.equal(g_at, g_ref), f"call {k}"


def test_grad_at_fp32_range_guard():
    """The fp32 range guard (reading R23) inside grad_at: round 1's failing fuzz catalog is
    redone by the fp64 kernels on the first call, and the following (captured) calls stay on
    fp64 and meet the fp64 gate."""
    from paper_2010_02994_b200 import HawkesContext
    from tests.test_parity_gpu import _fuzz_case
    N, D, x, t, th, _, _, _ = _fuzz_case(12, 290, 4000)
    ell_r, _, _, g_r, S = oracle_eval(x, t, th)
    with HawkesContext(N, D, precision="fp32") as ctx:
        ctx.set_times(t)
        ctx.set_params(th)
        xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        for k in range(4):
            g, ell = ctx.grad_at(xd)
            assert ctx.precision_in_use == "fp64", f"call {k}"
            assert_parity(ell, g.cpu().numpy(), ell_r, g_r, S, precision="fp64", what=f"guarded grad_at {k}")
