"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerance (from the north_star's 1e-9 fp64 bar):
|ell - ell*| <= 1e-9 |ell*| and, per gradient component, |g - g*| <= 1e-9 max(|g*|, 1e-3 S)
with S the component's conditioning scale sum_n' |c_nn' (x_n'd - x_nd)| from the oracle.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from tests.gpu_helpers import assert_parity, gpu_eval, oracle_eval

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def _check(c, what, precision="fp64", emulate_world=0, algorithm="auto"):
    ell, g, rates = gpu_eval(c.x, c.t, c.theta, precision=precision, emulate_world=emulate_world,
                             algorithm=algorithm)
    ell_ref, lam_ref, Lam_ref, g_ref, S = oracle_eval(c.x, c.t, c.theta)
    if ell_ref == -math.inf:
        assert ell == -math.inf, what
        return
    np.testing.assert_allclose(rates["lambda"], lam_ref, rtol=1e-11, err_msg=what)
    np.testing.assert_allclose(rates["Lambda"], Lam_ref, rtol=1e-12, atol=1e-15, err_msg=what)
    return assert_parity(ell, g, ell_ref, g_ref, S, precision=precision, what=what)


def test_library_is_in_tree():
    from paper_2010_02994_b200 import _lib
    lib = _lib.load()
    assert lib._name.endswith("paper_2010_02994_b200/libhawkes_b200.so")


@pytest.mark.parametrize("rep", range(10))
def test_c1_unit_square_seeds(rep):
    """BASELINE configs[0]: N=500, D=2, 10 seeded replicates."""
    _check(synth.config("C1", replicate=rep), f"C1 rep {rep}")


@pytest.mark.parametrize("N", [2, 3, 127, 128, 255, 256, 257, 511, 513, 1003, 4097, 16_383, 16_384, 16_411,
                               35_584, 35_841])
def test_ragged_sizes(N):
    """Tile edges: row tiles of 256, j tiles of 128, chunks >= 512; N = 16383 / 16384 / 16411
    straddle PAIRS' 256-event chunk floor (hawkes_plan.h chunk_pairs_of)."""
    _check(synth.unit_square(N, config=21, replicate=N), f"N={N}")


def test_c2_dc_shaped():
    """BASELINE configs[1]: DC-gunfire-shaped, N=5k, metres/hours, heavy underflow."""
    _check(synth.config("C2"), "C2")


def test_c3_alaska_shaped():
    """BASELINE configs[2]: Alaska-wildfire-shaped, N=20k, km/days."""
    _check(synth.config("C3"), "C3")


@pytest.mark.parametrize("N,k", [(700, 40), (2000, 300), (600, 3)])
def test_ties(N, k):
    """Equal times: the indicators of P:L82 / P:L99 on masked (diagonal) tiles."""
    _check(synth.with_ties(N, k), f"ties N={N} k={k}")


@pytest.mark.parametrize("algorithm", ["pairs", "rows"])
@pytest.mark.parametrize("D", [1, 3, 4, 5, 6, 7, 8])
def test_other_dimensions(D, algorithm):
    """D = 1..8 (the flu model's latent space uses D up to 8), both decompositions
    (AUTO runs PAIRS for every D)."""
    _check(synth.unit_square(900, config=22, D=D), f"D={D} {algorithm}", algorithm=algorithm)


def test_special_parameters():
    c = synth.unit_square(800, config=23)
    for th in [(0.6, 0.1, 0.1, 0.0, 20.0, 0.03),      # theta = 0: background only (KDE)
               (0.0, 0.1, 0.1, 0.4, 20.0, 0.03),      # mu0 = 0: self-excitation only
               (2.0, 0.5, 0.02, 1.5, 300.0, 0.005)]:  # sharp kernels, large omega
        cc = synth.Catalog(c.x, c.t, th, "special", 0)
        try:
            _check(cc, f"theta={th}")
        except AssertionError:
            raise


def test_single_event_and_isolated_events():
    """N=1 -> ell = -inf; events far apart -> lambda_n = 0 -> -inf, gradient undefined."""
    from paper_2010_02994_b200 import HawkesContext, HawkesError
    ell, g, _ = gpu_eval(np.array([[0.1, 0.2]]), np.array([0.3]), synth.THETA_UNIT)
    assert ell == -math.inf and g is None
    x = np.array([[0.0, 0.0], [1e4, 0.0], [0.0, 1e4]])
    t = np.array([0.1, 0.2, 0.3])
    ell_ref, _, _ = oracle.loglik(x, t, synth.THETA_UNIT)
    assert ell_ref == -math.inf
    with HawkesContext(3, 2) as ctx:
        ctx.set_times(t)
        ctx.set_locations(x)
        ctx.set_params(synth.THETA_UNIT)
        assert ctx.loglik() == -math.inf
        with pytest.raises(HawkesError) as ei:
            ctx.grad_locations()
        assert ei.value.status == "HAWKES_ERR_GRAD_UNDEFINED"


def test_abi_errors():
    from paper_2010_02994_b200 import HawkesContext, HawkesError
    with HawkesContext(4, 2) as ctx:
        with pytest.raises(HawkesError) as ei:
            ctx.loglik()
        assert ei.value.status == "HAWKES_ERR_STATE"
        with pytest.raises(HawkesError) as ei:
            ctx.set_times(np.array([0.1, 0.3, 0.2, 0.4]))
        assert ei.value.status == "HAWKES_ERR_UNSORTED"
        with pytest.raises(HawkesError) as ei:
            ctx.set_times(np.array([-0.1, 0.3, 0.5, 0.6]))
        assert ei.value.status == "HAWKES_ERR_NONFINITE"
        with pytest.raises(HawkesError) as ei:
            ctx.set_locations(np.array([[0, 0], [1, np.nan], [0, 0], [1, 1.0]]))
        assert ei.value.status == "HAWKES_ERR_NONFINITE"
        with pytest.raises(HawkesError) as ei:
            ctx.set_params((1.0, -0.1, 1.0, 1.0, 1.0, 1.0))
        assert ei.value.status == "HAWKES_ERR_PARAM"
        with pytest.raises(HawkesError) as ei:
            ctx.set_params((1.0, 1e-200, 1.0, 1.0, 1.0, 1.0))
        assert ei.value.status == "HAWKES_ERR_PARAM"
        # device-side validation of device inputs is reported by the next evaluation
        ctx.set_times(np.array([0.1, 0.2, 0.3, 0.4]))
        ctx.set_params(synth.THETA_UNIT)
        ctx.set_locations(torch.tensor([[0, 0], [1, float("inf")], [0, 0], [1, 1.0]],
                                       dtype=torch.float64, device="cuda"))
        with pytest.raises(HawkesError) as ei:
            ctx.loglik()
        assert ei.value.status == "HAWKES_ERR_NONFINITE"
        ctx.set_locations(np.array([[0, 0], [0.1, 0.0], [0, 0.1], [0.1, 0.1]]))
        assert np.isfinite(ctx.loglik())
    with pytest.raises(HawkesError) as ei:
        HawkesContext(10, 9)
    assert ei.value.status == "HAWKES_ERR_DIM"


def test_bitwise_determinism_and_emulated_world():
    """ROWS: repeat runs and W = 2, 3, 8 logical row shards give bit-identical ell, lambda, g
    (per-row summation order does not depend on W).  PAIRS: repeat runs
    are bit-identical; W logical shards (allreduce of per-event sums) agree to rounding."""
    c = synth.unit_square(3000, config=24)
    ell_ref, lam_ref, _, g_ref, S = oracle_eval(c.x, c.t, c.theta)
    ell1, g1, r1 = gpu_eval(c.x, c.t, c.theta, algorithm="rows")
    ell1b, g1b, r1b = gpu_eval(c.x, c.t, c.theta, algorithm="rows")
    assert ell1 == ell1b and np.array_equal(g1, g1b) and np.array_equal(r1["lambda"], r1b["lambda"])
    for W in (2, 3, 8):
        ellw, gw, rw = gpu_eval(c.x, c.t, c.theta, emulate_world=W, algorithm="rows")
        assert ellw == ell1, W
        assert np.array_equal(gw, g1), W
        for k in ("lambda", "mu", "xi", "Lambda"):
            assert np.array_equal(rw[k], r1[k]), (W, k)
    assert_parity(ell1, g1, ell_ref, g_ref, S, what="ROWS W-sweep reference")
    ep, gp, rp = gpu_eval(c.x, c.t, c.theta, algorithm="pairs")
    ep2, gp2, rp2 = gpu_eval(c.x, c.t, c.theta, algorithm="pairs")
    assert ep == ep2 and np.array_equal(gp, gp2) and np.array_equal(rp["lambda"], rp2["lambda"])
    assert_parity(ep, gp, ell_ref, g_ref, S, what="PAIRS")
    for W in (2, 3, 8):
        ew, gw, rw = gpu_eval(c.x, c.t, c.theta, emulate_world=W, algorithm="pairs")
        assert abs(ew - ep) <= 1e-13 * abs(ep), W
        assert np.all(np.abs(gw - gp) <= 1e-13 * (np.abs(gp) + S)), W
        np.testing.assert_allclose(rw["lambda"], rp["lambda"], rtol=1e-14)
        assert_parity(ew, gw, ell_ref, g_ref, S, what=f"PAIRS W={W}")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("D", [3, 6])
def test_emulated_world_other_dimensions(D, precision):
    """The sharded PAIRS path (per-rank slot sums, rank-ordered exchange) at D = 3 and 6 (the
    D >= 5 kernels run at 2 CTAs/SM), both precisions: W = 3 agrees with W = 1 to rounding
    and with the oracle under the tolerance rule."""
    c = synth.unit_square(1800, config=32, D=D)
    ell_ref, _, _, g_ref, S = oracle_eval(c.x, c.t, c.theta)
    e1, g1, r1 = gpu_eval(c.x, c.t, c.theta, precision=precision, algorithm="pairs")
    e3, g3, r3 = gpu_eval(c.x, c.t, c.theta, precision=precision, emulate_world=3, algorithm="pairs")
    # fp32: the plan's pieces (hawkes_plan.h choose_pieces) depend on W, and each piece sums
    # its terms in fp32 before they meet in fp64: W = 3 regroups fp32 partial sums
    tol = 1e-13 if precision == "fp64" else 4e-6
    assert abs(e3 - e1) <= tol * abs(e1)
    assert np.all(np.abs(g3 - g1) <= tol * (np.abs(g1) + S))
    assert_parity(e3, g3, ell_ref, g_ref, S, precision=precision, what=f"PAIRS W=3 D={D} {precision}")


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_rows_algorithm_configs(name):
    """The ordered-pair (ROWS) decomposition on the small configs."""
    c = synth.config(name)
    ell, g, rates = gpu_eval(c.x, c.t, c.theta, algorithm="rows")
    ell_ref, lam_ref, _, g_ref, S = oracle_eval(c.x, c.t, c.theta)
    np.testing.assert_allclose(rates["lambda"], lam_ref, rtol=1e-11)
    assert_parity(ell, g, ell_ref, g_ref, S, what=f"ROWS {name}")


@pytest.mark.parametrize("N", [257, 1003, 5000])
def test_rows_algorithm_ragged_and_ties(N):
    for c in (synth.unit_square(N, config=28, replicate=N), synth.with_ties(N, max(2, N // 7))):
        ell, g, _ = gpu_eval(c.x, c.t, c.theta, algorithm="rows")
        ell_ref, _, _, g_ref, S = oracle_eval(c.x, c.t, c.theta)
        assert_parity(ell, g, ell_ref, g_ref, S, what=f"ROWS {c.name}")


def test_full_size_c4_sampled_rows_and_properties():
    """BASELINE configs[3] at N=100k (the bench workload): lambda on sampled rows against
    the oracle computed row by row; sum_n g_n = 0 (App. A: c_nn' symmetric); the
    directional derivative of the GPU's own ell matches <g, V>."""
    c = synth.config("C4")
    from paper_2010_02994_b200 import HawkesContext
    N = c.N
    rows = np.unique(np.concatenate([np.arange(0, N, N // 48), [N - 1, N - 2, 255, 256, 257]]))
    with HawkesContext(N, 2) as ctx:
        ctx.set_times(c.t)
        ctx.set_locations(c.x)
        ctx.set_params(c.theta)
        g, ell = ctx.grad_locations()
        g = g.cpu().numpy()
        rates = ctx.get_rates()
        lam_ref = np.empty(len(rows))
        for k, r in enumerate(rows):
            lam_ref[k] = oracle.rates(c.x, c.t, c.theta, rows=slice(int(r), int(r) + 1))[0][r]
        np.testing.assert_allclose(rates["lambda"][rows], lam_ref, rtol=1e-11)
        Lam_ref = oracle.Lambda(c.t, c.theta)
        np.testing.assert_allclose(rates["Lambda"], Lam_ref, rtol=1e-12, atol=1e-15)
        assert np.all(np.abs(g.sum(axis=0)) <= 1e-11 * np.abs(g).sum(axis=0))
        V = np.random.default_rng(3).normal(size=c.x.shape)
        eps = 1e-6
        ctx.set_locations(c.x + eps * V)
        lp = ctx.loglik()
        ctx.set_locations(c.x - eps * V)
        lm = ctx.loglik()
        fd = (lp - lm) / (2 * eps)
        dir_ = float(np.sum(g * V))
        assert abs(fd - dir_) <= 1e-6 * np.sum(np.abs(g * V)), (fd, dir_)


def test_fast_exp_accuracy():
    """The kernels' exp (1024-entry table + degree-3 minimax polynomial, hawkes_kernels.cuh)
    against an 80-bit long-double exp: relative error <= 4e-16 + 1.2e-16 |a| on [-707, 700]
    (truncation 9.4e-17 from tools/fit_exp_poly.py 1024 3; the rest is the rounding of the
    table entry, the reduction r = a - k ln2/1024 and the final fma) -- u-accurate, as SURVEY
    §7 asks; below -707 the argument is clamped, so the result is e^(-707 +- 1e-3), never
    above e^-706 (R23)."""
    from paper_2010_02994_b200 import diag_exp
    a = np.concatenate([np.linspace(-800.0, 700.0, 600001), np.linspace(-1.0, 1.0, 100001),
                        [-1e300, -1e30, -745.2, -745.0, -709.0, -707.0, 0.0, 1e-300, -np.inf]])
    out = diag_exp(torch.from_numpy(a).cuda()).cpu().numpy()
    live = a >= -707.0
    ref = np.exp(a[live].astype(np.longdouble))
    rel = np.abs(out[live].astype(np.longdouble) - ref) / ref
    assert np.all(rel <= 4e-16 + 1.2e-16 * np.abs(a[live])), float(rel.max())
    dead = ~live
    assert np.all(out[dead] > 0) and np.all(out[dead] <= math.exp(-706.0))


def test_leapfrog_matches_oracle_and_reverses():
    """hawkes_leapfrog vs the oracle's literal leapfrog at N=500, L=20."""
    from paper_2010_02994_b200 import HawkesContext
    c = synth.config("C1")
    p0 = synth.momenta(c.N, c.D, seed=11)
    step, L = 2e-4, 20
    xr, pr, ellr, kr = oracle.leapfrog(c.x, p0, c.t, c.theta, step, L)
    with HawkesContext(c.N, c.D) as ctx:
        ctx.set_times(c.t)
        ctx.set_params(c.theta)
        x = torch.from_numpy(c.x.copy()).cuda()
        p = torch.from_numpy(p0.copy()).cuda()
        _, _, ell, kin = ctx.leapfrog(x, p, step, L)
        xg, pg = x.cpu().numpy(), p.cpu().numpy()
        scale_x = np.abs(c.x).max()
        assert np.max(np.abs(xg - xr)) <= 1e-9 * scale_x
        assert np.max(np.abs(pg - pr)) <= 1e-9 * np.abs(pr).max()
        assert ell == pytest.approx(ellr, rel=1e-9)
        assert kin == pytest.approx(kr, rel=1e-9)
        # reversibility: negate p, integrate back
        p.neg_()
        ctx.leapfrog(x, p, step, L)
        assert np.max(np.abs(x.cpu().numpy() - c.x)) <= 1e-10 * scale_x
        assert np.max(np.abs(-p.cpu().numpy() - p0)) <= 1e-9 * np.abs(p0).max()


def test_leapfrog_host_buffers_and_box():
    """Host-memory leapfrog with a reflecting box (the DC +-50 m prior, in C1 units)."""
    from paper_2010_02994_b200 import HawkesContext
    c = synth.config("C1", replicate=3)
    p0 = synth.momenta(c.N, c.D, seed=12) * 30.0
    lo, hi = c.x - 0.002, c.x + 0.002
    step, L = 2e-4, 10
    xr, pr, ellr, kr = oracle.leapfrog(c.x, p0, c.t, c.theta, step, L, box_lo=lo, box_hi=hi)
    with HawkesContext(c.N, c.D) as ctx:
        ctx.set_times(c.t)
        ctx.set_params(c.theta)
        x, p = c.x.copy(), p0.copy()
        _, _, ell, kin = ctx.leapfrog(x, p, step, L, box_lo=lo, box_hi=hi)
    assert np.all(x >= lo) and np.all(x <= hi)
    assert np.max(np.abs(x - xr)) <= 1e-9
    assert ell == pytest.approx(ellr, rel=1e-9)
    assert kin == pytest.approx(kr, rel=1e-9)


# ----------------------------------------------------------------------- fp32 path
@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_fp32_configs(name):
    """fp32-accumulate variant at the north_star's 1e-4 (normwise per component)."""
    _check_fp32(synth.config(name), f"fp32 {name}")


@pytest.mark.parametrize("N", [3, 257, 1003])
def test_fp32_ragged_and_ties(N):
    _check_fp32(synth.unit_square(N, config=25, replicate=N), f"fp32 N={N}")
    _check_fp32(synth.with_ties(N, max(2, N // 10)), f"fp32 ties N={N}")


@pytest.mark.parametrize("N", [16_384, 16_411])
def test_fp32_chunk_floor_sizes(N):
    """fp32 PAIRS at sizes that take the 256-event chunk floor (hawkes_plan.h chunk_pairs_of)."""
    _check_fp32(synth.unit_square(N, config=25, replicate=N), f"fp32 N={N}")


@pytest.mark.parametrize("algorithm", ["pairs", "rows"])
@pytest.mark.parametrize("D", [1, 3, 4, 5, 6, 7, 8])
def test_fp32_other_dimensions(D, algorithm):
    _check_fp32(synth.unit_square(700, config=26, D=D), f"fp32 D={D} {algorithm}", algorithm=algorithm)


def test_fp32_emulated_world():
    """fp32: ROWS is bitwise W-independent; PAIRS agrees across W to fp64 rounding of the
    exchanged per-event sums and stays within the fp32 tolerance."""
    c = synth.unit_square(2000, config=27)
    e1, g1, r1 = gpu_eval(c.x, c.t, c.theta, precision="fp32", algorithm="rows")
    e4, g4, r4 = gpu_eval(c.x, c.t, c.theta, precision="fp32", emulate_world=4, algorithm="rows")
    assert e1 == e4 and np.array_equal(g1, g4) and np.array_equal(r1["lambda"], r4["lambda"])
    ell_ref, _, _, g_ref, S = oracle_eval(c.x, c.t, c.theta)
    for W in (1, 3):
        ew, gw, _ = gpu_eval(c.x, c.t, c.theta, precision="fp32", emulate_world=W, algorithm="pairs")
        assert_parity(ew, gw, ell_ref, g_ref, S, precision="fp32", what=f"fp32 PAIRS W={W}")


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_fp32_rows_algorithm(name):
    c = synth.config(name)
    ell, g, _ = gpu_eval(c.x, c.t, c.theta, precision="fp32", algorithm="rows")
    ell_ref, _, _, g_ref, S = oracle_eval(c.x, c.t, c.theta)
    assert_parity(ell, g, ell_ref, g_ref, S, precision="fp32", what=f"fp32 ROWS {name}")


def _check_fp32(c, what, algorithm="auto"):
    ell, g, rates = gpu_eval(c.x, c.t, c.theta, precision="fp32", algorithm=algorithm)
    ell_ref, lam_ref, Lam_ref, g_ref, S = oracle_eval(c.x, c.t, c.theta)
    np.testing.assert_allclose(rates["lambda"], lam_ref, rtol=1e-4, err_msg=what)
    return assert_parity(ell, g, ell_ref, g_ref, S, precision="fp32", what=what)


def test_graph_replay_matches_fresh_contexts():
    """Repeated evaluations replay a captured CUDA graph; changing Theta or x between them
    must give bit-identical results to a fresh context (small-N latency)."""
    from paper_2010_02994_b200 import HawkesContext
    c = synth.unit_square(1500, config=29)
    th2 = (0.5, 0.12, 0.08, 0.5, 15.0, 0.04)
    x2 = c.x + 0.001

    def fresh(x, th):
        with HawkesContext(c.N, c.D) as f:
            f.set_times(c.t)
            f.set_locations(x)
            f.set_params(th)
            g, e = f.grad_locations()
            return e, g.cpu().numpy()

    with HawkesContext(c.N, c.D) as ctx:
        ctx.set_times(c.t)
        ctx.set_params(c.theta)
        seq = [(c.x, c.theta), (c.x, c.theta), (x2, c.theta), (x2, c.theta), (x2, th2),
               (x2, th2), (c.x, th2), (c.x, c.theta)]
        prev_th = c.theta
        for x, th in seq:
            if th is not prev_th:
                ctx.set_params(th)
                prev_th = th
            ctx.set_locations(torch.from_numpy(np.ascontiguousarray(x)).cuda())
            ell_l = ctx.loglik()
            g, e = ctx.grad_locations()
            ef, gf = fresh(x, th)
            assert e == ef and ell_l == ef
            assert np.array_equal(g.cpu().numpy(), gf)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_call_sequences_status_mirror_and_counter_rearm(precision):
    """The small-call path: the PAIRS finalizes re-arm the item counters (no
    memset in the captured evaluation) and k_fin1p writes the status into mapped host memory,
    read instead of a device-to-host copy only when this call ran k_fin1p.  Every order of
    calls -- gradient with and without a rate pass first, repeated calls, rates, an input
    error and recovery, a committed block move (which updates ell on the device without
    k_fin1p) -- must give a fresh context's results."""
    from paper_2010_02994_b200 import HawkesContext, HawkesError
    c = synth.unit_square(1500, config=29)
    x2 = c.x + 0.002
    xbad = c.x.copy()
    xbad[7, 1] = np.nan

    def fresh(x):
        with HawkesContext(c.N, c.D, precision=precision) as f:
            f.set_times(c.t)
            f.set_locations(x)
            f.set_params(c.theta)
            g, e = f.grad_locations()
            return e, g.cpu().numpy(), f.get_rates()["lambda"]

    e1, g1, l1 = fresh(c.x)
    e2, g2, l2 = fresh(x2)
    with HawkesContext(c.N, c.D, precision=precision) as ctx:
        ctx.set_times(c.t)
        ctx.set_params(c.theta)
        for rep in range(3):   # plain launches first, then graph replays
            ctx.set_locations(c.x)
            g, e = ctx.grad_locations()                      # rate + gradient pass
            assert e == e1 and np.array_equal(g.cpu().numpy(), g1)
            g, e = ctx.grad_locations()                      # gradient already held
            assert e == e1 and np.array_equal(g.cpu().numpy(), g1)
            ctx.set_locations(x2)
            assert np.array_equal(ctx.get_rates()["lambda"], l2)   # rate pass only
            assert ctx.loglik() == e2                        # rates held: no evaluation
            g, e = ctx.grad_locations()                      # gradient pass only
            assert e == e2 and np.array_equal(g.cpu().numpy(), g2)
            ctx.set_locations(torch.from_numpy(xbad).cuda())   # validated on the device
            with pytest.raises(HawkesError):
                ctx.grad_locations()
            ctx.set_locations(c.x)
            assert ctx.loglik() == e1
            assert np.array_equal(ctx.get_rates()["lambda"], l1)
        # a committed move updates ell on the device; loglik must not return the last mirror
        idx = np.array([3, 400], dtype=np.int32)
        new = c.x[idx] + 0.01
        d = ctx.propose_move(idx, new)
        ctx.accept_move()
        xm = c.x.copy()
        xm[idx] = new
        em, gm, _ = fresh(xm)
        # (fp32 contexts: the committed rates and ell come from the move kernels' own sums)
        assert ctx.loglik() == pytest.approx(e1 + d, rel=1e-12 if precision == "fp64" else 1e-9)
        assert ctx.loglik() == pytest.approx(em, rel=1e-9 if precision == "fp64" else 1e-5)
        g, e = ctx.grad_locations()
        assert e == pytest.approx(em, rel=1e-9 if precision == "fp64" else 1e-5)


def test_full_size_c4_gradient_rows_vs_oracle():
    """BASELINE configs[3] at N = 100k in the bench's launch configuration: the oracle's
    rates for all events (O(N^2), ~30 s on the host cores), then its App. A gradient for
    sampled rows, against the GPU gradient under the fp64 tolerance rule."""
    c = synth.config("C4")
    from paper_2010_02994_b200 import HawkesContext
    with HawkesContext(c.N, 2) as ctx:
        ctx.set_times(torch.from_numpy(c.t).cuda())
        ctx.set_params(c.theta)
        ctx.set_locations(torch.from_numpy(c.x).cuda())
        g, ell = ctx.grad_locations()
        g = g.cpu().numpy()
    lam, _, _ = oracle.rates(c.x, c.t, c.theta)
    Lam = oracle.Lambda(c.t, c.theta)
    ell_ref = math.fsum(np.log(lam) - Lam)
    assert abs(ell - ell_ref) <= 1e-9 * abs(ell_ref)
    rows = np.unique(np.concatenate([np.arange(0, c.N, 997), [c.N - 1, 127, 128, 767, 768]]))
    for r in rows[::8]:
        gr, S = oracle.grad(c.x, c.t, c.theta, lam=lam, rows=slice(int(r), int(r) + 1))
        bound = 1e-9 * np.maximum(np.abs(gr[r]), 1e-3 * S[r])
        assert np.all(np.abs(g[r] - gr[r]) <= bound), (r, g[r], gr[r])


def test_gpu_invariances():
    """SURVEY T3 on the GPU output: translation and rotation of X leave ell unchanged and
    rotate g; scaling X, tau_x and h by a gives ell - N D log a and g / a (P7)."""
    from paper_2010_02994_b200 import HawkesContext
    c = synth.unit_square(4000, config=30)
    ell, g, _ = gpu_eval(c.x, c.t, c.theta, with_rates=False)
    S = np.abs(g).sum()
    e2, g2, _ = gpu_eval(c.x + np.array([12.5, -3.25]), c.t, c.theta, with_rates=False)
    assert e2 == pytest.approx(ell, rel=1e-12) and np.abs(g2 - g).max() <= 1e-10 * np.abs(g).max()
    a = 0.3
    R = np.array([[math.cos(a), -math.sin(a)], [math.sin(a), math.cos(a)]])
    e3, g3, _ = gpu_eval(c.x @ R.T, c.t, c.theta, with_rates=False)
    assert e3 == pytest.approx(ell, rel=1e-12)
    assert np.abs(g3 - g @ R.T).max() <= 1e-10 * np.abs(g).max()
    s = 7.0
    th = list(c.theta)
    th[1] *= s
    th[5] *= s
    e4, g4, _ = gpu_eval(s * c.x, c.t, th, with_rates=False)
    assert e4 == pytest.approx(ell - c.N * c.D * math.log(s), rel=1e-12)
    assert np.abs(g4 - g / s).max() <= 1e-10 * np.abs(g).max() / s


def test_leapfrog_energy_error_is_second_order():
    """the leapfrog's energy error |Delta H| shrinks ~4x when the step halves
    (second-order integrator; H = -ell + K)."""
    from paper_2010_02994_b200 import HawkesContext
    c = synth.config("C1", replicate=5)
    p0 = synth.momenta(c.N, c.D, seed=21)
    with HawkesContext(c.N, c.D) as ctx:
        ctx.set_times(c.t)
        ctx.set_params(c.theta)
        ctx.set_locations(c.x)
        H0 = -ctx.loglik() + 0.5 * float(np.sum(p0 * p0))
        errs = []
        T = 4e-3
        for L in (8, 16, 32):
            x, p = c.x.copy(), p0.copy()
            _, _, ell, kin = ctx.leapfrog(x, p, T / L, L)
            errs.append(abs(-ell + kin - H0))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.0 < r1 < 5.5 and 3.0 < r2 < 5.5, errs


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_largest_size_1m_sampled_rows_and_properties(precision):
    """The scaling sweep's largest size (BASELINE configs[3], N = 1M): lambda on sampled rows
    against the oracle computed row by row (O(N) each), sum_n g_n = 0, and the directional
    derivative of the GPU's own ell against <g, V> -- the properties that hold at any size
    (the oracle's full gradient would need every rate, O(N^2) = 1e12 pair terms)."""
    from paper_2010_02994_b200 import HawkesContext
    c = synth.config("C4", 1_000_000)
    N = c.N
    rows = np.unique(np.concatenate([np.arange(0, N, N // 12), [N - 1, 767, 768]]))
    tol = 1e-11 if precision == "fp64" else 1e-4
    with HawkesContext(N, 2, precision=precision) as ctx:
        ctx.set_times(torch.from_numpy(c.t).cuda())
        ctx.set_params(c.theta)
        x = torch.from_numpy(c.x).cuda()
        ctx.set_locations(x)
        g, ell = ctx.grad_locations()
        g = g.cpu().numpy()
        lam = ctx.get_rates()["lambda"]
        for r in rows:
            ref = oracle.rates(c.x, c.t, c.theta, rows=slice(int(r), int(r) + 1))[0][r]
            assert abs(lam[r] - ref) <= tol * ref, (r, lam[r], ref)
        gs = np.abs(g).sum(axis=0)
        assert np.all(np.abs(g.sum(axis=0)) <= (1e-11 if precision == "fp64" else 1e-5) * gs)
        if precision == "fp64":
            V = np.random.default_rng(5).normal(size=c.x.shape)
            eps = 1e-6
            ctx.set_locations(x + eps * torch.from_numpy(V).cuda())
            lp = ctx.loglik()
            ctx.set_locations(x - eps * torch.from_numpy(V).cuda())
            lm = ctx.loglik()
            assert abs((lp - lm) / (2 * eps) - float(np.sum(g * V))) <= 1e-6 * np.sum(np.abs(g * V))


def _fuzz_case(seed, case, nmax):
    import importlib.util
    import os
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "fuzz_parity.py")
    spec = importlib.util.spec_from_file_location("fuzz_parity", p)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    rng = np.random.default_rng(seed)
    for _ in range(case + 1):
        out = mod.make_case(rng, nmax)
    return out


@pytest.mark.parametrize("algorithm", ["pairs", "rows"])
def test_fp32_range_guard_falls_back_to_fp64(algorithm):
    """Reading R23: round 1's one fuzz failure (seed 12, case 290: D = 7, lambda_n from 4e-35
    to 6e-11) lost rate terms to the fp32 flush.  The range guard now detects it, the call is
    redone by the fp64 kernels (precision_in_use reports fp64) and the result meets the fp32
    gate -- in fact the fp64 one; set_params re-arms fp32.  A well-scaled catalog stays on fp32."""
    from paper_2010_02994_b200 import HawkesContext
    N, D, x, t, th, _, _, _ = _fuzz_case(12, 290, 4000)
    ell_r, _, _, g_r, S = oracle_eval(x, t, th)
    with HawkesContext(N, D, precision="fp32", algorithm=algorithm) as ctx:
        ctx.set_times(t)
        ctx.set_locations(x)
        ctx.set_params(th)
        assert ctx.precision_in_use == "fp32"
        g, ell = ctx.grad_locations()
        assert ctx.precision_in_use == "fp64"
        assert_parity(ell, g.cpu().numpy(), ell_r, g_r, S, precision="fp64", what="guarded fp32")
        ctx.set_params(th)
        assert ctx.precision_in_use == "fp32"
        assert ctx.loglik() == pytest.approx(ell_r, rel=1e-9)      # loglik alone trips it too
        assert ctx.precision_in_use == "fp64"
    c = synth.config("C3", 3000)
    with HawkesContext(c.N, c.D, precision="fp32", algorithm=algorithm) as ctx:
        ctx.set_times(c.t)
        ctx.set_locations(c.x)
        ctx.set_params(c.theta)
        g, ell = ctx.grad_locations()
        assert ctx.precision_in_use == "fp32"
    ell_r, _, _, g_r, S = oracle_eval(c.x, c.t, c.theta)
    assert_parity(ell, g.cpu().numpy(), ell_r, g_r, S, precision="fp32", what="C3 fp32")


def test_fp32_range_guard_in_leapfrog_and_hmc():
    """The guarded catalog through the samplers: an fp32 leapfrog / HMC transition returns the
    fp64 trajectory / decision (same as an fp64 context)."""
    from paper_2010_02994_b200 import HawkesContext
    N, D, x, t, th, _, _, _ = _fuzz_case(12, 290, 4000)
    p0 = synth.momenta(N, D, seed=5)
    res = {}
    for prec in ("fp32", "fp64"):
        with HawkesContext(N, D, precision=prec) as ctx:
            ctx.set_times(t)
            ctx.set_params(th)
            xx = torch.from_numpy(x.copy()).cuda()
            pp = torch.from_numpy(p0.copy()).cuda()
            _, _, ell, kin = ctx.leapfrog(xx, pp, 1e-3, 3)
            ctx.set_params(th)                       # re-arm fp32 for the HMC transition
            ctx.set_locations(x)
            acc, la = ctx.hmc_step(3, 1, 1e-3, 3)
            res[prec] = (xx.cpu().numpy(), ell, kin, acc, la, ctx.precision_in_use)
    assert res["fp32"][5] == "fp64"
    assert np.allclose(res["fp32"][0], res["fp64"][0], rtol=0, atol=1e-12 * np.abs(x).max())
    assert res["fp32"][1] == pytest.approx(res["fp64"][1], rel=1e-12)
    assert res["fp32"][3] == res["fp64"][3] and res["fp32"][4] == pytest.approx(res["fp64"][4], abs=1e-9)
