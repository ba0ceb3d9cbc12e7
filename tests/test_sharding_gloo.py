"""Multi-process tests of the sharded paths on CPU (gloo, world size 2 and 3): the NCCL
unique-id hand-off; ROWS (rows by hawkes_plan, allgather of 1/lambda between the passes,
allgather of gradient rows); and PAIRS, the default (chunk pairs dealt by
hawkes_plan_pairs, per-rank per-event sums exchanged by allgather and added in rank order,
as hawkes_engine.cuh's reduce_pair_partials does).  The per-shard compute is the oracle's
pair terms restricted to the shard (the GPU kernels need a device); the plans are the
library's own (its C ABI, called on the CPU) and the exchange is the library's pattern."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2010_02994_b200 import sharding

        uid = sharding.broadcast_unique_id()
        c = synth.unit_square(700, config=31)
        N = c.N
        rows = np.array(sharding.rows_of(N, world, rank))
        # pass 1 on own rows
        lam_own, _, _ = oracle.rates(c.x, c.t, c.theta)
        lam_own = lam_own[rows]
        # allgather 1/lambda (fixed-size messages, padded)
        tiles, rt, _ = sharding.plan(N, world, rank)
        maxrows = max(len(sharding.rows_of(N, world, r)) for r in range(world))
        send = torch.zeros(maxrows, dtype=torch.float64)
        send[: len(rows)] = torch.from_numpy(1.0 / lam_own)
        bufs = [torch.zeros(maxrows, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, send)
        rho = np.empty(N)
        for r in range(world):
            rr = sharding.rows_of(N, world, r)
            rho[rr] = bufs[r].numpy()[: len(rr)]
        # pass 2 on own rows with the gathered rates
        g, _ = oracle.grad(c.x, c.t, c.theta, lam=1.0 / rho)
        send = torch.zeros(maxrows, 2, dtype=torch.float64)
        send[: len(rows)] = torch.from_numpy(g[rows])
        bufs = [torch.zeros(maxrows, 2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(bufs, send)
        gfull = np.empty((N, 2))
        for r in range(world):
            rr = sharding.rows_of(N, world, r)
            gfull[rr] = bufs[r].numpy()[: len(rr)]
        q.put((rank, uid, gfull))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_sharded_evaluation():
    import oracle
    import synth
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    assert res[0][1] == res[1][1] and len(res[0][1]) == 128   # same NCCL id on both ranks
    c = synth.unit_square(700, config=31)
    g_ref, _ = oracle.grad(c.x, c.t, c.theta)
    for _, _, g in res:
        np.testing.assert_allclose(g, g_ref, rtol=1e-13, atol=1e-13 * np.abs(g_ref).max())


# ---- PAIRS (the default decomposition): the library's chunk-pair plan and its exchange ----

def _pair_partials(c, items, chunk, rho=None):
    """Per-event sums over the unordered pairs {i < j} of this rank's chunk pairs (a, b), a <= b
    (hawkes_plan_pairs), evaluated pair by pair with the oracle's P:L98-99 terms.  rho None:
    rate partials (each pair adds mu_ij + xi_ij to lambda_i and mu_ji + xi_ji to lambda_j);
    else App. A gradient partials c_ij (x_j - x_i) to g_i and -c_ij (x_j - x_i) to g_j, with
    c_ij = (mu_ij rho_i + mu_ji rho_j)/tau_x^2 + (xi_ij rho_i + xi_ji rho_j)/h^2.
    Also returns the visit count of every ordered (i, j), i < j."""
    import ctypes

    import oracle
    lib = oracle._load()
    x = np.ascontiguousarray(c.x)
    t = np.ascontiguousarray(c.t)
    N, D = x.shape
    xp, tp = oracle._dptr(x), oracle._dptr(t)
    p = ctypes.byref(oracle._params(c.theta))
    mu, xi = lib.oracle_mu_pair, lib.oracle_xi_pair
    tx2, h2 = c.theta[1] ** 2, c.theta[5] ** 2
    out = np.zeros(N) if rho is None else np.zeros((N, D))
    seen = np.zeros((N, N), dtype=np.int8)
    for a, b in items:
        for i in range(a * chunk, min(N, (a + 1) * chunk)):
            j0 = i + 1 if a == b else b * chunk
            for j in range(j0, min(N, (b + 1) * chunk)):
                seen[i, j] += 1
                m_ij, m_ji = mu(D, xp, tp, i, j, p), mu(D, xp, tp, j, i, p)
                x_ij, x_ji = xi(D, xp, tp, i, j, p), xi(D, xp, tp, j, i, p)
                if rho is None:
                    out[i] += m_ij + x_ij
                    out[j] += m_ji + x_ji
                else:
                    cc = (m_ij * rho[i] + m_ji * rho[j]) / tx2 + (x_ij * rho[i] + x_ji * rho[j]) / h2
                    d = cc * (x[j] - x[i])
                    out[i] += d
                    out[j] -= d
    return out, seen


def _rank_ordered_sum(local):
    """The library's PAIRS exchange (hawkes_engine.cuh reduce_pair_partials): allgather of the
    per-rank per-event sums, then added in rank order (same bits on every rank)."""
    bufs = [torch.zeros_like(torch.from_numpy(local)) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, torch.from_numpy(local))
    tot = bufs[0].numpy().copy()
    for b in bufs[1:]:
        tot += b.numpy()
    return tot


def _pairs_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2010_02994_b200 import sharding

        c = synth.unit_square(PAIRS_N, config=32)
        items, chunk = sharding.plan_pairs(c.N, world, rank)
        lam_loc, seen = _pair_partials(c, items, chunk)
        lam = _rank_ordered_sum(lam_loc)                 # S4
        g_loc, _ = _pair_partials(c, items, chunk, rho=1.0 / lam)
        g = _rank_ordered_sum(g_loc)                     # S6
        q.put((rank, len(items), chunk, seen, lam, g))
    finally:
        dist.destroy_process_group()


PAIRS_N = 700


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_pairs_plan_and_exchange(world):
    """W gloo ranks run the PAIRS decomposition exactly as the library deals it
    (hawkes_plan_pairs: LPT-dealt chunk pairs) and exchange per-event sums by allgather +
    rank-ordered sum: every unordered pair is visited by exactly one rank, the load is
    balanced, every rank holds bitwise the same lambda and gradient, and both match the
    oracle's unsharded evaluation."""
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pairs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = synth.unit_square(PAIRS_N, config=32)
    N = c.N
    seen = sum(r[3].astype(np.int32) for r in res)
    iu = np.triu_indices(N, 1)
    assert np.all(seen[iu] == 1), "some unordered pair is not visited exactly once"
    assert np.all(np.tril(seen) == 0)
    pairs_per_rank = [int(r[3].sum()) for r in res]
    assert max(pairs_per_rank) <= 1.25 * (N * (N - 1) / 2) / world
    for r in res[1:]:                                    # same bits on every rank
        assert np.array_equal(r[4], res[0][4]) and np.array_equal(r[5], res[0][5])
    lam_ref, _, _ = oracle.rates(c.x, c.t, c.theta)
    g_ref, S = oracle.grad(c.x, c.t, c.theta, lam=lam_ref)
    np.testing.assert_allclose(res[0][4], lam_ref, rtol=1e-13)
    assert np.all(np.abs(res[0][5] - g_ref) <= 1e-12 * np.maximum(np.abs(g_ref), S))
