"""World-size-2 tests of the multi-process path on CPU (gloo): the NCCL unique-id hand-off,
and the sharded two-pass evaluation pattern (rows by hawkes_plan, allgather of 1/lambda
between the passes, allgather of gradient rows) reproducing the unsharded result.  The
per-shard compute here is the oracle restricted to the shard's rows (the GPU kernels need
a device); the plan and exchange pattern are the library's."""
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
