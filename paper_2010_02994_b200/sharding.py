"""Multi-process plumbing for row sharding; argument marshalling only.

One process per GPU.  torch.distributed hands rank 0's NCCL unique id to every rank;
the library then builds its own NCCL communicator and does the exchange steps itself
(allgather of rho' = 1/lambda and ell_n between the passes, allgather of gradient rows).
"""
from __future__ import annotations

import ctypes
from typing import List, Tuple

import torch
import torch.distributed as dist

from . import _lib
from .hawkes import HawkesContext, nccl_unique_id


def plan(N: int, world: int, rank: int) -> Tuple[List[int], int, int]:
    """hawkes_plan: (row tiles of `rank`, rows per tile, j-chunk length)."""
    lib = _lib.load()
    n, rt, ck = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _lib.check(lib.hawkes_plan(N, world, rank, None, ctypes.byref(n), ctypes.byref(rt),
                               ctypes.byref(ck)))
    buf = (ctypes.c_int32 * max(1, n.value))()
    _lib.check(lib.hawkes_plan(N, world, rank, buf, ctypes.byref(n), None, None))
    return list(buf[: n.value]), rt.value, ck.value


def plan_pairs(N: int, world: int, rank: int) -> Tuple[List[Tuple[int, int]], int]:
    """hawkes_plan_pairs: (chunk pairs (a, b), a <= b, of `rank`; chunk length)."""
    lib = _lib.load()
    n, ck = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(lib.hawkes_plan_pairs(N, world, rank, None, ctypes.byref(n), ctypes.byref(ck)))
    buf = (ctypes.c_int32 * max(2, 2 * n.value))()
    _lib.check(lib.hawkes_plan_pairs(N, world, rank, buf, ctypes.byref(n), None))
    return [(buf[2 * k], buf[2 * k + 1]) for k in range(n.value)], ck.value


def plan_slots(N: int, world: int, rank: int) -> Tuple[int, int]:
    """hawkes_plan_slots: (this rank's partial-slot events, the largest over the ranks)."""
    lib = _lib.load()
    s, m = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(lib.hawkes_plan_slots(N, world, rank, ctypes.byref(s), ctypes.byref(m)))
    return s.value, m.value


def plan_items(N: int, world: int, rank: int, resident: int = 0):
    """hawkes_plan_items: (items as (a, b, row offset, column offset, s0, s1), pieces per
    item, slot events) of `rank` for a gradient pass of `resident` CTA slots."""
    import numpy as np
    lib = _lib.load()
    n, k, se = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    _lib.check(lib.hawkes_plan_items(N, world, rank, resident, None, ctypes.byref(n), None, None))
    out = np.zeros((max(1, n.value), 6), dtype=np.int64)
    _lib.check(lib.hawkes_plan_items(N, world, rank, resident,
                                     out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                     ctypes.byref(n), ctypes.byref(k), ctypes.byref(se)))
    return out[: n.value], k.value, se.value


def plan_walk(x, t, theta) -> Tuple[List[int], Tuple[float, float]]:
    """hawkes_plan_walk: (the spatial walk permutation, (time-walk cost, spatial-walk cost))."""
    import numpy as np
    lib = _lib.load()
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.ndim == 1:
        x = x[:, None]
    t = np.ascontiguousarray(t, dtype=np.float64)
    N, D = x.shape
    perm = np.empty(N, dtype=np.int32)
    cost = np.zeros(2)
    p = _lib.Params(*[float(v) for v in theta])
    _lib.check(lib.hawkes_plan_walk(x.ctypes.data, t.ctypes.data, N, D, ctypes.byref(p),
                                    perm.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                    cost.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
    return perm.tolist(), (float(cost[0]), float(cost[1]))


def rows_of(N: int, world: int, rank: int) -> List[int]:
    tiles, rt, _ = plan(N, world, rank)
    return [i for k in tiles for i in range(k * rt, min(N, (k + 1) * rt))]


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 creates an NCCL unique id; every rank returns the same 128 bytes."""
    rank = dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().tolist())


def init_distributed_context(N: int, D: int, precision: str = "fp64", group=None,
                             algorithm: str = "auto") -> HawkesContext:
    """hawkes_create on every rank of an initialised process group (world > 1 shards rows)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.cuda.current_device()
    if world == 1:
        return HawkesContext(N, D, device=dev, precision=precision, algorithm=algorithm)
    uid = broadcast_unique_id(group)
    return HawkesContext(N, D, device=dev, precision=precision, rank=rank, world=world, nccl_id=uid,
                         algorithm=algorithm)
