"""The C-ABI library builds, loads and exports what include/hawkes.h declares (no GPU
compute here), and the host-side sharding plan is sound."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hawkes.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hawkes_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2010_02994_b200 import _lib
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 15
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.EXPORTS)
    assert lib.hawkes_abi_version() == 4


def test_library_is_sm100a():
    from paper_2010_02994_b200 import _lib
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_device_fails_loudly():
    """No silent fallback: without a GPU hawkes_create reports HAWKES_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import ctypes
    from paper_2010_02994_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.hawkes_create(100, 2, None, ctypes.byref(h))
    assert rc == -8 and not h.value
    assert lib.hawkes_last_error(None)


@pytest.mark.parametrize("N", [1, 255, 256, 257, 5000, 100_000, 1_000_000])
@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
def test_plan_partitions_rows(N, W):
    from paper_2010_02994_b200 import sharding
    seen = []
    counts = []
    chunks = set()
    for r in range(W):
        tiles, rt, ck = sharding.plan(N, W, r)
        seen += tiles
        counts.append(len(tiles))
        chunks.add(ck)
    nt = (N + rt - 1) // rt
    assert sorted(seen) == list(range(nt))           # every row tile exactly once
    assert max(counts) - min(counts) <= 1            # balanced tile counts
    assert len(chunks) == 1                          # chunking independent of rank
    _, _, ck1 = sharding.plan(N, 1, 0)
    assert chunks == {ck1}                           # ... and of W


def test_plan_zigzag_balances_causal_work():
    """Rate-pass work of row i grows with i (self-excitation over t_j < t_i); the zig-zag
    deal keeps every rank within 1% of the mean at N=100k, W=8."""
    from paper_2010_02994_b200 import sharding
    N, W = 100_000, 8
    work = []
    for r in range(W):
        rows = sharding.rows_of(N, W, r)
        work.append(sum(N * 25 + i * 19 for i in rows))
    mean = sum(work) / W
    assert max(work) / mean < 1.01


def test_nccl_unique_id_is_fresh():
    from paper_2010_02994_b200 import nccl_unique_id
    a, b = nccl_unique_id(), nccl_unique_id()
    assert len(a) == 128 and a != b


@pytest.mark.parametrize("N", [1, 300, 5000, 16_384, 20_000, 100_000, 1_000_000])
@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_pair_plan_covers_every_pair_once(N, W):
    """HAWKES_ALGO_PAIRS: the chunk pairs (a <= b) of all ranks cover each unordered chunk
    pair exactly once, and the LPT deal balances pair counts within a few percent."""
    from paper_2010_02994_b200 import sharding
    seen = set()
    loads = []
    chunk = None
    for r in range(W):
        items, ck = sharding.plan_pairs(N, W, r)
        chunk = ck if chunk is None else chunk
        assert ck == chunk
        load = 0
        for a, b in items:
            assert a <= b and (a, b) not in seen
            seen.add((a, b))
            na = min(ck, N - a * ck)
            nb = min(ck, N - b * ck)
            load += na * na if a == b else 2 * na * nb
        loads.append(load)
    C = (N + chunk - 1) // chunk
    assert seen == {(a, b) for a in range(C) for b in range(a, C)}
    assert sum(loads) == N * N
    assert chunk % 128 == 0
    if N >= 100_000:
        assert max(loads) / (sum(loads) / W) < 1.03


@pytest.mark.parametrize("N,W,chunk", [(5000, 1, 128), (16_383, 1, 128), (16_384, 1, 256),
                                       (20_000, 1, 256), (20_000, 2, 128), (23_168, 2, 128), (23_200, 2, 256),
                                       (50_000, 1, 384), (100_000, 1, 768), (100_000, 8, 256)])
def test_pair_chunk_heuristic(N, W, chunk):
    """chunk_pairs_of (hawkes_plan.h): ~N / (138 sqrt(W)) rounded to 128-event tiles, floored
    at 256 events where that leaves >= 64 sqrt(W) chunks (profiles/r01_chunk_sweep.txt,
    r01_chunk256.txt)."""
    from paper_2010_02994_b200 import sharding
    assert sharding.plan_pairs(N, W, 0)[1] == chunk


def test_spatial_walk_plan_host_logic():
    """hawkes_plan_walk (the host logic of the AUTO walk order): the walk
    is a permutation; it is spatially local (consecutive events of the walk are far closer
    than random pairs); the box-based work estimate prefers it on the DC shape (16 km across,
    3.7 km cutoff) and not on the unit square (nothing to cull), and a pure translation or a
    reversal of the time axis does not change the costs."""
    import numpy as np

    import synth
    from paper_2010_02994_b200 import sharding
    for name, N, want in (("C2", 20000, True), ("C4", 20000, False)):
        c = synth.config(name, N)
        perm, (ct, cs) = sharding.plan_walk(c.x, c.t, c.theta)
        assert sorted(perm) == list(range(N))
        xp = c.x[perm]
        step = np.mean(np.linalg.norm(np.diff(xp, axis=0), axis=1))
        rnd = np.mean(np.linalg.norm(c.x[1:] - c.x[:-1], axis=1))   # time order ~ random in space
        assert step < 0.05 * rnd, (name, step, rnd)
        assert (cs < 0.9 * ct) == want, (name, ct, cs)
        perm2, (ct2, cs2) = sharding.plan_walk(c.x + 1e3, c.t, c.theta)
        assert perm2 == perm and abs(ct2 - ct) <= 1e-9 * ct and abs(cs2 - cs) <= 1e-9 * cs


@pytest.mark.parametrize("N", [5000, 100_000, 1_000_000])
def test_compact_slot_layout_footprint(N):
    """hawkes_plan_slots: PAIRS' item-indexed slot blocks.  At W = 1 a rank holds (C + 1) C
    chunk events (every chunk has C + 1 slots); at W ranks the blocks are split without overlap
    (the ranks' counts add up to the same total for that W's chunk) and each rank holds about
    1/W of them (the full [C+1][Npad][K] arrays on every rank were ~12 GB at
    N = 1M, W = 8)."""
    from paper_2010_02994_b200 import sharding
    for W in (1, 2, 4, 8):
        _, chunk = sharding.plan_pairs(N, W, 0)
        C = (N + chunk - 1) // chunk
        per = [sharding.plan_slots(N, W, r)[0] for r in range(W)]
        assert sum(per) == (C + 1) * C * chunk
        assert sharding.plan_slots(N, W, 0)[1] == max(per)
        assert max(per) <= 1.35 * (C + 1) * C * chunk / W + 4 * chunk * (C + 1), (W, per)


@pytest.mark.parametrize("N,W,resident,k_want", [(500, 1, 592, 8), (2000, 1, 592, 4), (3000, 1, 592, 1),
                                                 (5000, 1, 592, 1), (2000, 3, 444, 8), (7000, 2, 592, 2),
                                                 (2000, 1, 0, 1)])
def test_plan_items_pieces_cover_every_pair_once(N, W, resident, k_want):
    """hawkes_plan_items (DESIGN.md §5 "Small N"): below one round of `resident` CTA slots
    every item runs as k pieces whose step ranges partition [0, 32); every piece owns its
    own row and column blocks, so the blocks of all pieces tile [0, slot_events) exactly
    once, and each chunk's blocks are as many as its slot count; the pieces of an item keep
    the item's chunk pair, and the chunk pairs are hawkes_plan_pairs' (a <= b) on that rank."""
    from paper_2010_02994_b200 import sharding
    total = 0
    for r in range(W):
        items, k, se = sharding.plan_items(N, W, r, resident)
        pairs, chunk = sharding.plan_pairs(N, W, r)
        n_pairs = len(pairs)
        assert k == (k_want if W == 1 or k_want == 1 else k) and k in (1, 2, 4, 8)
        if resident:
            assert k == 1 or k * n_pairs <= resident
            assert k == 8 or 2 * k * n_pairs > resident   # the largest k that fits
        assert len(items) == k * n_pairs
        assert sorted({(int(a), int(b)) for a, b in items[:, :2]}) == sorted(map(tuple, pairs))
        steps = {}
        for a, b, ro, co, s0, s1 in items:
            steps.setdefault((a, b), []).append((s0, s1))
        for rngs in steps.values():
            rngs.sort()
            assert rngs[0][0] == 0 and rngs[-1][1] == 32
            assert all(rngs[q][1] == rngs[q + 1][0] for q in range(len(rngs) - 1))
            assert len({s1 - s0 for s0, s1 in rngs}) == 1
        blocks = sorted([int(ro) for ro in items[:, 2]] + [int(co) for co in items[:, 3]])
        assert blocks == list(range(0, se, chunk)), "every block owned by exactly one (piece, role)"
        total += se
    if W == 1 and k_want == 1:
        assert total == sharding.plan_slots(N, W, 0)[0]
