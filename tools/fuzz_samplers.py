"""Randomised sampler parity: MH sweeps (random region kind / D, k, block count, scale) and
HMC transitions (random step, length, diagonal mass) on random small catalogs, against the
oracle's transitions (decisions, log alpha, final state).  Decisions within 1e-6 of
log u are not compared (genuine ties).

    python tools/fuzz_samplers.py [--cases 60] [--seed 1]
"""
import argparse
import json
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=60)
ap.add_argument("--seed", type=int, default=1)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
fails = 0
for case in range(a.cases):
    kind = "disc" if rng.uniform() < 0.4 else "square"
    D = 2 if kind == "disc" else int(rng.integers(1, 5))
    N = int(rng.integers(20, 600))
    c0 = synth.unit_square(N, config=40 + case % 7, replicate=case, D=D)
    if kind == "square":
        hw = float(10 ** rng.uniform(-3, -1.5))
        centre = 2 * hw * np.round(c0.x / (2 * hw))
        size = np.full(N, hw)
    else:
        size = 10 ** rng.uniform(-3, -1.5, size=N)
        ang = rng.uniform(0, 2 * np.pi, N)
        rad = size * np.sqrt(rng.uniform(size=N)) * 0.999
        centre = c0.x - np.column_stack([rad * np.cos(ang), rad * np.sin(ang)])
    k = int(rng.integers(1, min(16, N) + 1))
    nb = int(rng.integers(1, 20))
    blocks = np.stack([rng.choice(N, size=k, replace=False) for _ in range(nb)]).astype(np.int32)
    scale = float(10 ** rng.uniform(-1, 0.5))
    seed, it = int(rng.integers(0, 2**40)), int(rng.integers(0, 2**33))
    info = {"case": case, "kind": kind, "D": D, "N": N, "k": k, "blocks": nb, "scale": scale}
    try:
        x_ref, acc_ref, la_ref = oracle.mh_sweep(c0.x, c0.t, c0.theta, kind, centre, size, blocks, scale, seed, it)
        with HawkesContext(N, D) as ctx:
            ctx.set_times(c0.t)
            ctx.set_locations(c0.x)
            ctx.set_params(c0.theta)
            ctx.set_regions(kind, centre, size)
            acc, la = ctx.mh_sweep(blocks, scale, seed, it)
            same = True
            for b in range(nb):
                lu = np.log(oracle.mh_uniforms(seed, it, b, 0xC0000000)[0])
                if abs(la_ref[b] - lu) > 1e-6 and bool(acc[b]) != bool(acc_ref[b]):
                    same = False
            if not same:
                fails += 1
                print(json.dumps({**info, "fail": "mh decision"}), flush=True)
                continue
            if list(acc) == list(acc_ref):
                x = ctx.get_locations().cpu().numpy()
                if np.max(np.abs(x - x_ref)) > 1e-12 * max(1.0, np.abs(x_ref).max()):
                    fails += 1
                    print(json.dumps({**info, "fail": "mh state"}), flush=True)
                    continue
                if not np.allclose(la, la_ref, rtol=1e-7, atol=1e-7):
                    fails += 1
                    print(json.dumps({**info, "fail": "mh log alpha"}), flush=True)
                    continue
            # an HMC transition from the chain's state
            step = float(10 ** rng.uniform(-4, -2.3))
            L = int(rng.integers(0, 8))
            minv = rng.uniform(0.5, 2.0, size=x_ref.shape) if rng.uniform() < 0.5 else None
            ctx.set_locations(x_ref)
            xr, ar, lr = oracle.hmc_step(x_ref, c0.t, c0.theta, seed, it, step, L, inv_mass=minv)
            xo = np.empty_like(x_ref)
            ah, lh = ctx.hmc_step(seed, it, step, L, inv_mass=minv, x_out=xo)
            lu = np.log(oracle.hmc_uniform(seed, it))
            if abs(lr - lu) > 1e-6 and ah != ar:
                fails += 1
                print(json.dumps({**info, "fail": "hmc decision", "la": lh, "la_ref": lr}), flush=True)
            elif ah == ar and np.max(np.abs(xo - xr)) > 1e-9 * max(1.0, np.abs(xr).max()):
                fails += 1
                print(json.dumps({**info, "fail": "hmc state"}), flush=True)
    except Exception as e:  # noqa: BLE001
        fails += 1
        print(json.dumps({**info, "fail": "exception", "error": repr(e)[:300]}), flush=True)
        traceback.print_exc()
print(json.dumps({"summary": True, "cases": a.cases, "fails": fails}), flush=True)
