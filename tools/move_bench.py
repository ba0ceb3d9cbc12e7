"""Block-MH proposal throughput (hawkes_propose_move + 50 % accepts), fp64.

    python tools/move_bench.py [--sizes 3982,20000,100000] [--ks 1,16,64]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="3982,20000,100000")
ap.add_argument("--ks", default="1,16,64")
ap.add_argument("--reps", type=int, default=200)
a = ap.parse_args()
for N in [int(s) for s in a.sizes.split(",")]:
    c = synth.dc_shaped(N) if N < 10000 else synth.unit_square(N, config=4)
    ctx = HawkesContext(N, 2)
    ctx.set_times(c.t)
    ctx.set_locations(c.x)
    ctx.set_params(c.theta)
    rng = np.random.default_rng(0)
    step = 30.0 if N < 10000 else 0.005
    for k in [int(s) for s in a.ks.split(",")]:
        moves = [(rng.choice(N, size=k, replace=False).astype(np.int32)) for _ in range(a.reps)]
        ctx.propose_move(moves[0], c.x[moves[0]])      # first call computes the rates
        t0 = time.perf_counter()
        for r, idx in enumerate(moves):
            new = c.x[idx] + rng.uniform(-step, step, size=(k, 2))
            ctx.propose_move(idx, new)
            if r % 2 == 0:
                ctx.accept_move()
                c.x[idx] = new
        dt = (time.perf_counter() - t0) / a.reps
        print(json.dumps({"N": N, "k": k, "us_per_proposal": dt * 1e6, "proposals_per_s": 1.0 / dt,
                          "pair_terms_per_s": 2 * k * N / dt}), flush=True)
    ctx.close()
