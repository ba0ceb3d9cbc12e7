"""Per-call latency of a Theta update: set_params (new constants) + loglik, as an MH step over
the Hawkes parameters makes it (the locations unchanged), at the paper's catalog sizes.

    python tools/theta_latency.py [--sizes 2925,3982,4733,20000]
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
ap.add_argument("--sizes", default="2925,3982,4733,20000")
ap.add_argument("--reps", type=int, default=300)
a = ap.parse_args()
for N in [int(v) for v in a.sizes.split(",")]:
    c = synth.config("C1", N)
    ctx = HawkesContext(N, 2)
    ctx.set_times(c.t)
    ctx.set_locations(c.x)
    ctx.set_params(c.theta)
    ctx.loglik()
    rng = np.random.default_rng(0)
    thetas = [tuple(v * f for v, f in zip(c.theta, 1 + 0.01 * rng.standard_normal(6))) for _ in range(a.reps)]
    for th in thetas[:20]:
        ctx.set_params(th)
        ctx.loglik()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for th in thetas:
        ctx.set_params(th)
        ctx.loglik()
    dt = (time.perf_counter() - t0) / a.reps
    # same-Theta repeated loglik (graph replay) for comparison
    ctx.set_params(c.theta)
    for _ in range(5):
        ctx.set_locations(c.x)
        ctx.loglik()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        ctx.set_locations(c.x)
        ctx.loglik()
    dt2 = (time.perf_counter() - t0) / a.reps
    print(json.dumps({"N": N, "theta_update_us": dt * 1e6, "same_theta_us": dt2 * 1e6}), flush=True)
    ctx.close()
