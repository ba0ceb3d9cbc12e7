"""Per-call latency of ell + gradient at small N (the paper's catalogs are N ~ 3-5k, called
millions of times by MCMC): device-input set_locations + grad_locations, host sync each call.

    python tools/latency.py [--sizes 500,2000,5000,20000] [--at]

--at: the one-call hawkes_grad_at (set_locations + grad_locations as one graph launch) as well.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="500,2000,5000,20000")
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--precision", default="fp64")
ap.add_argument("--at", action="store_true")
a = ap.parse_args()
for N in [int(s) for s in a.sizes.split(",")]:
    c = synth.unit_square(N, config=4)
    ctx = HawkesContext(N, 2, precision=a.precision)
    x = torch.from_numpy(c.x).cuda()
    ctx.set_times(torch.from_numpy(c.t).cuda())
    ctx.set_params(c.theta)
    g = torch.empty_like(x)
    for _ in range(5):
        ctx.set_locations(x)
        ctx.grad_locations(g)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        ctx.set_locations(x)
        _, ell = ctx.grad_locations(g)      # returns ell to the host: one sync per call
    dt = (time.perf_counter() - t0) / a.reps
    t0 = time.perf_counter()
    for _ in range(a.reps):
        ctx.set_locations(x)
        ell = ctx.loglik()
    dl = (time.perf_counter() - t0) / a.reps
    rec = {"N": N, "grad_us": dt * 1e6, "loglik_us": dl * 1e6, "pairs_per_s": N * (N - 1) / dt}
    if a.at:
        for _ in range(5):
            ctx.grad_at(x, g)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.reps):
            _, ell = ctx.grad_at(x, g)      # one call, one sync
        da = (time.perf_counter() - t0) / a.reps
        rec.update(grad_at_us=da * 1e6, grad_at_pairs_per_s=N * (N - 1) / da)
    print(json.dumps(rec), flush=True)
    ctx.close()
