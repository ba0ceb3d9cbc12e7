"""BMDS log density + gradient timing, and the flu model's joint HMC trajectory
(Hawkes + BMDS potential) on the flu shape (N = 4733, D = 6).

    python tools/bmds_bench.py [--sizes 4733,20000] [--D 6]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="4733,20000")
ap.add_argument("--D", type=int, default=6)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
for N in [int(v) for v in a.sizes.split(",")]:
    c, Y, s = synth.flu_shaped(N, a.D)
    ctx = HawkesContext(N, a.D)
    ctx.set_times(c.t)
    ctx.set_locations(torch.from_numpy(c.x).cuda())
    ctx.set_params(c.theta)
    ctx.set_bmds(torch.from_numpy(Y).cuda(), s)
    del Y
    g = torch.empty((N, a.D), dtype=torch.float64, device="cuda")
    ctx.bmds_logdensity(out=g)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        ctx.bmds_logdensity(out=g)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    ctx.set_potential(hawkes=True, bmds=True)
    x = torch.from_numpy(c.x.copy()).cuda()
    p = torch.from_numpy(synth.momenta(N, a.D)).cuda()
    ctx.leapfrog(x, p, 1e-4, 2)
    e0.record()
    ctx.leapfrog(x, p, 1e-4, 20)
    e1.record()
    torch.cuda.synchronize()
    traj = e0.elapsed_time(e1)
    print(json.dumps({"N": N, "D": a.D, "bmds_ms": ms, "bmds_pairs_per_s": N * (N - 1) / (ms * 1e-3),
                      "joint_trajectory_20_steps_ms": traj}), flush=True)
    ctx.close()
