"""On-device block-MH sweep throughput (hawkes_mh_sweep), fp64.

    python tools/mh_bench.py [--configs C2:3982,C3:2925,C2:100000,C3:100000] [--ks 1,8,32]

Each line: one sweep of B blocks of k events (random distinct indices), timed with CUDA
events around the call (one host sync per sweep); blocks/s, event updates/s, acceptance.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C2:3982,C3:2925,C2:100000,C3:100000")
ap.add_argument("--ks", default="1,8,32")
ap.add_argument("--blocks", type=int, default=2000)
a = ap.parse_args()
for spec in a.configs.split(","):
    name, N = spec.split(":")
    N = int(N)
    c = synth.config(name, N)
    ctx = HawkesContext(N, 2)
    ctx.set_times(c.t)
    ctx.set_locations(c.x)
    ctx.set_params(c.theta)
    ctx.set_regions(c.region, c.centre, c.size)
    rng = np.random.default_rng(0)
    scale = 0.5 if c.region == "square" else 0.7
    for k in [int(s) for s in a.ks.split(",")]:
        B = max(50, a.blocks // max(1, k // 4))
        blocks = np.stack([rng.choice(N, size=k, replace=False) for _ in range(B)]).astype(np.int32)
        ctx.mh_sweep(blocks[:20], scale, 1, 0)         # warm-up (rates computed once)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(ctx.stream)
        acc, la = ctx.mh_sweep(blocks, scale, 1, 1)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"config": name, "N": N, "region": c.region, "k": k, "blocks": B,
                          "scale": scale, "us_per_block": ms * 1e3 / B, "blocks_per_s": B / (ms * 1e-3),
                          "event_updates_per_s": B * k / (ms * 1e-3), "acceptance": float(acc.mean())}),
              flush=True)
    ctx.close()
