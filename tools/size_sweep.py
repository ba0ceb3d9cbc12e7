"""ell + gradient time vs N (C4 generator, fp64 and fp32): BASELINE configs[3] sweep.

    python tools/size_sweep.py [--sizes 100000,250000,500000,1000000] [--precision fp64]
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
ap.add_argument("--sizes", default="100000,250000,500000,1000000")
ap.add_argument("--precision", default="fp64")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
for N in [int(s) for s in a.sizes.split(",")]:
    c = synth.config("C4", N=N)
    ctx = HawkesContext(N, 2, precision=a.precision)
    x = torch.from_numpy(c.x).cuda()
    ctx.set_times(torch.from_numpy(c.t).cuda())
    ctx.set_params(c.theta)
    g = torch.empty_like(x)
    for _ in range(3):               # warm-up (the second call captures the CUDA graph)
        ctx.set_locations(x)
        ctx.grad_locations(g)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        ctx.set_locations(x)
        _, ell = ctx.grad_locations(g)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / a.reps
    print(json.dumps({"N": N, "precision": a.precision, "ms_per_eval": ms,
                      "pairs_per_s": N * (N - 1) / (ms * 1e-3), "ell": ell,
                      "grad_sum_abs": float(g.sum(0).abs().max()),
                      "mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
    ctx.close()
