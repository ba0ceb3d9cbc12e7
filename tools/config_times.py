"""ell + gradient time on the BASELINE config shapes (C1..C4, plus larger DC/Alaska-shaped
catalogs), fp64 and fp32, after 3 warm-ups (graph replay).

    python tools/config_times.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

cases = [("C1", None), ("C2", None), ("C3", None), ("C2", 100_000), ("C3", 100_000), ("C4", None)]
for prec in ("fp64", "fp32"):
    for name, N in cases:
        c = synth.config(name, N=N)
        ctx = HawkesContext(c.N, c.D, precision=prec)
        x = torch.from_numpy(c.x).cuda()
        ctx.set_times(torch.from_numpy(c.t).cuda())
        ctx.set_params(c.theta)
        g = torch.empty_like(x)
        for _ in range(3):
            ctx.set_locations(x)
            ctx.grad_locations(g)
        reps = 20 if c.N <= 20000 else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            ctx.set_locations(x)
            ctx.grad_locations(g)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"config": name, "N": c.N, "precision": prec, "ms_per_eval": round(ms, 4),
                          "pairs_per_s": c.N * (c.N - 1) / (ms * 1e-3)}), flush=True)
        ctx.close()
