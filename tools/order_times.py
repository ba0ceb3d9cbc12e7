"""Evaluation time of the PAIRS fp64 path per walk order (time / space / auto's choice) on the
config shapes: one ell + gradient evaluation (set_locations + grad_locations, the walk's
record gather included), CUDA events, median of reps.  SURVEY.md §8(f) NEXT-2.

    python tools/order_times.py [C2:5000 C2:100000 ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

PREC = "fp32" if "--fp32" in sys.argv else "fp64"
SIZES = [a.split(":") for a in sys.argv[1:] if a != "--fp32"] or [["C2", "5000"], ["C2", "20000"], ["C2", "100000"],
                                                  ["C3", "20000"], ["C3", "100000"], ["C4", "100000"]]
for name, n in SIZES:
    c = synth.config(name, int(n))
    x = torch.from_numpy(c.x).cuda()
    for mode in ("time", "space", "auto"):
        ctx = HawkesContext(c.N, c.D, precision=PREC)
        ctx.set_ordering(mode)
        ctx.set_times(torch.from_numpy(c.t).cuda())
        ctx.set_params(c.theta)
        g = torch.empty_like(x)
        for _ in range(3):
            ctx.set_locations(x)
            ctx.grad_locations(g)
        reps = 20 if c.N <= 20000 else 6
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            ctx.set_locations(x)
            _, ell = ctx.grad_locations(g)
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        order, cost = ctx.ordering_in_use
        print(json.dumps({"config": name, "N": c.N, "precision": PREC, "mode": mode, "order": order, "ms": ts[len(ts) // 2],
                          "pairs_per_s": c.N * (c.N - 1) / (ts[len(ts) // 2] * 1e-3),
                          "cost_time": cost[0], "cost_space": cost[1], "ell": ell}), flush=True)
        ctx.close()
