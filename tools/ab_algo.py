"""PAIRS (unordered-pair sym kernels) vs ROWS (ordered-pair pass kernels) per D: ms per
ell + gradient evaluation (library CUDA events), unit-square catalogs.

    python tools/ab_algo.py [--dims 2,3,4,5,6,7,8] [--sizes 4733,20000] [--precision fp64]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dims", default="2,3,4,5,6,7,8")
ap.add_argument("--sizes", default="4733,20000")
ap.add_argument("--precision", default="fp64")
a = ap.parse_args()
for N in [int(v) for v in a.sizes.split(",")]:
    for D in [int(v) for v in a.dims.split(",")]:
        c = synth.unit_square(N, config=4, D=D)
        row = {"N": N, "D": D, "precision": a.precision}
        for alg in ("pairs", "rows"):
            ctx = HawkesContext(N, D, precision=a.precision, algorithm=alg)
            ctx.set_times(c.t)
            x = torch.from_numpy(c.x).cuda()
            ctx.set_params(c.theta)
            g = torch.empty_like(x)
            for _ in range(3):
                ctx.set_locations(x)
                ctx.grad_locations(g)
            ctx.enable_timing(True)
            for _ in range(5):
                ctx.set_locations(x)
                ctx.grad_locations(g)
            kt = ctx.kernel_times()
            row[alg + "_ms"] = (kt["rate_ms"] + kt["grad_ms"]) / 5
            ctx.close()
        print(json.dumps(row), flush=True)
