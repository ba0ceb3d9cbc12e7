"""Uninitialised-memory probe: fill most of the device with NaN, release it to the driver, then
evaluate ell + gradient in each precision / algorithm and check for NaN against a clean run.

    python tools/nan_poison.py [N ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402


def poison(gb=40):
    x = torch.full((gb * (1 << 27),), float("nan"), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    del x
    torch.cuda.empty_cache()


def run(c, **kw):
    with HawkesContext(c.N, c.D, **kw) as ctx:
        ctx.set_times(c.t)
        ctx.set_locations(c.x)
        ctx.set_params(c.theta)
        ell = ctx.loglik()
        g, _ = ctx.grad_locations()
        lam = ctx.get_rates()["lambda"]
        return ell, g.cpu().numpy(), lam


sizes = [int(a) for a in sys.argv[1:]] or [1500, 777, 5000]
bad = 0
for N in sizes:
    c = synth.config("C1", N)
    for prec in ("fp64", "fp32"):
        for alg in ("pairs", "rows"):
            poison()
            ell, g, lam = run(c, precision=prec, algorithm=alg)
            nan = (not np.isfinite(ell)) or np.isnan(g).any() or np.isnan(lam).any()
            rows = np.where(np.isnan(g).any(axis=1))[0]
            print(f"N={N} {prec} {alg}: ell={ell!r} nan={nan} nan_rows={rows[:10].tolist()} "
                  f"n_nan_rows={len(rows)}", flush=True)
            bad += nan
print("BAD" if bad else "OK", bad)
