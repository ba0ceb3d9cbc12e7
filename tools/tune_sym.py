"""Time the PAIRS pass kernels for each sym_kernel variant (HAWKES_SYM_VARIANT = 10*R + V)
at N = 100k fp64 and check every variant against the default on a small catalog.

    python tools/tune_sym.py [--n 100000] [--variants 40,41,20,21]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--variants", default="40,41,20,21")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()


def run(c, variant, reps, timing=True):
    os.environ["HAWKES_SYM_VARIANT"] = str(variant)
    ctx = HawkesContext(c.N, c.D, algorithm="pairs")
    x = torch.from_numpy(c.x).cuda()
    ctx.set_times(torch.from_numpy(c.t).cuda())
    ctx.set_params(c.theta)
    g = torch.empty_like(x)
    ctx.set_locations(x)
    ctx.grad_locations(g)
    ctx.enable_timing(True)
    for _ in range(reps):
        ctx.set_locations(x)
        _, ell = ctx.grad_locations(g)
    kt = ctx.kernel_times()
    out = (ell, g.cpu().numpy(), kt["rate_ms"] / max(1, kt["rate_launches"]),
           kt["grad_ms"] / max(1, kt["grad_launches"]))
    ctx.close()
    return out


small = synth.unit_square(3000, config=41)
big = synth.config("C4", N=a.n)
ref = run(small, 40, 1)
for v in [int(s) for s in a.variants.split(",")]:
    e, g, _, _ = run(small, v, 1)
    ok = abs(e - ref[0]) <= 1e-12 * abs(ref[0]) and np.allclose(g, ref[1], rtol=1e-10, atol=1e-12)
    _, _, r_ms, g_ms = run(big, v, a.reps)
    print(f"variant {v}: rate {r_ms:7.3f} ms  grad {g_ms:7.3f} ms  total {r_ms + g_ms:7.3f} ms  match={ok}",
          flush=True)
