"""Small driver for ncu / compute-sanitizer: W warm-up evaluations then K timed-free
evaluations of ell + gradient on the C4 catalog (default N = 100k, fp64).

    python tools/prof_step.py [--n 100000] [--warmup 3] [--evals 1] [--precision fp64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--evals", type=int, default=1)
ap.add_argument("--precision", default="fp64")
ap.add_argument("--config", default="C4")
ap.add_argument("--algorithm", default="auto")
ap.add_argument("--leapfrog", type=int, default=0)
a = ap.parse_args()

c = synth.config(a.config, N=a.n)
ctx = HawkesContext(c.N, c.D, precision=a.precision, algorithm=a.algorithm)
x = torch.from_numpy(c.x).cuda()
ctx.set_times(torch.from_numpy(c.t).cuda())
ctx.set_params(c.theta)
g = torch.empty_like(x)
for _ in range(a.warmup + a.evals):
    ctx.set_locations(x)
    _, ell = ctx.grad_locations(g)
if a.leapfrog:
    p = torch.ones_like(x)
    ctx.leapfrog(x.clone(), p, 1e-5, a.leapfrog, box_lo=x - 0.01, box_hi=x + 0.01)
torch.cuda.synchronize()
print(f"N={c.N} ell={ell!r} |g|max={g.abs().max().item():.6g}")
ctx.close()
