"""Driver for ncu: BMDS density + gradient at the flu shape (N = 4733, D = 6), W warm-up calls
then one more.

    python tools/prof_bmds.py [--n 4733] [--warmup 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4733)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
c, Y, s = synth.flu_shaped(a.n, 6)
ctx = HawkesContext(a.n, 6)
ctx.set_locations(torch.from_numpy(c.x).cuda())
ctx.set_bmds(torch.from_numpy(Y).cuda(), s)
for _ in range(a.warmup + 1):
    ctx.bmds_logdensity()
torch.cuda.synchronize()
