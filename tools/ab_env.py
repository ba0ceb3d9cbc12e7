"""Per-pass kernel times (ms per launch) of the current build at C4 N (default 100k), for A/B
runs that select kernel variants with environment variables (HAWKES_SYM_V, HAWKES_SYM32_SOA).

    HAWKES_SYM32_SOA=0 python tools/ab_env.py [N] [fp64|fp32]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
prec = sys.argv[2] if len(sys.argv) > 2 else "fp64"
c = synth.config("C4", N=N)
ctx = HawkesContext(N, 2, precision=prec)
x = torch.from_numpy(c.x).cuda()
ctx.set_times(torch.from_numpy(c.t).cuda())
ctx.set_params(c.theta)
g = torch.empty_like(x)
ctx.set_locations(x)
ctx.grad_locations(g)
ctx.enable_timing(True)
for _ in range(5):
    ctx.set_locations(x)
    ctx.grad_locations(g)
kt = ctx.kernel_times()
env = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("HAWKES_"))
print(f"{prec} N={N} {env or 'default'}: rate {kt['rate_ms'] / kt['rate_launches']:.3f} "
      f"grad {kt['grad_ms'] / kt['grad_launches']:.3f}")
