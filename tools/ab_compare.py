"""A/B timing of two builds of the library on the same box: prints the PAIRS pass times of
the package found first on sys.path (PYTHONPATH=tools/old_build selects an old build)."""
import os
import sys
import torch
sys.path.append(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2010_02994_b200 as P  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
c = synth.config("C4", N=N)
ctx = HawkesContext(N, 2)
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
print(P.__file__, f"rate {kt['rate_ms']/kt['rate_launches']:.3f} grad {kt['grad_ms']/kt['grad_launches']:.3f}")
