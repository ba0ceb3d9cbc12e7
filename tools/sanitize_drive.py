"""Every public entry point once at small N -- PAIRS and ROWS, fp64 and fp32, D = 1, 2, 3, 6,
ragged tiles, an emulated 2-rank world, leapfrog, the HMC transition, block moves, the MH
sweep (the cooperative kernel and the launch path), BMDS and the joint potential -- as one
process, for tools that wrap a whole run (compute-sanitizer where available; it is closed
on this round's GPU pool, where tools/nan_poison.py and the parity fuzzers stand in).

    python tools/sanitize_drive.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402


def hawkes(c, **kw):
    ctx = HawkesContext(c.N, c.D, **kw)
    ctx.set_times(torch.from_numpy(c.t).cuda())
    ctx.set_locations(torch.from_numpy(c.x).cuda())
    ctx.set_params(c.theta)
    return ctx


def evals(ctx, c, n=3):
    g = torch.empty((c.N, c.D), dtype=torch.float64, device="cuda")
    for _ in range(n):   # the second and later calls replay the captured graphs
        ctx.set_locations(torch.from_numpy(c.x).cuda())
        ctx.loglik()
        ctx.grad_locations(g)
    return g


def main():
    for D in (1, 2, 3, 6):
        c = synth.unit_square(300 + 37 * D, config=1, D=D)
        for algo in ("pairs", "rows"):
            for prec in ("fp64", "fp32"):
                ctx = hawkes(c, algorithm=algo, precision=prec)
                evals(ctx, c)
                ctx.get_rates()
                ctx.close()
    c = synth.config("C1", N=517)
    ctx = hawkes(c, emulate_world=2)
    evals(ctx, c)
    ctx.close()
    # leapfrog + HMC transition (box reflection, diagonal mass)
    ctx = hawkes(c)
    x = torch.from_numpy(c.x).cuda()
    p = torch.ones_like(x)
    ctx.leapfrog(x.clone(), p, 1e-4, 4, box_lo=x - 0.05, box_hi=x + 0.05)
    minv = torch.full_like(x, 0.5)
    for it in range(3):
        ctx.hmc_step(5, it, 1e-4, 4, inv_mass=minv, box_lo=x - 0.05, box_hi=x + 0.05)
    ctx.close()
    # block moves and MH sweeps on the DC / Alaska shapes
    for name in ("C2", "C3"):
        c = synth.config(name, N=700)
        ctx = hawkes(c)
        ctx.set_regions(c.region, c.centre, c.size)
        ctx.loglik()
        idx = np.array([3, 77, 400], dtype=np.int32)
        ctx.propose_move(idx, torch.from_numpy(c.x[idx] + 1.0).cuda())
        ctx.accept_move()
        rng = np.random.default_rng(1)
        for k in (1, 8, 12):   # k <= 8: cooperative sweep kernel; 12: graph launches
            blocks = np.stack([rng.choice(c.N, size=k, replace=False) for _ in range(6)]).astype(np.int32)
            ctx.mh_sweep(blocks, 0.7, 3, k)
        ctx.get_locations()
        ctx.close()
    # BMDS and the joint potential
    c, Y, s = synth.flu_shaped(300, 6)
    ctx = hawkes(c)
    ctx.set_bmds(torch.from_numpy(Y).cuda(), s)
    ctx.bmds_logdensity()
    ctx.set_potential(hawkes=True, bmds=True)
    x = torch.from_numpy(c.x).cuda()
    ctx.leapfrog(x.clone(), torch.ones_like(x), 1e-4, 3)
    ctx.close()
    torch.cuda.synchronize()
    print("sanitize_drive: ok")


if __name__ == "__main__":
    main()
