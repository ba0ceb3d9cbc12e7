"""Overhead of the sharded (multi-GPU) code path measured on one GPU: a one-rank NCCL
communicator runs the per-rank slot sums, the ncclAllReduce calls and the finalize from the
exchanged sums; the plain context runs neither.  ms per ell + gradient evaluation (CUDA
events around the call, C4 catalog).

    python tools/exchange_overhead.py [N]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext, nccl_unique_id  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
c = synth.config("C4", N=N)
for label, nccl in (("plain (graphs)", False), ("one-rank NCCL (sharded path, no graphs)", True)):
    for alg in ("pairs", "rows"):
        kw = {"nccl_id": nccl_unique_id()} if nccl else {}   # a fresh id per communicator
        ctx = HawkesContext(N, 2, algorithm=alg, **kw)
        x = torch.from_numpy(c.x).cuda()
        ctx.set_times(torch.from_numpy(c.t).cuda())
        ctx.set_params(c.theta)
        g = torch.empty_like(x)
        for _ in range(3):
            ctx.set_locations(x)
            ctx.grad_locations(g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        for _ in range(5):
            ctx.set_locations(x)
            ctx.grad_locations(g)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        print(f"N={N} {alg:5s} {label}: {e0.elapsed_time(e1) / 5:.3f} ms per evaluation", flush=True)
        ctx.close()
