"""Per-call host overhead at small N: host wall time of set_locations (no sync) and of
grad_locations (one sync), against the GPU time of the same evaluation (CUDA events), and the
same calls through the raw ctypes entry points (no Python wrapper).

    python tools/call_overhead.py [--n 500] [--reps 2000]
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=500)
ap.add_argument("--reps", type=int, default=2000)
a = ap.parse_args()
c = synth.unit_square(a.n, config=4)
ctx = HawkesContext(c.N, 2)
x = torch.from_numpy(c.x).cuda()
g = torch.empty_like(x)
ctx.set_times(torch.from_numpy(c.t).cuda())
ctx.set_params(c.theta)
for _ in range(20):
    ctx.set_locations(x)
    ctx.grad_locations(g)
torch.cuda.synchronize()

ts, tg = 0.0, 0.0
for _ in range(a.reps):
    t0 = time.perf_counter()
    ctx.set_locations(x)
    t1 = time.perf_counter()
    ctx.grad_locations(g)
    t2 = time.perf_counter()
    ts += t1 - t0
    tg += t2 - t1
lib = _lib.load()
h = ctx._h
xp, gp = x.data_ptr(), g.data_ptr()
ll = ctypes.c_double()
t0 = time.perf_counter()
for _ in range(a.reps):
    lib.hawkes_set_locations(h, xp, 1)
    lib.hawkes_grad_locations(h, gp, 1, ctypes.byref(ll))
t_raw = (time.perf_counter() - t0) / a.reps
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ctx.stream)
for _ in range(200):
    ctx.set_locations(x)
    ctx.grad_locations(g)
e1.record(ctx.stream)
torch.cuda.synchronize()
print(json.dumps({"N": a.n, "set_locations_us": 1e6 * ts / a.reps, "grad_locations_us": 1e6 * tg / a.reps,
                  "raw_ctypes_pair_us": 1e6 * t_raw, "stream_span_per_call_us": e0.elapsed_time(e1) * 1e3 / 200}))
