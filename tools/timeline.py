"""Timeline of small-N calls (diagnostics; CUPTI activity through torch.profiler, so the
absolute numbers carry the tracer's overhead and are never bench values): per call of
set_locations + grad_locations (host sync each call), every device activity's start and end
relative to the call's first one, averaged over the calls: kernel durations, the gaps between
consecutive activities, and the idle gap from one call's last activity to the next call's first.

    python tools/timeline.py [--sizes 500,5000] [--calls 50] [--precision fp64]
"""
import argparse
import json
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import synth  # noqa: E402
from paper_2010_02994_b200 import HawkesContext  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="500,5000")
ap.add_argument("--calls", type=int, default=50)
ap.add_argument("--precision", default="fp64")
ap.add_argument("--config", default="C4", help="catalog shape (synth.config name)")
ap.add_argument("--at", action="store_true", help="hawkes_grad_at calls instead of set_locations + grad_locations")
a = ap.parse_args()


def short(name):
    name = name.split("(")[0]
    return name.replace("void ", "").replace("hk::", "")[:48]


for N in [int(s) for s in a.sizes.split(",")]:
    c = synth.unit_square(N, config=4) if a.config == "C4" else synth.config(a.config, N=N)
    ctx = HawkesContext(N, 2, precision=a.precision)
    x = torch.from_numpy(c.x).cuda()
    ctx.set_times(torch.from_numpy(c.t).cuda())
    ctx.set_params(c.theta)
    g = torch.empty_like(x)
    def call():
        if a.at:
            ctx.grad_at(x, g)
        else:
            ctx.set_locations(x)
            ctx.grad_locations(g)
    for _ in range(10):
        call()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(a.calls):
            call()
        torch.cuda.synchronize()
    ev = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            ev.append((e.time_range.start, e.time_range.end, short(e.name)))
    ev.sort()
    # split into calls: an activity whose name is the first one's starts a call
    first = ev[0][2]
    calls, cur = [], []
    for s, t, n in ev:
        if n == first and cur:
            calls.append(cur)
            cur = []
        cur.append((s, t, n))
    calls.append(cur)
    calls = calls[1:-1]   # drop the partial first / last
    dur, gap, order = defaultdict(list), defaultdict(list), []
    spans, idle = [], []
    for k, cl in enumerate(calls):
        t0 = cl[0][0]
        for q, (s, t, n) in enumerate(cl):
            key = f"{q}:{n}"
            if k == 0:
                order.append(key)
            dur[key].append(t - s)
            if q:
                gap[key].append(s - cl[q - 1][1])
        spans.append(cl[-1][1] - t0)
        if k + 1 < len(calls):
            idle.append(calls[k + 1][0][0] - cl[-1][1])
    med = lambda v: sorted(v)[len(v) // 2] if v else None  # noqa: E731
    out = {"N": N, "config": a.config, "grad_at": a.at, "precision": a.precision, "calls": len(calls), "device_span_us": med(spans),
           "host_idle_between_calls_us": med(idle), "activities": []}
    for key in order:
        out["activities"].append({"name": key, "dur_us": med(dur[key]), "gap_before_us": med(gap[key])})
    print(json.dumps(out), flush=True)
    ctx.close()
