"""The CPU oracle timed in full on this host (SURVEY.md §8(d) "Oracle timing beside it":
N in {500, 5k, 20k, 100k}, full ell + gradient evaluation of the C4 generator, all host
cores through OpenMP), with the CPU model and thread count.  One JSON line per N.

    python tools/oracle_timing.py [--sizes 500,5000,20000,100000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle  # noqa: E402
import synth  # noqa: E402
from bench import cpu_model  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="500,5000,20000,100000")
a = ap.parse_args()
for N in [int(s) for s in a.sizes.split(",")]:
    c = synth.config("C4", N=N)
    t0 = time.perf_counter()
    ell, lam, _ = oracle.loglik(c.x, c.t, c.theta)
    t1 = time.perf_counter()
    oracle.grad(c.x, c.t, c.theta, lam=lam)
    t2 = time.perf_counter()
    print(json.dumps({"N": N, "loglik_s": t1 - t0, "grad_s": t2 - t1, "eval_s": t2 - t0,
                      "pairs_per_s": N * (N - 1) / (t2 - t0), "evals_per_s": 1.0 / (t2 - t0),
                      "threads": oracle.num_threads(), "cpu": cpu_model(), "ell": ell}), flush=True)
