"""Plain-error report of the CUDA path against the oracle (SURVEY.md §8(c) rule 16: "also
report plain relative error (max, p99) and the kappa of the worst component").

For each config and precision, per gradient component (n, d):
  plain   |g - g*| / |g*|                      (north_star's literal "relative error")
  kappa   S_nd / |g*_nd|                       (condition number of the cancelling sum)
  ulpS    |g - g*| / (u S_nd), u = 2^-53        (error in units of the sum's rounding scale)
  gate    |g - g*| / (tol max(|g*|, floor S))   (the parity gate of tests/gpu_helpers.py)
and the ell relative error.  Components whose plain error exceeds tol are listed by kappa:
a u-accurate evaluation (any summation order, the oracle's included) has plain error up to
~kappa * sqrt(N) * u, so such components are expected only where kappa is large.

    python tools/parity_report.py [C1:500 C4:20000 ...] [--out profiles/r02_plain_error.jsonl]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from tests.gpu_helpers import TOL, gpu_eval, oracle_eval  # noqa: E402

U = 2.0 ** -53


def report(name, N, prec, c, ell_r, g_r, S):
    ell, g, _ = gpu_eval(c.x, c.t, c.theta, precision=prec, with_rates=False)
    tol, floor = TOL[prec]
    err = np.abs(g - g_r)
    ag = np.abs(g_r)
    with np.errstate(divide="ignore", invalid="ignore"):
        plain = np.where(ag > 0, err / ag, np.where(err > 0, np.inf, 0.0))
        kappa = np.where(ag > 0, S / ag, np.inf)
        ulps = np.where(S > 0, err / (U * S), 0.0)
    gate = err / np.maximum(tol * np.maximum(ag, floor * S), 1e-300)
    flat = plain.ravel()
    iw = int(np.argmax(flat))
    over = plain > tol
    rec = {
        "config": name, "N": N, "precision": prec,
        "ell_rel": abs(ell - ell_r) / abs(ell_r),
        "plain_max": float(flat[iw]), "plain_p99": float(np.quantile(flat, 0.99)),
        "plain_p50": float(np.quantile(flat, 0.5)),
        "kappa_of_worst": float(kappa.ravel()[iw]),
        "kappa_max": float(np.max(kappa[np.isfinite(kappa)])) if np.isfinite(kappa).any() else None,
        "kappa_p99": float(np.quantile(kappa[np.isfinite(kappa)], 0.99)),
        "n_components": int(g.size),
        "n_plain_over_tol": int(over.sum()),
        "min_kappa_over_tol": float(kappa[over].min()) if over.any() else None,
        "ulpS_max": float(np.max(ulps)), "ulpS_p99": float(np.quantile(ulps, 0.99)),
        "gate_max": float(np.max(gate)),
    }
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sizes", nargs="*")
    ap.add_argument("--out", default=None)
    ap.add_argument("--precisions", default="fp64,fp32")
    a = ap.parse_args()
    sizes = [(s.split(":")[0], int(s.split(":")[1])) for s in a.sizes] or \
        [("C1", 500), ("C1", 3000), ("C2", 5000), ("C3", 6000), ("C3", 20000), ("C4", 20000)]
    out = open(a.out, "a") if a.out else None
    for name, N in sizes:
        c = synth.config(name, N)
        ell_r, _, _, g_r, S = oracle_eval(c.x, c.t, c.theta)
        for prec in a.precisions.split(","):
            rec = report(name, N, prec, c, ell_r, g_r, S)
            line = json.dumps(rec)
            print(line, flush=True)
            if out:
                out.write(line + "\n")
                out.flush()


if __name__ == "__main__":
    main()
