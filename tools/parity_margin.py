"""Worst gradient error / tolerance bound and relative ell
error of the CUDA path against the oracle, per config: how much of the parity budget the
arithmetic uses.

    python tools/parity_margin.py [C1:20000 ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from tests.gpu_helpers import assert_parity, gpu_eval, oracle_eval  # noqa: E402

SIZES = [tuple((a.split(":")[0], int(a.split(":")[1]))) for a in sys.argv[1:]] or [("C1", 500), ("C1", 3000), ("C2", 5000), ("C3", 6000)]
for name, N in SIZES:
    c = synth.config(name, N)
    ell_r, _, _, g_r, S = oracle_eval(c.x, c.t, c.theta)
    for prec in ("fp64", "fp32"):
        ell, g, _ = gpu_eval(c.x, c.t, c.theta, precision=prec, with_rates=False)
        worst = assert_parity(ell, g, ell_r, g_r, S, precision=prec, what=name)
        print(f"{name} N={N} {prec}: worst err/bound {worst:.3g}  ell rel err {abs(ell - ell_r) / abs(ell_r):.3g}",
              flush=True)
