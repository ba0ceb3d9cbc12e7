"""Ground truth for one fuzz case (tools/fuzz_parity.py) where the oracle and the GPU disagree:
lambda_n and the App. A gradient evaluated with 30-digit mpmath arithmetic (every
pair term separately, no scaling), then the oracle's and (optionally) the GPU's results
measured against it under the parity tolerance rule.

    python tools/mp_check_case.py --seed 41 --case 602 [--nmax 3000] [--gpu gpu.npz]

The GPU arrays come from a separate run (keys <label>_g, <label>_lam), e.g. gpu_eval on a B200.
O(N^2) mpmath work: minutes for N ~ 1000.
"""
import argparse
import importlib.util
import json
import os
import sys

import mpmath as mp
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def fuzz_case(seed, case, nmax):
    spec = importlib.util.spec_from_file_location("fz", os.path.join(ROOT, "tools", "fuzz_parity.py"))
    fz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(fz)
    rng = np.random.default_rng(seed)
    for _ in range(case + 1):
        out = fz.make_case(rng, nmax)
    return out


def mp_truth(x, t, th, dps=30):
    """lambda_n and g_n = sum_m c_nm (x_m - x_n) (App. A) at dps digits."""
    mp.mp.dps = dps
    N, D = x.shape
    mu0, tx, tt, the, om, h = [mp.mpf(float(v)) for v in th]
    two_pi = 2 * mp.pi
    cb = mu0 / (tx ** D * tt) / two_pi ** (mp.mpf(D) / 2) / mp.sqrt(two_pi)
    cs = the * om / h ** D / two_pi ** (mp.mpf(D) / 2)
    X = [[mp.mpf(float(v)) for v in r] for r in x]
    T = [mp.mpf(float(v)) for v in t]
    mu, xi, lam = {}, {}, []
    for n in range(N):
        s = mp.mpf(0)
        for m in range(N):
            if m == n:
                continue
            d2 = sum((X[n][k] - X[m][k]) ** 2 for k in range(D))
            if t[n] != t[m]:
                v = cb * mp.exp(-d2 / (2 * tx * tx) - (T[n] - T[m]) ** 2 / (2 * tt * tt))
                mu[(n, m)] = v
                s += v
            if t[m] < t[n]:
                v = cs * mp.exp(-om * (T[n] - T[m]) - d2 / (2 * h * h))
                xi[(n, m)] = v
                s += v
        lam.append(s)
    g = np.zeros((N, D))
    for n in range(N):
        for k in range(D):
            acc = mp.mpf(0)
            for m in range(N):
                if m == n:
                    continue
                c = ((mu.get((n, m), 0) / lam[n] + mu.get((m, n), 0) / lam[m]) / (tx * tx)
                     + (xi.get((n, m), 0) / lam[n] + xi.get((m, n), 0) / lam[m]) / (h * h))
                acc += c * (X[m][k] - X[n][k])
            g[n, k] = float(acc)
    return np.array([float(v) for v in lam]), g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, required=True)
    ap.add_argument("--case", type=int, required=True)
    ap.add_argument("--nmax", type=int, default=3000)
    ap.add_argument("--gpu", default=None)
    a = ap.parse_args()
    N, D, x, t, th, prec, alg, W = fuzz_case(a.seed, a.case, a.nmax)
    ell_o, lam_o, _ = oracle.loglik(x, t, th)
    g_o, S = oracle.grad(x, t, th, lam=lam_o)
    lam_m, g_m = mp_truth(x, t, th)
    bound = 1e-9 * np.maximum(np.abs(g_m), 1e-3 * S)
    res = {"seed": a.seed, "case": a.case, "N": N, "D": D, "theta": list(th),
           "lambda_min": float(lam_m.min()), "lambda_max": float(lam_m.max()),
           "oracle": {"grad_ratio": float(np.max(np.abs(g_o - g_m) / bound)),
                      "lambda_rel": float(np.max(np.abs(lam_o - lam_m) / lam_m))}}
    if a.gpu:
        G = np.load(a.gpu)
        for k in sorted(G.files):
            if k.endswith("_g"):
                lab = k[:-2]
                res[lab] = {"grad_ratio": float(np.max(np.abs(G[k] - g_m) / bound)),
                            "lambda_rel": float(np.max(np.abs(G[lab + "_lam"] - lam_m) / lam_m))}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
