"""Minimax (Remez) fit of e^r - 1 = r (1 + c2 r + ... ) on |r| <= ln2/(2*TABLE) (+margin),
relative error, at 60 digits; prints the coefficients used by fexp in hawkes_kernels.cuh.

    python tools/fit_exp_poly.py [TABLE] [DEGREE]      (current kernels: 256 3)
"""
import sys

import mpmath as mp

mp.mp.dps = 60
TABLE = int(sys.argv[1]) if len(sys.argv) > 1 else 256
DEG = int(sys.argv[2]) if len(sys.argv) > 2 else 3
R = mp.log(2) / (2 * TABLE) * (1 + mp.mpf("1e-6"))


def fit(deg=3):
    # q(r) ~ (e^r - 1 - r)/r^2 = c2 + c3 r + c4 r^2 ; minimise max |(r + r^2 q(r)) - (e^r - 1)| / e^r
    n = deg  # unknowns c2..c4 plus E
    xs = [R * mp.cos(mp.pi * k / (n + 1)) for k in range(n + 2)]
    for _ in range(30):
        A = mp.matrix(n + 1, n + 1)
        b = mp.matrix(n + 1, 1)
        for i, x in enumerate(xs[: n + 1]):
            w = mp.e ** x
            for j in range(n):
                A[i, j] = x ** (2 + j) / w
            A[i, n] = (-1) ** i
            b[i] = (mp.e ** x - 1 - x) / w
        sol = mp.lu_solve(A, b)
        cs = [sol[j] for j in range(n)]
        err = lambda x: (x + sum(c * x ** (2 + j) for j, c in enumerate(cs)) - (mp.e ** x - 1)) / mp.e ** x
        # new extrema by dense sampling
        grid = [R * (2 * mp.mpf(k) / 4000 - 1) for k in range(4001)]
        vals = [err(x) for x in grid]
        ext = [grid[0]]
        for k in range(1, 4000):
            if (vals[k] - vals[k - 1]) * (vals[k + 1] - vals[k]) <= 0:
                ext.append(grid[k])
        ext.append(grid[-1])
        if len(ext) >= n + 1:
            xs = ext[: n + 1] if len(ext) == n + 1 else sorted(ext, key=lambda x: -abs(err(x)))[: n + 1]
            xs.sort()
    maxerr = max(abs(err(R * (2 * mp.mpf(k) / 20000 - 1))) for k in range(20001))
    return cs, maxerr


cs, e = fit(DEG - 1)
print("max rel err", mp.nstr(e, 5))
for j, c in enumerate(cs):
    print(f"c{j+2} = {mp.nstr(c, 20)}  double: {float(c).hex()}  {float(c)!r}")
