"""Host-side estimate of SURVEY NEXT-2's spatial culling (no GPU): the share of cross-chunk pairs
whose (row tile, column tile) bounding boxes and time ranges put both pair terms below the
exp's clamp (exponent < CULL_EXPONENT = -708 in the kernels' scaled domain), i.e. the tile
pairs a bounding-box test could skip, for a given chunk size and in-chunk ordering.

    python tools/cull_estimate.py [N] [chunk ...]

Orderings: "time" = the shipped layout (chunks and tiles in time order); "morton" = events
re-ordered by a Morton key inside each chunk (tiles spatially compact; chunks still time
ranges, so cross-chunk tile pairs keep the row-earlier direction).  The scaled-domain
constant lnc (log of the weight times 2^64, ~44) is taken as 44.4 for every term.
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

CULL = -708.0
LNC = 44.4
TILE = 128


def morton(q):
    q = q.astype(np.uint64)
    r = np.zeros(len(q), np.uint64)
    for b in range(16):
        r |= ((q[:, 0] >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
        r |= ((q[:, 1] >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b + 1)
    return r


def estimate(x, t, theta, chunk, mode):
    N = len(t)
    _, tx, tt, _, om, h = theta
    C = (N + chunk - 1) // chunk
    order = np.arange(N)
    if mode == "morton":
        lo = x.min(0)
        q = ((x - lo) / (x.max(0) - lo + 1e-9) * 65535).astype(np.int64)
        order = np.concatenate([a * chunk + np.argsort(morton(q[a * chunk:(a + 1) * chunk]), kind="stable")
                                for a in range(C)])
    xs, ts = x[order], t[order]
    nt = (N + TILE - 1) // TILE
    tl = np.array([xs[k * TILE:(k + 1) * TILE].min(0) for k in range(nt)])
    th = np.array([xs[k * TILE:(k + 1) * TILE].max(0) for k in range(nt)])
    tmin = np.array([ts[k * TILE:(k + 1) * TILE].min() for k in range(nt)])
    tmax = np.array([ts[k * TILE:(k + 1) * TILE].max() for k in range(nt)])
    cnt = np.array([min(TILE, N - k * TILE) for k in range(nt)], dtype=np.float64)
    chunk_of = np.arange(nt) * TILE // chunk
    tot = skip = 0.0
    for r in range(nt):
        cs = np.nonzero(chunk_of > chunk_of[r])[0]
        if len(cs) == 0:
            continue
        gap = np.maximum(0.0, np.maximum(tl[cs] - th[r], tl[r] - th[cs]))
        d2 = (gap ** 2).sum(1)
        dtmin = np.maximum(0.0, tmin[cs] - tmax[r])
        ab = -d2 / (2 * tx * tx) - dtmin ** 2 / (2 * tt * tt) + LNC
        a_s = -d2 / (2 * h * h) - om * dtmin + LNC
        w = cnt[r] * cnt[cs]
        tot += w.sum()
        skip += w[(ab < CULL) & (a_s < CULL)].sum()
    return skip / tot if tot else float("nan")


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    chunks = [int(a) for a in sys.argv[2:]] or [768, 6144, 25088]
    for name in ("C2", "C3", "C4"):
        c = synth.config(name, N=N)
        for ck in chunks:
            for mode in ("time", "morton"):
                f = estimate(c.x, c.t, c.theta, ck, mode)
                print(f"{name} N={N} chunk={ck:6d} {mode:6s}: cross-chunk pairs in skippable tile pairs {f:.3f}")


if __name__ == "__main__":
    main()
