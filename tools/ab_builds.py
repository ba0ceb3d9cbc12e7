"""A/B builds of the library with compile-time variants (-D flags), into tools/alt_build/
(git-ignored; travels to the GPU box with the snapshot), and a timing run of each.

    python tools/ab_builds.py build NAME=FLAG[,FLAG] ...     # on the CPU host, in parallel
    python tools/ab_builds.py time NAME ... [--n 100000]      # on the GPU: per-pass kernel ms

`time` runs bench-like evaluations (C4, D = 2, fp64) with HAWKES_LIB_AB pointing at each build
(the default build is "base") and prints one JSON line per build.
"""
import json
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALT = os.path.join(ROOT, "tools", "alt_build")


def do_build(spec):
    name, _, flags = spec.partition("=")
    sys.path.insert(0, ROOT)
    from paper_2010_02994_b200 import build as b
    out = os.path.join(ALT, f"lib_{name}.so")
    b.build(force=True, defines=[f for f in flags.split(",") if f], out=out)
    return name, out


def time_one(name, n, precision, reps):
    """name = BUILD[@ENV=VALUE[@ENV=VALUE]]: a build (base = the in-tree library) and runtime
    environment switches (e.g. base@HAWKES_SYM_V=6)."""
    build, *envs = name.split("@")
    lib = "" if build == "base" else os.path.join(ALT, f"lib_{build}.so")
    code = f"""
import json, sys, torch
sys.path.insert(0, {ROOT!r})
import synth
from paper_2010_02994_b200 import HawkesContext
c = synth.config("C4", N={n})
ctx = HawkesContext(c.N, 2, precision={precision!r})
x = torch.from_numpy(c.x).cuda(); ctx.set_times(torch.from_numpy(c.t).cuda()); ctx.set_params(c.theta)
g = torch.empty_like(x)
for _ in range(3):
    ctx.set_locations(x); ctx.grad_locations(g)
ctx.enable_timing(True)
for _ in range({reps}):
    ctx.set_locations(x); ctx.grad_locations(g)
kt = ctx.kernel_times()
print(json.dumps({{"rate_ms": kt["rate_ms"] / kt["rate_launches"], "grad_ms": kt["grad_ms"] / kt["grad_launches"]}}))
"""
    env = dict(os.environ)
    for e in envs:
        k, _, v = e.partition("=")
        env[k] = v
    if lib:
        env["HAWKES_LIB_AB"] = lib
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    if r.returncode:
        return {"build": name, "error": r.stderr[-400:]}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    d.update(build=name, N=n, precision=precision)
    return d


def main():
    if sys.argv[1] == "build":
        os.makedirs(ALT, exist_ok=True)
        with ThreadPoolExecutor(max_workers=4) as ex:
            for name, out in ex.map(do_build, sys.argv[2:]):
                print(name, out, flush=True)
    else:
        args = sys.argv[2:]
        n = 100000
        prec = "fp64"
        reps = 10
        if "--n" in args:
            i = args.index("--n")
            n = int(args[i + 1])
            del args[i:i + 2]
        if "--fp32" in args:
            args.remove("--fp32")
            prec = "fp32"
        for rnd in range(2):          # two rounds, interleaved, to see box drift
            for name in args:
                print(json.dumps({**time_one(name, n, prec, reps), "round": rnd}), flush=True)


if __name__ == "__main__":
    main()
