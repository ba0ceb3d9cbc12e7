#!/usr/bin/env python
"""Benchmark of the Hawkes ell + location-gradient hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--n 100000]

One *step* = one evaluation of ell and d ell/dx at the current locations (SURVEY.md §8(a)
S0-S6: locations staged into the event records, rate pass, finalize, exchange, gradient
pass, finalize, exchange), on BASELINE configs[3] = C4 at N = 100k, D = 2, fp64.  With
N > 1 GPUs (torchrun) the rows are sharded (strong scaling: the whole job evaluates the
same N = 100k catalog).  Rank 0 prints one JSON line.

--impl reference times the CPU oracle (oracle/, the reference arm for this tier) on the
host cores: each step is a full oracle evaluation on a bounded sample of the workload
(the same generator at a smaller N), scaled to evals/s at N = 100k by the pair count.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "loglik+location-gradient evals/s and pair-interactions/s at N=100k, 1-8 B200"
# Roofline basis (DESIGN.md §4 "Roofline"), per ORDERED pair, D = 2, (rate pass, gradient pass):
#   F_ALG   frozen algorithmic FP64 work of the unordered-pair method with a u-accurate table
#           exp costed at 7 FP64 operations (range reduction 3, degree-3 polynomial 3,
#           reconstruction 1), per unordered pair: rate pass 10 (dx, dy, r^2 (2), dt, background
#           exponent 3, self-excitation exponent 2) + 14 (two exps) + 3 (row mu, column mu, column
#           xi sums) = 27; gradient pass 10 + 14 + 3 (c = rho_i mu + rho_j (mu + xi)) + 4 (two
#           gradient updates) = 31.  It does not move when the shipped instruction count moves,
#           so removing instructions raises frac (the headline).
#   F_PIPE  FP64-pipe instructions per ordered pair of the shipped sym_kernel's unmasked hot loop
#           (tools/falg_count.py --shipped): pipe utilisation, reported beside it.  The gradient
#           pass's (and, D <= 2, the rate pass's) 8 I2F.F64 per step run on the conversion pipe and are not counted.
#   F_SURVEY SURVEY.md §8(d)'s frozen ordered-pair F_alg (libdevice exp, ordered pairs): context.
F_ALG = (13.5, 15.5)
F_PIPE = (11.0, 14.5)   # rate pass: product-form exps (each sum one fma), I2F k, rebased times: 22 per unordered pair
# fp32 variant: FMA-pipe instructions per ordered pair of sym_kernel_f32's hot loop (packed
# FFMA2 / FADD2 / FMUL2 = 1 per lane; SASS); its peak is one packed warp-instruction per 2
# cycles per SMSP = 64 lanes/clk/SM.  MUFU: one ex2 per ordered pair per pass (two per unordered
# pair), 16 / clk / SM.
F_IMPL32 = (5.0, 6.0)
MUFU_PER_SM = 16
F_SURVEY = (34.5, 49.0)
FP64_LANES_PER_SM = 64


def _ncu_traffic(kernel):
    """dram__bytes_read + dram__bytes_write per launch of `kernel` from the committed
    ncu --set full capture (profiles/r02_ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    try:
        with open(path) as f:
            caps = json.load(f)
    except (OSError, ValueError):
        return None
    if kernel in caps:
        return caps[kernel]["bytes"]
    # the capture names every template argument; bench names the leading ones
    # (GEN, PIECE, NW) = (0, 0, 4): the time-walk whole-item 4-warp kernel
    stem = kernel[:-1] + ","
    for k, v in caps.items():
        if k.startswith(stem):
            rest = [a.strip() for a in k[len(stem):-1].split(",")]
            if rest == ["0", "0", "4"][:len(rest)]:
                return v["bytes"]
    return None


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


def _oracle_eval(c):
    import oracle
    ll, lam, _ = oracle.loglik(c.x, c.t, c.theta)
    oracle.grad(c.x, c.t, c.theta, lam=lam)


def _oracle_rate():
    """Ordered pairs per second of one oracle ell + gradient evaluation on this host
    (warm-up at N=500, then a probe at N=3000)."""
    import synth
    _oracle_eval(synth.unit_square(500, config=4))
    c = synth.unit_square(3000, config=4)
    t0 = time.perf_counter()
    _oracle_eval(c)
    return 3000 * 2999 / (time.perf_counter() - t0)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(target_s: float = 12.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload:
    full ell + gradient evaluation of the C4 generator at a smaller N chosen for ~10-15 s."""
    import oracle
    import synth
    Ns = int(min(100_000, max(1000, (target_s * _oracle_rate()) ** 0.5)))
    c = synth.unit_square(Ns, config=4)
    t0 = time.perf_counter()
    _oracle_eval(c)
    dt = time.perf_counter() - t0
    pairs = Ns * (Ns - 1)
    return {"pairs_per_s": pairs / dt, "Ns": Ns, "seconds": dt, "cores": oracle.num_threads(),
            "cpu": cpu_model()}


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    import numpy as np
    import oracle
    import synth
    N = args.n
    # each step: a full oracle evaluation sized for ~4 s on this host
    Ns = int(min(N, max(1000, (4.0 * _oracle_rate()) ** 0.5)))
    c = synth.unit_square(Ns, config=4)

    def step():
        _oracle_eval(c)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    pairs_per_s = Ns * (Ns - 1) / dt
    evals_per_s = pairs_per_s / (N * (N - 1))
    cores = oracle.num_threads()
    sample = (f"full oracle ell+gradient of the C4 generator at N={Ns} per step "
              f"(bounded sample of the N={N} workload), scaled by N(N-1) ordered pairs")
    line = {
        "impl": "reference", "metric": METRIC, "value": evals_per_s, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # a step is the bounded sample (the time the driver's clock sees); the full N-event
        # evaluation it stands for would take ms_per_full_eval (N(N-1) scaling)
        "ms_per_step": dt * 1e3,
        "ms_per_full_eval": dt * 1e3 * (N * (N - 1)) / (Ns * (Ns - 1)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "pairs_per_s": pairs_per_s,
        "config": {"workload": f"C4 unit-square Hawkes catalog N={N} D=2 (BASELINE configs[3])",
                   "N": N, "D": 2, "precision": "fp64", "sample_N": Ns},
        "cpu_baseline": {"value": evals_per_s, "unit": "evals/s", "cores": cores, "kind": "oracle",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": evals_per_s, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import synth
    from paper_2010_02994_b200 import HawkesContext, diag_fp64_peak
    from paper_2010_02994_b200.sharding import init_distributed_context

    N, D = args.n, 2
    c = synth.config("C4", N=N)
    if world > 1:
        ctx = init_distributed_context(N, D, precision=args.precision, algorithm=args.algorithm)
    else:
        ctx = HawkesContext(N, D, device=local, precision=args.precision, algorithm=args.algorithm)
    stream = ctx.stream
    x_dev = torch.from_numpy(c.x).to(dev)
    t_dev = torch.from_numpy(c.t).to(dev)
    ctx.set_times(t_dev)
    ctx.set_params(c.theta)
    g_dev = torch.empty((N, D), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    def step():
        ctx.set_locations(x_dev)             # stage this step's locations (invalidates caches)
        _, ell = ctx.grad_locations(g_dev)   # rate pass + gradient pass (+ exchanges)
        return ell

    for _ in range(max(3, args.warmup)):
        ell = step()
    torch.cuda.synchronize()

    # ---- device-timed region: K steps, L2 flushed before each (flush not timed)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler = ClockSampler(local)
    ctx.enable_timing(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.fill_(k)
            ev[k][0].record(stream)
            ell = step()
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    kt = ctx.kernel_times()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    tmax = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_total = float(tmax.item())
    ms_per_step = ms_total / args.steps
    evals_per_s = args.steps / (ms_total * 1e-3)
    pairs = N * (N - 1)

    # ---- end-to-end through the C ABI with pinned HOST buffers (copies inside the region)
    ctx.enable_timing(False)
    x_host = torch.from_numpy(c.x.copy()).pin_memory()
    g_host = torch.empty((N, D), dtype=torch.float64).pin_memory()
    e2e_steps = max(3, args.steps // 2)
    for _ in range(2):
        ctx.set_locations(x_host)
        ctx.grad_locations(g_host)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        ctx.set_locations(x_host)
        _, ell_e2e = ctx.grad_locations(g_host)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_val = e2e_steps / (float(e2e_ms.item()) * 1e-3)

    # ---- loglik-only evaluations (S0-S4: rate pass, finalize, exchange),
    # same staging and L2 flush as the timed step
    with torch.cuda.stream(stream):
        for _ in range(3):
            ctx.set_locations(x_dev)
            ctx.loglik()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    lev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.fill_(k)
            lev[k][0].record(stream)
            ctx.set_locations(x_dev)
            ctx.loglik()
            lev[k][1].record(stream)
    torch.cuda.synchronize()
    lms = torch.tensor([sum(a.elapsed_time(b) for a, b in lev)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(lms, op=dist.ReduceOp.MAX)
    loglik_only = {"evals_per_s": args.steps / (float(lms.item()) * 1e-3),
                   "ms_per_eval": float(lms.item()) / args.steps,
                   "note": "ell alone (rate pass + finalize), same staging and L2 flush"}

    # ---- C5 (BASELINE configs[4]): full HMC transitions over X at N = 50k through
    # hawkes_hmc_step -- on-device Philox momenta, a 20-step leapfrog, the Metropolis decision;
    # an accepted transition leaves the end-point gradient cached for the next one
    hmc = None
    if not args.no_hmc:
        c5 = synth.config("C5")
        if world > 1:
            hctx = init_distributed_context(c5.N, D, precision=args.precision, algorithm=args.algorithm)
        else:
            hctx = HawkesContext(c5.N, D, device=local, precision=args.precision,
                                 algorithm=args.algorithm)
        hctx.set_times(torch.from_numpy(c5.t).to(dev))
        hctx.set_params(c5.theta)
        hctx.set_locations(torch.from_numpy(c5.x).to(dev))
        hstep, hL, hK = 1e-4, 20, 5
        hctx.hmc_step(2010, 0, hstep, 2)            # warm-up (graph capture)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(hctx.stream)
        accs, las = [], []
        for it in range(1, hK + 1):
            acc, la = hctx.hmc_step(2010, it, hstep, hL)
            accs.append(acc)
            las.append(la)
        h1.record(hctx.stream)
        torch.cuda.synchronize()
        hms = torch.tensor([h0.elapsed_time(h1) / hK], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(hms, op=dist.ReduceOp.MAX)
        hmc = {"config": f"C5 N=50000 D=2, {hK} HMC transitions of {hL} leapfrog steps, step {hstep}, "
                         "identity mass, Philox momenta + Metropolis on the device",
               "ms_per_transition": float(hms.item()), "transitions_per_s": 1e3 / float(hms.item()),
               "grad_evals_per_transition": hL,   # (hL + 1 after a rejected transition)
               "grad_evals_per_s": hL * 1e3 / float(hms.item()),
               "acceptance": sum(accs) / hK, "log_alpha": las}
        hctx.close()

    # ---- the paper's location sampler for the coarsened DC / Alaska catalogs:
    # on-device block-MH sweeps (k = 1 event per block) at the catalogs' sizes
    mh = None
    if not args.no_hmc:
        mh = {}
        for name, nev, rkind in (("C2", 3982, "square"), ("C3", 2925, "disc")):
            cm = synth.config(name, nev)
            if world > 1:
                mctx = init_distributed_context(cm.N, D, precision=args.precision, algorithm=args.algorithm)
            else:
                mctx = HawkesContext(cm.N, D, device=local, precision=args.precision, algorithm=args.algorithm)
            mctx.set_times(torch.from_numpy(cm.t).to(dev))
            mctx.set_params(cm.theta)
            mctx.set_locations(torch.from_numpy(cm.x).to(dev))
            mctx.set_regions(rkind, cm.centre, cm.size)
            nblk = 4000
            blk = np.random.default_rng(11).integers(0, cm.N, size=(nblk, 1)).astype(np.int32)
            mctx.mh_sweep(blk[:50], 0.5, 2010, 0)        # warm-up (rates computed once)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            m0.record(mctx.stream)
            acc, _ = mctx.mh_sweep(blk, 0.5, 2010, 1)
            m1.record(mctx.stream)
            torch.cuda.synchronize()
            us = m0.elapsed_time(m1) * 1e3 / nblk
            mh[name] = {"config": f"{name}-shaped N={cm.N}, {rkind} regions, {nblk} blocks of k=1, "
                                  "scale 0.5", "us_per_block": us, "blocks_per_s": 1e6 / us,
                        "acceptance": float(acc.mean())}
            mctx.close()

    # ---- the paper's catalog shapes at N = 100k (SURVEY §8(d) C2 / C3 recipes): the walk
    # order AUTO picks (spatial for the DC shape: exact box culling, NEXT-2) and its time
    shaped = None
    if not args.no_hmc:
        shaped = {}
        for name in ("C2", "C3"):
            cs = synth.config(name, N=N)
            sctx = (init_distributed_context(N, D, precision=args.precision, algorithm=args.algorithm)
                    if world > 1 else HawkesContext(N, D, device=local, precision=args.precision,
                                                     algorithm=args.algorithm))
            xs = torch.from_numpy(cs.x).to(dev)
            sctx.set_times(torch.from_numpy(cs.t).to(dev))
            sctx.set_params(cs.theta)
            gs = torch.empty_like(xs)
            for _ in range(3):
                sctx.set_locations(xs)
                sctx.grad_locations(gs)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(sctx.stream)
            for _ in range(5):
                sctx.set_locations(xs)
                sctx.grad_locations(gs)
            s1.record(sctx.stream)
            torch.cuda.synchronize()
            sms_ = torch.tensor([s0.elapsed_time(s1) / 5], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(sms_, op=dist.ReduceOp.MAX)
            order, cost = sctx.ordering_in_use
            shaped[name] = {"config": f"{name}-shaped N={N} D=2 {args.precision}", "ms_per_eval": float(sms_.item()),
                            "pairs_per_s": N * (N - 1) / (float(sms_.item()) * 1e-3), "walk_order": order,
                            "walk_cost_time_space": cost,
                            "note": "effective pairs/s: culled pairs (exact, below the exp clamp) counted"}
            sctx.close()

    # ---- the paper's catalog sizes (BASELINE configs[1] DC-shaped N = 5000, configs[2]
    # Alaska-shaped N = 20k): per call of hawkes_grad_at (new locations + ell + gradient, one
    # graph launch) with the host synchronised on ell every call, as an MCMC driver calls it;
    # one process (rank 0), 1 GPU
    paper_sized = None
    if not args.no_hmc and rank == 0:
        paper_sized = {}
        for name, Nc in (("C2", 5000), ("C3", 20000)):
            cc = synth.config(name, N=Nc)
            pctx = HawkesContext(Nc, D, device=local, precision=args.precision, algorithm=args.algorithm)
            xc = torch.from_numpy(cc.x).to(dev)
            pctx.set_times(torch.from_numpy(cc.t).to(dev))
            pctx.set_params(cc.theta)
            gc = torch.empty_like(xc)
            for _ in range(10):
                pctx.grad_at(xc, gc)
            torch.cuda.synchronize()
            reps = 400 if Nc <= 5000 else 100
            t0 = time.perf_counter()
            for _ in range(reps):
                pctx.grad_at(xc, gc)
            dt_call = (time.perf_counter() - t0) / reps
            order, _ = pctx.ordering_in_use
            paper_sized[name] = {"config": f"{name}-shaped N={Nc} D=2 {args.precision} (BASELINE configs[{1 if name == 'C2' else 2}])",
                                 "us_per_call": dt_call * 1e6, "calls_per_s": 1.0 / dt_call,
                                 "pairs_per_s": Nc * (Nc - 1) / dt_call, "walk_order": order,
                                 "note": "hawkes_grad_at per call, host wall clock incl. the ell sync"}
            pctx.close()

    # ---- per-rank pass-kernel time (library CUDA events): the load balance of the plan
    pass_ms = [float(kt["rate_ms"] + kt["grad_ms"]) / max(1, kt["rate_launches"])]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, pass_ms[0])
        pass_ms = [float(v) for v in allr]
    ranks = {"world": world, "pass_kernel_ms_per_rank": pass_ms,
             "balance": (sum(pass_ms) / len(pass_ms)) / max(pass_ms) if max(pass_ms) > 0 else None,
             "note": "mean / max over ranks of the per-evaluation pass-kernel time (1 = perfect deal)"}

    # ---- roofline of the dominant pass (FP64 pipe), from the library's own CUDA events
    rate_avg = kt["rate_ms"] / max(1, kt["rate_launches"])
    grad_avg = kt["grad_ms"] / max(1, kt["grad_launches"])
    pairs_alg = pairs / world                   # each rank's launches cover 1/W of the pairs
    unordered = ctx.algorithm in ("auto", "pairs") and args.precision == "fp64"
    fp32_pairs = ctx.algorithm in ("auto", "pairs") and args.precision == "fp32"
    if unordered:
        names = ("rate pass: sym_kernel<2,1,4,4>", "gradient pass: sym_kernel<2,2,4,4>")
        F_impl = F_PIPE
    elif fp32_pairs:
        names = ("rate pass: sym_kernel_f32<2,1,4,1>", "gradient pass: sym_kernel_f32<2,2,4,1>")
        F_impl = F_IMPL32
    else:
        names = ("rate pass: pass_kernel<2,1>", "gradient pass: pass_kernel<2,2>")
        F_impl = (26.5, 26.0)                  # ROWS: ordered pairs, FP64 instructions (SASS)
    pi = 1 if grad_avg >= rate_avg else 0
    dom, avg_ms = names[pi], (grad_avg if pi else rate_avg)
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    sm_max = clocks.get("sm_max_mhz") or 1965.0
    peak = sms * FP64_LANES_PER_SM * sm_max * 1e6 / 1e12   # T lane-ops/s (FP64 pipe / FMA pipe)
    rate_units = pairs_alg / (avg_ms * 1e-3) / 1e12      # T ordered pairs/s
    traffic = _ncu_traffic(dom.split(": ")[1]) if unordered else None
    try:
        dfma_peak = diag_fp64_peak() / 1e12
    except Exception:
        dfma_peak = None

    if fp32_pairs:
        mufu_peak = sms * MUFU_PER_SM * sm_max * 1e6 / 1e12
        achieved = F_impl[pi] * rate_units
        roofline = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak,
                    "unit": "T FMA-pipe instructions/s (one per lane; packed FFMA2/FADD2/FMUL2 = 1)",
                    "frac": achieved / peak, "traffic": traffic,
                    "peak_basis": f"{sms} SMs x 64 lanes x {sm_max:.0f} MHz "
                                  "(one packed FP32 warp-instruction per 2 cycles per SMSP)",
                    "ops_per_pair": F_impl[pi],
                    "ops_per_pair_basis": "FMA-pipe instructions per ordered pair of the shipped "
                                          "sym_kernel_f32's hot loop (SASS)",
                    "mufu": {"achieved": rate_units, "peak": mufu_peak, "frac": rate_units / mufu_peak,
                             "unit": "T ex2/s", "basis": f"1 MUFU ex2 per ordered pair; {sms} SMs x 16 "
                                                         f"/clk x {sm_max:.0f} MHz"}}
    elif unordered:
        achieved = F_ALG[pi] * rate_units
        roofline = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak,
                    "unit": "T FP64 ops/s (algorithmic; DFMA = 1)", "frac": achieved / peak,
                    "traffic": traffic,
                    "peak_basis": f"{sms} SMs x 64 FP64 lanes x {sm_max:.0f} MHz",
                    "ops_per_pair": F_ALG[pi],
                    "ops_per_pair_basis": "frozen algorithmic FP64 operations per ordered pair of the "
                                          "unordered-pair method with a u-accurate 7-op table exp "
                                          "(DESIGN.md §4 Roofline)",
                    "fp64_pipe": {"instr_per_pair": F_impl[pi], "frac": F_impl[pi] * rate_units / peak,
                                  "basis": "FP64 instructions per ordered pair of the shipped hot loop "
                                           "(tools/falg_count.py --shipped): pipe utilisation"},
                    "survey_falg": {"ops_per_pair": F_SURVEY[pi], "frac": F_SURVEY[pi] * rate_units / peak,
                                    "basis": "SURVEY.md 8(d) ordered-pair F_alg (frozen; libdevice exp, "
                                             "ordered pairs)"},
                    "measured_dfma_peak": dfma_peak}
    else:
        achieved = F_impl[pi] * rate_units
        roofline = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak,
                    "unit": "T FP64-pipe instructions/s (DFMA = 1)", "frac": achieved / peak,
                    "traffic": None, "peak_basis": f"{sms} SMs x 64 FP64 lanes x {sm_max:.0f} MHz",
                    "ops_per_pair": F_impl[pi], "ops_per_pair_basis": "ROWS kernel SASS count"}
    out = {
        "metric": METRIC, "value": evals_per_s, "unit": "evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        # the pair arithmetic's type: fp64, or fp32 pair terms (per-tile sums promoted to fp64)
        "dtype": "f64" if args.precision == "fp64" else "f32",
        "data": "synthetic (C4 generator: seeded Philox cluster process, SURVEY.md §8(d))",
        "pairs_per_s": evals_per_s * pairs, "loglik": ell,
        "config": {"workload": f"C4 unit-square Hawkes catalog N={N} D=2 (BASELINE configs[3])",
                   "N": N, "D": 2, "precision": args.precision, "algorithm": ctx.algorithm,
                   "l2": "flushed before every timed step (256 MiB device write, outside the step events)",
                   "parallelism": (f"chunk-pair sharded x{world} (LPT-dealt unordered chunk pairs, NCCL "
                                   "allgather of per-event partial sums per pass, added in rank order)"
                                   if ctx.algorithm in ("auto", "pairs") else
                                   f"row-sharded x{world} (zig-zag tiles, NCCL allgather of 1/lambda)")
                   if world > 1 else "1 GPU"},
        "clocks": clocks,
        "ranks": ranks,
        "gpu_launches": kt["total_launches"],
        "kernel_ms": {"rate_pass_avg": rate_avg, "grad_pass_avg": grad_avg,
                      "rate_launches": kt["rate_launches"], "grad_launches": kt["grad_launches"]},
        "roofline": roofline,
        "e2e": {"value": e2e_val, "unit": "evals/s", "h2d_bytes_per_step": N * D * 8,
                "d2h_bytes_per_step": N * D * 8 + 8},
        "loglik_only": loglik_only,
        "hmc": hmc,
        "mh_sweep": mh,
        "shaped": shaped,
        "paper_sized": paper_sized,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline()
        out["cpu_baseline"] = {
            "value": cb["pairs_per_s"] / pairs, "unit": "evals/s", "cores": cb["cores"],
            "kind": "oracle", "pairs_per_s": cb["pairs_per_s"], "cpu": cb["cpu"],
            "sample": f"full oracle ell+gradient of the C4 generator at N={cb['Ns']} "
                      f"({cb['seconds']:.1f} s), scaled to N={N} by N(N-1) ordered pairs"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=100_000)
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64")
    ap.add_argument("--algorithm", choices=["auto", "rows", "pairs"], default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-hmc", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


def relaunch(args):
    """`--gpus N > 1` without a torchrun environment: re-launch this command as N ranks
    (one process per GPU, rendezvous on 127.0.0.1), as the driver would."""
    if args.impl == "ours":
        import torch
        n = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if n < args.gpus:
            print(json.dumps({"metric": METRIC, "n_gpus": args.gpus, "value": None,
                              "error": f"--gpus {args.gpus} needs {args.gpus} visible GPUs, found {n}"}),
                  flush=True)
            return 1
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
