"""Python binding of the C ABI (include/hawkes.h): same names, argument marshalling only.

Every step of the computation runs in libhawkes_b200.so; torch is used for device memory
(tensors passed in / out), the current CUDA stream and the process group that hands the
NCCL unique id to every rank.

    ctx = HawkesContext(N, D)                 # hawkes_create
    ctx.set_times(t); ctx.set_locations(x); ctx.set_params(theta)
    ell = ctx.loglik()                        # Eq. 1
    g, ell = ctx.grad_locations()             # App. A
    x, p, ell, kin = ctx.leapfrog(x, p, step, n_steps)   # HMC over X
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import HAWKES_FP32, HAWKES_FP64, HAWKES_MEM_DEVICE, HAWKES_MEM_HOST, HawkesError, check

__all__ = ["HawkesContext", "HawkesError", "nccl_unique_id", "diag_exp", "diag_fp64_peak"]


def _ptr_mem(a) -> Tuple[int, int, object]:
    """(pointer, hawkes_mem, keep-alive) for a float64 torch tensor or numpy array."""
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.float64:
            raise TypeError("arrays must be float64")
        if not a.is_contiguous():
            raise ValueError("arrays must be contiguous")
        return a.data_ptr(), (HAWKES_MEM_DEVICE if a.is_cuda else HAWKES_MEM_HOST), a
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return arr.ctypes.data, HAWKES_MEM_HOST, arr


def nccl_unique_id() -> bytes:
    """hawkes_nccl_unique_id: 128 bytes for opts.nccl_unique_id (rank 0 calls this)."""
    lib = _lib.load()
    buf = ctypes.create_string_buffer(128)
    check(lib.hawkes_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


class HawkesContext:
    """hawkes_create / hawkes_destroy and the calls on one context."""

    def __init__(self, N: int, D: int, device: int = 0, stream: Optional[torch.cuda.Stream] = None,
                 precision: str = "fp64", rank: int = 0, world: int = 1,
                 nccl_id: Optional[bytes] = None, emulate_world: int = 0,
                 algorithm: str = "auto"):
        self._lib = _lib.load()
        self.N, self.D, self.device = int(N), int(D), int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        o = _lib.Opts()
        self._lib.hawkes_default_opts(ctypes.byref(o))
        o.device = self.device
        o.cuda_stream = stream.cuda_stream
        o.precision = {"fp64": HAWKES_FP64, "fp32": HAWKES_FP32}[precision]
        o.rank, o.world = int(rank), int(world)
        self._id = None
        if nccl_id is not None:
            self._id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_unique_id = ctypes.cast(self._id, ctypes.c_void_p)
        o.emulate_world = int(emulate_world)
        o.algorithm = _lib.ALGORITHMS[algorithm]
        self.algorithm = algorithm
        h = ctypes.c_void_p()
        check(self._lib.hawkes_create(self.N, self.D, ctypes.byref(o), ctypes.byref(h)))
        self._h = h

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._lib.hawkes_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- inputs
    def set_times(self, t):
        p, mem, keep = _ptr_mem(t)
        check(self._lib.hawkes_set_times(self._h, p, mem), self._h)

    def set_locations(self, x):
        p, mem, keep = _ptr_mem(x)
        check(self._lib.hawkes_set_locations(self._h, p, mem), self._h)

    def set_params(self, theta: Sequence[float]):
        """Theta = (mu0, tau_x, tau_t, theta, omega, h) in the paper's order."""
        prm = _lib.Params(*[float(v) for v in theta])
        check(self._lib.hawkes_set_params(self._h, ctypes.byref(prm)), self._h)

    # -- evaluations
    def loglik(self) -> float:
        out = ctypes.c_double()
        check(self._lib.hawkes_loglik(self._h, ctypes.byref(out)), self._h)
        return out.value

    def grad_locations(self, out=None) -> Tuple[object, float]:
        """Returns (gradient N x D, ell).  ``out`` may be a float64 CUDA tensor or a host
        array/tensor; default: a new CUDA tensor on this context's device."""
        if out is None:
            out = torch.empty((self.N, self.D), dtype=torch.float64, device=f"cuda:{self.device}")
        p, mem, keep = _ptr_mem(out)
        ll = ctypes.c_double()
        check(self._lib.hawkes_grad_locations(self._h, p, mem, ctypes.byref(ll)), self._h)
        return out, ll.value

    def grad_at(self, x, out=None) -> Tuple[object, float]:
        """set_locations(x) + grad_locations(out) in one call (hawkes_grad_at): x and out are
        float64 CUDA tensors (N x D); returns (out, ell)."""
        if out is None:
            out = torch.empty((self.N, self.D), dtype=torch.float64, device=f"cuda:{self.device}")
        px, memx, kx = _ptr_mem(x)
        po, memo, ko = _ptr_mem(out)
        if memx != HAWKES_MEM_DEVICE or memo != HAWKES_MEM_DEVICE:
            raise ValueError("grad_at takes device arrays (float64 CUDA tensors)")
        ll = ctypes.c_double()
        check(self._lib.hawkes_grad_at(self._h, px, po, ctypes.byref(ll)), self._h)
        return out, ll.value

    def get_rates(self) -> dict:
        """lambda_n, mu_n, xi_n, Lambda_n of the current state (numpy, host)."""
        arrs = {k: np.empty(self.N) for k in ("lambda", "mu", "xi", "Lambda")}
        ptrs = [arrs[k].ctypes.data for k in ("lambda", "mu", "xi", "Lambda")]
        check(self._lib.hawkes_get_rates(self._h, *ptrs, HAWKES_MEM_HOST), self._h)
        return arrs

    def leapfrog(self, x, p, step: float, n_steps: int, inv_mass=None, box_lo=None, box_hi=None):
        """Runs hawkes_leapfrog in place on x and p (same memory kind); returns
        (x, p, ell_end, kinetic_end)."""
        px, mem, kx = _ptr_mem(x)
        pp, memp, kp = _ptr_mem(p)
        if memp != mem:
            raise ValueError("x and p must live in the same memory")
        if kx is not x or kp is not p:
            raise ValueError("x and p must be contiguous float64 arrays/tensors (updated in place)")
        extra = []
        for a in (inv_mass, box_lo, box_hi):
            if a is None:
                extra.append((None, None))
            else:
                pa, ma, ka = _ptr_mem(a)
                if ma != mem:
                    raise ValueError("inv_mass / box arrays must live with x")
                extra.append((pa, ka))
        ll, kin = ctypes.c_double(), ctypes.c_double()
        check(self._lib.hawkes_leapfrog(self._h, px, pp, mem, float(step), int(n_steps),
                                        extra[0][0], extra[1][0], extra[2][0],
                                        ctypes.byref(ll), ctypes.byref(kin)), self._h)
        return x, p, ll.value, kin.value

    def hmc_step(self, seed: int, iteration: int, step: float, n_steps: int, inv_mass=None,
                 box_lo=None, box_hi=None, x_out=None):
        """hawkes_hmc_step: one HMC transition from the context's locations with on-device
        Philox momenta and Metropolis decision.  inv_mass / box / x_out share one memory kind
        (host numpy or CUDA tensors).  Returns (accepted: bool, log_alpha: float); the new
        state is written into x_out when given."""
        arrs = [inv_mass, box_lo, box_hi, x_out]
        ptrs, mems, keep = [], set(), []
        for a in arrs:
            if a is None:
                ptrs.append(None)
                continue
            pa, ma, ka = _ptr_mem(a)
            ptrs.append(pa)
            mems.add(ma)
            keep.append(ka)
        if len(mems) > 1:
            raise ValueError("inv_mass, box and x_out must live in the same memory")
        if x_out is not None and keep[-1] is not x_out:
            raise ValueError("x_out must be a contiguous float64 array/tensor")
        mem = mems.pop() if mems else HAWKES_MEM_DEVICE
        acc, la = ctypes.c_int32(), ctypes.c_double()
        check(self._lib.hawkes_hmc_step(self._h, int(seed), int(iteration), float(step),
                                        int(n_steps), ptrs[0], ptrs[1], ptrs[2], mem, ptrs[3],
                                        ctypes.byref(acc), ctypes.byref(la)), self._h)
        return bool(acc.value), la.value

    # -- block Metropolis-Hastings over coarsened locations
    def set_regions(self, kind: str, centre, size):
        """hawkes_set_regions: "square" (Eq. locsPrior1, size = half-width) or "disc"
        (Eq. locsPrior2, size = radius) uniform location priors, N x D centres, N sizes."""
        pc, mc, kc = _ptr_mem(centre)
        ps, ms, ks = _ptr_mem(size)
        if mc != ms:
            raise ValueError("centre and size must live in the same memory")
        check(self._lib.hawkes_set_regions(self._h, _lib.REGIONS[kind], pc, ps, mc), self._h)

    def mh_sweep(self, blocks, scale: float, seed: int, iteration: int):
        """hawkes_mh_sweep: sequential block MH updates, blocks = (n_blocks, k) int array of
        distinct event indices per row.  Returns (accepted bool array, log_alpha array)."""
        blk = np.ascontiguousarray(np.asarray(blocks, dtype=np.int32))
        if blk.ndim != 2:
            raise ValueError("blocks must be (n_blocks, k)")
        nb, k = blk.shape
        acc = np.zeros(nb, dtype=np.int32)
        la = np.zeros(nb, dtype=np.float64)
        nacc = ctypes.c_int32()
        check(self._lib.hawkes_mh_sweep(self._h, nb, k, blk.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                        float(scale), int(seed), int(iteration),
                                        acc.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                        la.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                        ctypes.byref(nacc)), self._h)
        return acc.astype(bool), la

    def get_locations(self, out=None):
        """The context's current locations (N x D float64 CUDA tensor), e.g. after MH sweeps."""
        if out is None:
            out = torch.empty((self.N, self.D), dtype=torch.float64, device=f"cuda:{self.device}")
        p, mem, keep = _ptr_mem(out)
        check(self._lib.hawkes_get_locations(self._h, p, mem), self._h)
        return out

    # -- Bayesian MDS and the HMC potential
    def set_bmds(self, Y, sigma: float):
        """hawkes_set_bmds: N x N dissimilarities (lower triangle read) and sigma."""
        p, mem, keep = _ptr_mem(Y)
        check(self._lib.hawkes_set_bmds(self._h, p, mem, float(sigma)), self._h)

    def bmds_logdensity(self, grad: bool = True, out=None):
        """hawkes_bmds_logdensity: (log p(Y | X), gradient N x D or None)."""
        lp = ctypes.c_double()
        if grad and out is None:
            out = torch.empty((self.N, self.D), dtype=torch.float64, device=f"cuda:{self.device}")
        if grad:
            p, mem, keep = _ptr_mem(out)
        else:
            p, mem = None, HAWKES_MEM_DEVICE
        check(self._lib.hawkes_bmds_logdensity(self._h, p, mem, ctypes.byref(lp)), self._h)
        return lp.value, (out if grad else None)

    def set_potential(self, hawkes: bool = True, bmds: bool = False):
        """hawkes_set_potential: which log densities the leapfrog potential includes."""
        flags = (_lib.POTENTIAL_HAWKES if hawkes else 0) | (_lib.POTENTIAL_BMDS if bmds else 0)
        check(self._lib.hawkes_set_potential(self._h, flags), self._h)

    # -- block Metropolis-Hastings moves
    def propose_move(self, idx, new_x) -> float:
        """hawkes_propose_move: ell(X') - ell(X) for events idx moved to new_x (k x D)."""
        idx = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1)
        p, mem, keep = _ptr_mem(new_x)
        out = ctypes.c_double()
        check(self._lib.hawkes_propose_move(self._h, int(idx.size),
                                            idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                            p, mem, ctypes.byref(out)), self._h)
        return out.value

    def accept_move(self):
        """hawkes_accept_move: commit the pending proposal."""
        check(self._lib.hawkes_accept_move(self._h), self._h)

    # -- timing (CUDA events recorded by the library around the two pass kernels)
    @property
    def precision_in_use(self) -> str:
        """hawkes_precision_in_use: "fp32", or "fp64" once an fp32 context's range guard
        (reading R23) sent it to the fp64 kernels."""
        v = ctypes.c_int32()
        check(self._lib.hawkes_precision_in_use(self._h, ctypes.byref(v)), self._h)
        return "fp32" if v.value == HAWKES_FP32 else "fp64"

    def set_ordering(self, mode: str = "auto"):
        """hawkes_set_ordering: walk order of the PAIRS fp64 kernels, "auto" | "time" | "space"
        (include/hawkes.h hawkes_ordering)."""
        check(self._lib.hawkes_set_ordering(self._h, _lib.ORDERINGS[mode]), self._h)

    @property
    def ordering_in_use(self) -> Tuple[str, Tuple[float, float]]:
        """hawkes_ordering_in_use: ("time" | "space", (time-order cost, space-order cost))."""
        v = ctypes.c_int32()
        cost = (ctypes.c_double * 2)()
        check(self._lib.hawkes_ordering_in_use(self._h, ctypes.byref(v), cost), self._h)
        return ("space" if v.value == 2 else "time"), (cost[0], cost[1])

    def enable_timing(self, enable: bool = True):
        check(self._lib.hawkes_enable_timing(self._h, int(bool(enable))), self._h)

    def kernel_times(self) -> dict:
        r, g = ctypes.c_double(), ctypes.c_double()
        nr, ng, tot = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(self._lib.hawkes_get_kernel_times(self._h, ctypes.byref(r), ctypes.byref(nr),
                                                ctypes.byref(g), ctypes.byref(ng),
                                                ctypes.byref(tot)), self._h)
        return {"rate_ms": r.value, "rate_launches": nr.value, "grad_ms": g.value,
                "grad_launches": ng.value, "total_launches": tot.value}


def diag_exp(a: torch.Tensor) -> torch.Tensor:
    """The kernels' fast exp applied to a float64 CUDA tensor (accuracy tests)."""
    a = a.contiguous()
    out = torch.empty_like(a)
    check(_lib.load().hawkes_diag_exp(a.data_ptr(), out.data_ptr(), a.numel()))
    return out


def diag_normals(seed: int, iteration: int, n: int, device: int = 0) -> torch.Tensor:
    """The standard normals hawkes_hmc_step draws for (seed, iteration) (RNG parity tests)."""
    out = torch.empty(n, dtype=torch.float64, device=f"cuda:{device}")
    check(_lib.load().hawkes_diag_normals(int(seed), int(iteration), out.data_ptr(), int(n)))
    return out


def diag_fp64_peak() -> float:
    """Measured dependent-DFMA throughput of the current device, FP64 lane-ops/s."""
    v = ctypes.c_double()
    check(_lib.load().hawkes_diag_fp64_peak(ctypes.byref(v)))
    return v.value
