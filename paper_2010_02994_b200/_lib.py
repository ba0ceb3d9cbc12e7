"""ctypes declarations for libhawkes_b200.so (include/hawkes.h).  Marshalling only.

There is no fallback: if the in-tree library is missing or fails to load, importing
the binding raises, so nothing can silently run the computation elsewhere.
"""
from __future__ import annotations

import ctypes
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhawkes_b200.so")
# diagnostics only (tools/ab_builds.py): load an A/B build of the same sources instead
LIB_PATH = os.environ.get("HAWKES_LIB_AB", LIB_PATH)

HAWKES_OK = 0
STATUS = {
    0: "HAWKES_OK", -1: "HAWKES_ERR_ARG", -2: "HAWKES_ERR_DIM", -3: "HAWKES_ERR_UNSORTED",
    -4: "HAWKES_ERR_NONFINITE", -5: "HAWKES_ERR_PARAM", -6: "HAWKES_ERR_STATE",
    -7: "HAWKES_ERR_GRAD_UNDEFINED", -8: "HAWKES_ERR_CUDA", -9: "HAWKES_ERR_NCCL",
    -10: "HAWKES_ERR_OOM",
}
HAWKES_FP64, HAWKES_FP32 = 0, 1
HAWKES_MEM_HOST, HAWKES_MEM_DEVICE = 0, 1
ALGORITHMS = {"auto": 0, "rows": 1, "pairs": 2}
POTENTIAL_HAWKES, POTENTIAL_BMDS = 1, 2
REGIONS = {"square": 1, "disc": 2}

# every symbol include/hawkes.h declares (checked by tests/test_abi_cpu.py)
EXPORTS = (
    "hawkes_default_opts", "hawkes_create", "hawkes_destroy", "hawkes_set_times",
    "hawkes_set_locations", "hawkes_set_params", "hawkes_loglik", "hawkes_grad_locations",
    "hawkes_grad_at",
    "hawkes_leapfrog", "hawkes_hmc_step", "hawkes_get_rates", "hawkes_propose_move", "hawkes_accept_move",
    "hawkes_set_regions", "hawkes_mh_sweep", "hawkes_get_locations",
    "hawkes_set_bmds", "hawkes_bmds_logdensity", "hawkes_set_potential", "hawkes_enable_timing", "hawkes_get_kernel_times",
    "hawkes_plan", "hawkes_plan_pairs", "hawkes_nccl_unique_id", "hawkes_diag_exp", "hawkes_diag_normals", "hawkes_diag_fp64_peak", "hawkes_diag_fp64_mode", "hawkes_last_error",
    "hawkes_abi_version", "hawkes_precision_in_use", "hawkes_set_ordering", "hawkes_ordering_in_use",
    "hawkes_plan_walk", "hawkes_plan_slots", "hawkes_plan_items",
)
ORDERINGS = {"auto": 0, "time": 1, "space": 2}


class Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("cuda_stream", ctypes.c_void_p),
                ("precision", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("emulate_world", ctypes.c_int32),
                ("algorithm", ctypes.c_int32)]


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("mu0", "tau_x", "tau_t", "theta", "omega", "sigma_x")]


class HawkesError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        self.status = STATUS.get(code, str(code))
        super().__init__(f"{self.status}: {msg}")


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2010_02994_b200.build`"
                          " (or __graft_entry__.build()); there is no fallback implementation")
    lib = ctypes.CDLL(LIB_PATH)
    P, vp, dp = ctypes.POINTER, ctypes.c_void_p, ctypes.c_void_p
    i32, i64 = ctypes.c_int32, ctypes.c_int64
    lib.hawkes_default_opts.argtypes = [P(Opts)]
    lib.hawkes_create.argtypes = [i64, i32, P(Opts), P(vp)]
    lib.hawkes_destroy.argtypes = [vp]
    lib.hawkes_set_times.argtypes = [vp, dp, i32]
    lib.hawkes_set_locations.argtypes = [vp, dp, i32]
    lib.hawkes_set_params.argtypes = [vp, P(Params)]
    lib.hawkes_loglik.argtypes = [vp, P(ctypes.c_double)]
    lib.hawkes_grad_locations.argtypes = [vp, dp, i32, P(ctypes.c_double)]
    lib.hawkes_grad_at.argtypes = [vp, dp, dp, P(ctypes.c_double)]
    lib.hawkes_leapfrog.argtypes = [vp, dp, dp, i32, ctypes.c_double, i32, dp, dp, dp,
                                    P(ctypes.c_double), P(ctypes.c_double)]
    u64 = ctypes.c_uint64
    lib.hawkes_hmc_step.argtypes = [vp, u64, u64, ctypes.c_double, i32, dp, dp, dp, i32, dp,
                                    P(i32), P(ctypes.c_double)]
    lib.hawkes_get_locations.argtypes = [vp, dp, i32]
    lib.hawkes_set_regions.argtypes = [vp, i32, dp, dp, i32]
    lib.hawkes_mh_sweep.argtypes = [vp, i32, i32, P(i32), ctypes.c_double, u64, u64, P(i32),
                                    P(ctypes.c_double), P(i32)]
    lib.hawkes_diag_normals.argtypes = [u64, u64, dp, i64]
    lib.hawkes_get_rates.argtypes = [vp, dp, dp, dp, dp, i32]
    lib.hawkes_propose_move.argtypes = [vp, i32, P(i32), dp, i32, P(ctypes.c_double)]
    lib.hawkes_accept_move.argtypes = [vp]
    lib.hawkes_set_bmds.argtypes = [vp, dp, i32, ctypes.c_double]
    lib.hawkes_bmds_logdensity.argtypes = [vp, dp, i32, P(ctypes.c_double)]
    lib.hawkes_set_potential.argtypes = [vp, i32]
    lib.hawkes_enable_timing.argtypes = [vp, i32]
    lib.hawkes_precision_in_use.argtypes = [vp, P(i32)]
    lib.hawkes_set_ordering.argtypes = [vp, i32]
    lib.hawkes_plan_walk.argtypes = [dp, dp, i64, i32, P(Params), P(i32), P(ctypes.c_double)]
    lib.hawkes_plan_slots.argtypes = [i64, i32, i32, P(i64), P(i64)]
    lib.hawkes_plan_items.argtypes = [i64, i32, i32, i32, P(i64), P(i32), P(i32), P(i64)]
    lib.hawkes_ordering_in_use.argtypes = [vp, P(i32), P(ctypes.c_double)]
    lib.hawkes_get_kernel_times.argtypes = [vp, P(ctypes.c_double), P(i64), P(ctypes.c_double),
                                            P(i64), P(i64)]
    lib.hawkes_nccl_unique_id.argtypes = [vp]
    lib.hawkes_plan.argtypes = [i64, i32, i32, P(i32), P(i32), P(i32), P(i32)]
    lib.hawkes_plan_pairs.argtypes = [i64, i32, i32, P(i32), P(i32), P(i32)]
    lib.hawkes_diag_exp.argtypes = [dp, dp, i64]
    lib.hawkes_diag_fp64_peak.argtypes = [P(ctypes.c_double)]
    lib.hawkes_diag_fp64_mode.argtypes = [i32, i32, P(ctypes.c_double)]
    lib.hawkes_last_error.argtypes = [vp]
    lib.hawkes_last_error.restype = ctypes.c_char_p
    lib.hawkes_abi_version.restype = ctypes.c_int
    _lib = lib
    return lib


def check(rc: int, ctx=None):
    if rc != HAWKES_OK:
        msg = load().hawkes_last_error(ctx)
        raise HawkesError(rc, (msg or b"").decode(errors="replace"))
