"""Build the in-tree C-ABI library libhawkes_b200.so for sm_100a (nvcc, no torch extension).

    python -m paper_2010_02994_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhawkes_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _nccl_include() -> str:
    cands = glob.glob(os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl", "include"))
    cands += ["/usr/include"]
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h"))
                  + [os.path.join(ROOT, "include", "hawkes.h")])


def build(force: bool = False, verbose: bool = False, defines=(), out: str = None) -> str:
    """Build the library (out: another path, with extra -D defines, for A/B builds)."""
    srcs = sources()
    lib = out or LIB
    if not force and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(s) <= t for s in srcs):
            return lib
    cus = [s for s in srcs if s.endswith(".cu")]
    cmd = [_nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
           "-Xptxas", "-v" if verbose else "-O3", "-shared", "-I", os.path.join(ROOT, "include"),
           "-I", _nccl_include(), *[f"-D{d}" for d in defines], *cus, "-o", lib + ".tmp",
           "-ldl", "-lcudart"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
