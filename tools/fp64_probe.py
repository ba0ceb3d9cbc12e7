"""FP64 pipe throughput per operand pattern (hawkes_diag_fp64_mode)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_02994_b200 import _lib
lib = _lib.load()
peak = 148 * 64 * 1.965e9
names = {0: "DFMA r,imm,imm", 1: "DFMA r,r,r", 2: "DADD r,r", 3: "DMUL r,r", 4: "fast exp (7 FP64)",
         5: "DFMA r,r,imm", 6: "DFMA/DADD alt",
         9: "1 dep chain", 10: "DFMA/DMUL alt", 11: "DFMA/DFMA(1.0)",
         13: "DFMA + I2F.F64", 14: "I2F.F64 alone", 15: "exp kf=I2F (6 FP64)"}
for w in (12, 16, 32):
    for m in (0, 1, 2, 3, 4, 5, 6, 10, 11, 13, 14, 15):
        v = ctypes.c_double()
        _lib.check(lib.hawkes_diag_fp64_mode(m, w, ctypes.byref(v)))
        ops = v.value * {4: 7, 15: 6}.get(m, 1)
        print(f"warps/SM={w:2d} mode {m} {names[m]:18s} {ops/1e12:7.2f} T FP64 ops/s  ({ops/peak*100:5.1f}% of 148x64x1965MHz)")
