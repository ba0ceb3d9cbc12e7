"""FP64 pipe throughput per operand pattern (hawkes_diag_fp64_mode)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_02994_b200 import _lib
lib = _lib.load()
peak = 148 * 64 * 1.965e9
names = {0: "DFMA r,imm,imm", 1: "DFMA r,r,r", 2: "DADD r,r", 3: "DMUL r,r", 4: "fast exp (9 ops)",
         5: "DFMA r,r,imm", 6: "DFMA/DADD alt", 7: "exp FP64 only(10)", 8: "exp no select(9)",
         9: "1 dep chain", 10: "DFMA/DMUL alt", 11: "DFMA/DFMA(1.0)", 12: "exp cheap-int(9)"}
for w in (12, 16, 32):
    for m in range(13):
        v = ctypes.c_double()
        _lib.check(lib.hawkes_diag_fp64_mode(m, w, ctypes.byref(v)))
        ops = v.value * {4: 9, 7: 10, 8: 9, 12: 9}.get(m, 1)
        print(f"warps/SM={w:2d} mode {m} {names[m]:18s} {ops/1e12:7.2f} T FP64 ops/s  ({ops/peak*100:5.1f}% of 148x64x1965MHz)")
