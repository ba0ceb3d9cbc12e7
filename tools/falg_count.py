"""Algorithmic FP64 work per pair, counted the way SURVEY.md 8(d) froze F_alg: compile naive
per-pair bodies (libdevice exp) for sm_100a and count the FP64-pipe instructions (DFMA,
DADD, DMUL, DSETP) in each kernel's hot loop (the instructions between a backward branch's
target and the branch).  tools/falg/naive_pairs.cu holds ordered-pair (SURVEY's accounting)
and unordered-pair ("report against an unordered-pair F_alg") bodies.

    python tools/falg_count.py            # prints one line per kernel; no GPU needed

It also counts the shipped sym_kernel<2, PASS, 4, V> hot loops (the unmasked 32-step loop:
one step = 4 unordered pairs) in the built library, i.e. the FP64-pipe instructions this
implementation needs per pair.
"""
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

HERE = os.path.dirname(os.path.abspath(__file__))
FP64 = ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX")


def main():
    src = os.path.join(HERE, "falg", "naive_pairs.cu")
    with tempfile.TemporaryDirectory() as d:
        cubin = os.path.join(d, "n.cubin")
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-cubin",
                               "-o", cubin, src])
        sass = subprocess.check_output(["cuobjdump", "-sass", cubin], text=True)
    for f in re.split(r"\n\s+Function : ", sass)[1:]:
        name = f.split("\n")[0].strip()
        ins = [(int(a, 16), b) for a, b in
               re.findall(r"/\*([0-9a-f]{4})\*/\s+((?:@!?U?P\w+\s+)?[A-Z0-9_.]+[^;]*);", f)]
        for addr, s in ins:
            if "BRA" not in s:
                continue
            m = re.search(r"0x([0-9a-f]+)", s)
            if not m or int(m.group(1), 16) >= addr:
                continue
            tgt = int(m.group(1), 16)
            body = [re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
                    for a, t in ins if tgt <= a <= addr]
            c = Counter(o for o in body if o in FP64)
            per = "unordered" if name.startswith("uno") else "ordered"
            print(f"{name}: hot loop {len(body)} instructions, FP64 pipe {sum(c.values())} per {per} pair "
                  f"{dict(c)}")


def shipped():
    """FP64-pipe and other instructions per 4-pair step of the shipped sym_kernel<2, PASS, 4, V>
    hot loops: among the back-edge loops without selects (the unmasked ones), the self-exciting
    variant (8 exps = 8 VIMNMX clamps per step; the loop may be unrolled, steps = VIMNMX / 8)."""
    lib = os.path.join(os.path.dirname(HERE), "paper_2010_02994_b200", "libhawkes_b200.so")
    lib = os.environ.get("HAWKES_LIB_AB", lib)
    sass = subprocess.check_output(["cuobjdump", "-sass", lib], text=True, stderr=subprocess.DEVNULL)
    for f in re.split(r"\n\s+Function : ", sass)[1:]:
        name = f.split("\n")[0].strip()
        m = re.match(r"_ZN2hk10sym_kernelILi2ELi([12])ELi4ELi(\d)ELb0ELb0E(?:Li4E)?EEvNS_7SymArgsE", name)
        if not m:
            continue
        ins = [(int(a, 16), b) for a, b in
               re.findall(r"/\*([0-9a-f]{4,5})\*/\s+((?:@!?U?P\w+\s+)?[A-Z0-9_.]+[^;]*);", f)]
        best = None
        for addr, s in ins:
            if "BRA" not in s:
                continue
            mm = re.search(r"0x([0-9a-f]+)", s)
            if not mm or int(mm.group(1), 16) >= addr:
                continue
            tgt = int(mm.group(1), 16)
            body = [re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
                    for a, t in ins if tgt <= a <= addr]
            c = Counter(body)
            n64 = sum(c[o] for o in FP64)
            if not n64 or c["VIMNMX"] == 0 or c["SEL"] + c["FSEL"] + c["DSETP"] > 0:
                continue
            if best is None or c["VIMNMX"] / n64 > best[0]:
                best = (c["VIMNMX"] / n64, body, n64, c["VIMNMX"] // 8)
        _, body, n64, steps = best
        n64 /= steps
        other = len(body) / steps - n64
        print(f"sym_kernel<2,{m.group(1)},4,{m.group(2)}>: step {len(body) / steps:.1f} instructions "
              f"({steps} step(s) per loop iteration), FP64 pipe {n64:.1f} per 4 unordered pairs = "
              f"{n64 / 8:.2f} per ordered pair, other {other:.1f}; dispatch-model FP64 utilisation "
              f"{2 * n64 / (2 * n64 + other):.3f}, dispatch cycles per step {2 * n64 + other:.1f}")


if __name__ == "__main__":
    if "--shipped" in sys.argv:
        sys.exit(shipped())
    sys.exit(main())
