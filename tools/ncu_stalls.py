"""Warp-stall breakdown of each kernel in an ncu --set full report's SASS source page: the
sampled stall reasons summed over all instructions (share of samples), the issue share, and
per opcode the samples and the shared-memory wavefronts / excess (bank-conflict) wavefronts.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_stalls.py src.csv [--kernel SUBSTR] [--hot]

--hot restricts the per-opcode table to the kernel's hottest loop (the instructions between
the back-edge with the most samples and its target).
"""
import csv
import re
import sys
from collections import defaultdict


def sections(path):
    rows = list(csv.reader(open(path)))
    cur, hdr, out = None, None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            out.append(cur)
            hdr = None
        elif r and r[0] == "Address":
            hdr = r
        elif hdr and cur is not None and len(r) == len(hdr):
            cur["rows"].append(dict(zip(hdr, r)))
    return out


def num(v):
    try:
        return float(v.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main():
    args = sys.argv[1:]
    path = args[0]
    want = None
    if "--kernel" in args:
        want = args[args.index("--kernel") + 1]
    hot = "--hot" in args
    for sec in sections(path):
        if want and want not in sec["name"]:
            continue
        rows = sec["rows"]
        stall_cols = [c for c in rows[0] if c.startswith("stall_") and "(Not Issued)" not in c]
        tot = defaultdict(float)
        for r in rows:
            for c in stall_cols:
                tot[c] += num(r[c])
        n = sum(tot.values())
        print(f"== {sec['name']}  ({int(n)} stall samples)")
        for c, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            if v / max(n, 1) >= 0.005:
                print(f"   {c:28s} {100 * v / n:6.2f} %")
        sel = rows
        if hot:
            addr = [int(r["Address"], 16) for r in rows]
            best = None
            for k, r in enumerate(rows):
                m = re.search(r"BRA.*?(0x[0-9a-f]+)", r["Source"])
                if not m:
                    continue
                tgt = int(m.group(1), 16)
                if tgt >= addr[k]:
                    continue
                body = [q for q in rows if tgt <= int(q["Address"], 16) <= addr[k]]
                s = sum(num(q["# Samples"]) for q in body)
                if best is None or s > best[0]:
                    best = (s, body)
            if best:
                sel = best[1]
                print(f"   hottest loop: {len(sel)} instructions, "
                      f"{100 * best[0] / max(1, sum(num(q['# Samples']) for q in rows)):.1f} % of samples")
        per = defaultdict(lambda: defaultdict(float))
        for r in sel:
            op = r["Source"].strip().split()
            if not op:
                continue
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            o = o.split(".")[0] + ("." + o.split(".")[1] if o.startswith("LDS") and "." in o else "")
            p = per[o]
            p["samples"] += num(r["# Samples"])
            p["inst"] += num(r["Instructions Executed"])
            p["wf"] += num(r["L1 Wavefronts Shared"])
            p["wf_ideal"] += num(r["L1 Wavefronts Shared Ideal"])
            for c in ("stall_short_sb", "stall_mio", "stall_math", "stall_wait", "stall_dispatch",
                      "stall_not_selected", "stall_selected", "stall_long_sb", "stall_barrier"):
                p[c] += num(r.get(c, "0"))
        S = sum(p["samples"] for p in per.values())
        print(f"   {'opcode':14s} {'samples%':>8s} {'inst':>12s} {'smem wf':>12s} {'excess wf':>10s}  top stalls")
        for o, p in sorted(per.items(), key=lambda kv: -kv[1]["samples"])[:14]:
            st = sorted(((c, p[c]) for c in p if c.startswith("stall_")), key=lambda kv: -kv[1])[:3]
            sts = ", ".join(f"{c[6:]} {100 * v / max(p['samples'], 1):.0f}%" for c, v in st if v)
            print(f"   {o:14s} {100 * p['samples'] / max(S, 1):8.2f} {p['inst']:12.3g} {p['wf']:12.3g} "
                  f"{p['wf'] - p['wf_ideal']:10.3g}  {sts}")
        print()


if __name__ == "__main__":
    main()
