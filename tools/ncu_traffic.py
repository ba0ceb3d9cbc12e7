"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of each kernel in an
ncu --set full raw-page CSV, averaged over its captured launches, as JSON keyed by the short
kernel name bench.py reports (e.g. "sym_kernel<2,1,4,6>").

    ncu -i rep.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_traffic.py raw.csv [source-label] > profiles/r01_ncu_traffic.json
"""
import csv
import json
import re
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    m = re.match(r"void (?:hk::)?(\w+)<([^>]*)>", name)
    if not m:
        return name
    args = ",".join(re.sub(r"\(int\)|\(bool\)", "", a).strip() for a in m.group(2).split(","))
    return f"{m.group(1)}<{args}>"


def main(path, label=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    acc = {}
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        k = short(r[col["Kernel Name"]])
        b = {}
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b[m] = float(r[col[m]].replace(",", "")) * SCALE.get(units[col[m]], 1)
        a = acc.setdefault(k, {"read": 0.0, "write": 0.0, "launches": 0})
        a["read"] += b["dram__bytes_read.sum"]
        a["write"] += b["dram__bytes_write.sum"]
        a["launches"] += 1
    out = {}
    for k, a in acc.items():
        n = a["launches"]
        out[k] = {"bytes": (a["read"] + a["write"]) / n, "read": a["read"] / n, "write": a["write"] / n,
                  "launches": n, "source": label or path}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(*sys.argv[1:])
