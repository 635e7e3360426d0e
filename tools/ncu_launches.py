"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/ncu_launches.py gpurun_out/launches.csv [more.csv ...]
"""
import csv
import sys


def totals(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    tot = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        t = tot.setdefault(name, [0.0, 0])
        t[0] += v
        t[1] += 1
    return tot


if __name__ == "__main__":
    for path in sys.argv[1:]:
        tot = totals(path)
        print(f"# {path}: {sum(v[0] for v in tot.values()):.2f} ms in {sum(v[1] for v in tot.values())} launches")
        for name, (ms, n) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
            print(f"  {ms:9.3f} ms {n:5d}  {name}")
