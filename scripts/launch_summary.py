"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python scripts/launch_summary.py gpurun_out/launches.csv > profiles/<name>.md
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
    h = rows[hdr_i]
    kn, mv, mu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr_i + 1:]:
        if len(r) <= mv:
            continue
        name = r[kn].replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "").split("<")[0].split("(")[0].split("::")[-1]
        v = float(r[mv].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[mu], 1.0)
        tot[name][0] += 1
        tot[name][1] += v * scale
    allus = sum(t[1] for t in tot.values())
    print(f"| kernel | launches | total us | share | us/launch |")
    print("|---|---:|---:|---:|---:|")
    for name, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {n} | {us:.1f} | {100 * us / allus:.1f}% | {us / n:.2f} |")
    print(f"\n{sum(t[0] for t in tot.values())} launches, {allus / 1e3:.2f} ms of kernel time (serialised, cold-cache ncu replay)")


if __name__ == "__main__":
    main(sys.argv[1])
