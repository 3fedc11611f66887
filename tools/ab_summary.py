"""Summarise ncu --csv launch lists (gpu__time_duration.sum) of tools/ab_probe.py runs: median
duration per (shape, GEMM) for each run, ratio against the first (baseline) run.
Usage: python tools/ab_summary.py base.csv other.csv [...]"""
import csv
import os
import sys


def load(path):
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    return [float(r["Metric Value"]) for r in rows
            if r.get("Metric Name") == "gpu__time_duration.sum" and "gemm" in r["Kernel Name"]]


runs = [(os.path.basename(p).replace(".csv", ""), load(p)) for p in sys.argv[1:]]
names = ["fwd", "dx", "dw_split"]
n = min(len(v) for _, v in runs)
print("shape gemm      " + "".join(f"{name[:22]:>24s}" for name, _ in runs))
for i in range(0, n, 9):
    for j, g in enumerate(names):
        med = [sorted(v[i + j + 3 * k] for k in range(3))[1] for _, v in runs]
        cells = "".join(f"{m / 1e3:10.1f} us ({med[0] / m:5.3f}x)" for m in med)
        print(f"{i // 9:5d} {g:9s} {cells}")
