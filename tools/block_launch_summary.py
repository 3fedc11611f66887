"""Summarises a block step's ncu launch list: totals by kernel kind, and the per-layer
sequence of one steady-state layer (forward and backward) in launch order with the GEMM
shapes implied by the block's op order (bench/DESIGN tables)."""
import collections
import csv
import io
import json
import sys


def load(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    out = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        out.append((r["Kernel Name"], us, r.get("Grid Size", ""), r.get("Stream", "")))
    return out


def kind(name):
    n = name.split("(")[0]
    if "gemm" in n:
        return n.split("<")[0] + "<" + name.split("<", 1)[1].split(">")[0] + ">" if "<" in name else n
    return n.split("<")[0]


def main(path, out_json=None):
    rows = load(path)
    tot = sum(us for _, us, _, _ in rows)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us, _, _ in rows:
        k = kind(name)
        agg[k][0] += 1
        agg[k][1] += us
    print(f"{len(rows)} launches, {tot / 1e3:.3f} ms serialised kernel time")
    summary = []
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{us / 1e3:9.3f} ms {100 * us / tot:5.1f}%  n={n:4d} avg={us / n:8.1f} us  {k[:110]}")
        summary.append({"kernel": k, "launches": n, "ms": us / 1e3, "share": us / tot})
    if out_json:
        json.dump({"launches": len(rows), "serialised_ms": tot / 1e3, "by_kernel": summary}, open(out_json, "w"),
                  indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
