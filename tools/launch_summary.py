"""Summarises an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel name."""
import collections
import csv
import io
import sys


def load(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def main(path):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        v = v / 1e3 if unit in ("nsecond", "ns") else (v * 1e3 if unit in ("msecond", "ms") else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"{len(rows)} launches, {tot / 1e3:.3f} ms serialised kernel time")
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{v:10.1f} us {100 * v / tot:5.1f}%  n={n:4d} avg={v / n:8.1f} us  {k[:90]}")


if __name__ == "__main__":
    main(sys.argv[1])
