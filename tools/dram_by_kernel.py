"""Per-kernel DRAM bytes and time from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (CSV): one line per
launch, in launch order, and per-kernel sums.
Usage: python tools/dram_by_kernel.py LIST.csv [LIST2.csv ...]"""
import collections
import csv
import sys

SC = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
TS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault((r[ii], r[ki].split("(")[0].replace("void ", "")), {})[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    print(path)
    sums, tts = collections.defaultdict(float), collections.defaultdict(float)
    for (i, n), m in per.items():
        t, rd, wr = m["gpu__time_duration.sum"], m["dram__bytes_read.sum"], m["dram__bytes_write.sum"]
        us = TS[t[1]] * t[0]
        mb_r, mb_w = rd[0] * SC[rd[1]], wr[0] * SC[wr[1]]
        print(f"  {i:>4} {n[:44]:44s} {us:8.1f} us  rd {mb_r:8.1f} MB  wr {mb_w:7.1f} MB")
        sums[n] += mb_r + mb_w
        tts[n] += us
    print("  per kernel:")
    for n in sorted(sums, key=lambda k: -tts[k]):
        print(f"    {n[:44]:44s} {tts[n]:9.1f} us  {sums[n]:9.1f} MB")
    print(f"  total {sum(tts.values()):.1f} us, {sum(sums.values()):.1f} MB")
