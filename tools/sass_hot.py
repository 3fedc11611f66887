"""Hot SASS lines of an ncu report's source page: samples and stall reasons per instruction.
  ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv; python tools/sass_hot.py x.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
isrc, iss, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in cols}
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = sum(int(r[iss] or 0) for r in data)
print("samples", tot, "instructions", sum(int(r[iex] or 0) for r in data))
by = collections.Counter()
for r in data:
    for c in cols:
        by[c] += int(r[idx[c]] or 0)
print("by reason:", by.most_common(8))
for i, r in sorted(enumerate(data), key=lambda x: -int(x[1][iss] or 0))[:n]:
    top = sorted(((int(r[idx[c]] or 0), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{i:5d} {r[iss]:>6} {r[iex]:>9}  {r[isrc][:70]:70s} {top}")
