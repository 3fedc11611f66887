"""Writes the profiles/ summaries from ncu artifacts: per-kernel key metrics of a `--set full`
report (one block per captured launch) and, optionally, the roofline traffic record bench.py
reads (profiles/gemm_traffic.json). Usage:
  python tools/profile_summary.py REPORT.ncu-rep OUT.txt "command line" [traffic.json ALGO_BYTES]"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__cluster_dim_x",
           "launch__shared_mem_per_block_dynamic"]
rep, out, cmd = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
lines = [f"ncu --set full --clock-control none --import-source on ({cmd})", ""]
launches = []
for r in data:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    lines.append(f"  Kernel Name: {d['Kernel Name']}")
    for m in METRICS:
        if m in d:
            lines.append(f"  {m}: {d[m]} {u.get(m, '')}".rstrip())
    lines.append("")
    launches.append(d)
open(out, "w").write("\n".join(lines))
print("\n".join(lines))
if len(sys.argv) > 5:
    d = launches[0]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    u = dict(zip(hdr, units))
    tot = sum(float(d[m]) * scale[u[m]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    json.dump({"kernel": d["Kernel Name"], "bytes_per_launch": tot,
               "algorithmic_bytes_per_launch": float(sys.argv[5]), "source": out},
              open(sys.argv[4], "w"), indent=1)
