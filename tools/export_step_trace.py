"""Overlap evidence for the bench step: one traced C2 train step (48 x 1600, 16384 rows,
SP(4,2), bf16, steady state: warm ring, pending write-backs from the previous step) exported in
the reference's trace CSV format (trace.cpp:147) plus a per-engine busy/overlap summary.
Usage: python tools/export_step_trace.py OUT_PREFIX [layers d rows k kp]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi, trace_io  # noqa: E402

prefix = sys.argv[1]
L, d, rows, k, kp = (int(v) for v in (sys.argv[2:7] if len(sys.argv) > 6 else (48, 1600, 16384, 4, 2)))
ex = sp.Executor(L, d, sp.StrategyConfig(sp.SUPERPIPELINE, k, kp), numerics=sp.BF16, trace=True)
W = np.empty((d, d), np.float32)
b = np.empty((d,), np.float32)
for i in range(L):
    _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data)
    ex.register_layer(i, W, b)
x = torch.from_numpy(sp.make_input(7, 0, rows, d)).cuda()
t = torch.from_numpy(sp.make_input(7, 1, rows, d)).cuda()
for _ in range(4):
    ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
st = ex.stats()
lb = (d * d + d) * 4
trace_rows = trace_io.trace_rows(ex, lb, rows * d * 4)
trace_io.export_trace_csv(trace_rows, prefix + ".csv")


def busy(kind, bwd=None):
    iv = sorted((e["t_start"], e["t_end"]) for e in ex.trace()
                if e["kind"] == kind and (bwd is None or bool(e["backward"]) == bwd))
    tot, cur = 0.0, None
    for a, z in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, z]
        else:
            cur[1] = max(cur[1], z)
    return tot + (cur[1] - cur[0] if cur else 0.0)


summary = {"config": f"{L}x{d}, {rows} rows, SP({k},{kp}), bf16 train step (steady state, trace=1)",
           "makespan_ms": st["makespan_ms"], "compute_ms": st["compute_ms"], "stall_ms": st["stall_ms"],
           "h2d_busy_ms": busy("H2D"), "d2h_busy_ms": busy("D2H"), "compute_busy_ms": busy("Compute"),
           "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"],
           "h2d_busy_frac_of_makespan": busy("H2D") / st["makespan_ms"],
           "compute_busy_frac_of_makespan": busy("Compute") / st["makespan_ms"],
           "rows_in_csv": len(trace_rows)}
with open(prefix + "_summary.json", "w") as f:
    json.dump(summary, f, indent=1)
    f.write("\n")
print(json.dumps(summary))
