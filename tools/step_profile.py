"""Breaks one Superpipeline train step into its measured timeline (CUDA events per op) and
host-side call time. Usage: python tools/step_profile.py [layers d rows k kp]"""
import json
import os
import sys
import time
from collections import defaultdict

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402

L, d, rows, k, kp = (int(v) for v in (sys.argv[1:6] if len(sys.argv) > 5 else (48, 1600, 16384, 4, 2)))
ex = sp.Executor(L, d, sp.StrategyConfig(sp.SUPERPIPELINE, k, kp), numerics=sp.BF16,
                 trace=os.environ.get("TRACE", "1") != "0")
W = np.empty((d, d), np.float32)
b = np.empty((d,), np.float32)
for i in range(L):
    _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data)
    ex.register_layer(i, W, b)
x = torch.from_numpy(sp.make_input(7, 0, rows, d)).cuda()
t = torch.from_numpy(sp.make_input(7, 1, rows, d)).cuda()
for i in range(3):
    t0 = time.perf_counter()
    loss = ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
    host = time.perf_counter() - t0
    st = ex.stats()
    print(json.dumps({"step": i, "host_s": host, "loss": loss, "makespan_ms": st["makespan_ms"],
                      "compute_ms": st["compute_ms"], "stall_ms": st["stall_ms"],
                      "gemm_ms": st["gemm_ms"], "kernels": st["kernels_launched"], "enqueue_ms": st["host_enqueue_ms"], "replays": st["graph_replays"],
                      "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"]}))
tr = ex.trace()
agg = defaultdict(lambda: [0, 0.0, 0.0])
for e in tr:
    key = (e["kind"], e["backward"])
    agg[key][0] += 1
    agg[key][1] += e["t_end"] - e["t_start"]
    agg[key][2] = max(agg[key][2], e["t_end"] - e["t_start"])
for key, (n, tot, mx) in sorted(agg.items()):
    print(f"{key[0]:8s} bwd={int(key[1])} n={n:4d} total={tot:9.3f} ms max={mx:8.3f} ms")
top = sorted(tr, key=lambda e: e["t_end"] - e["t_start"], reverse=True)[:12]
for e in top:
    print(f"  {e['kind']:8s} layer={e['layer']:3d} bwd={int(e['backward'])} "
          f"[{e['t_start']:9.3f}, {e['t_end']:9.3f}] dur={e['t_end'] - e['t_start']:8.3f}")
first = [e for e in tr if e["kind"] == "Compute"][:6]
for e in first:
    print("  first computes", e["layer"], round(e["t_start"], 3), round(e["t_end"], 3))
