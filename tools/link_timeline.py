"""Where does a train step lose time against the link bound? Runs traced steps (per-op CUDA
events) and reports, per copy direction, busy time, idle gaps and effective bandwidth, plus
the phase boundaries (forward end, first backward load, last write-back).
Usage: python tools/link_timeline.py [layers d rows k kp optimizer]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402

args = sys.argv[1:]
L, d, rows, k, kp = (int(v) for v in (args[:5] if len(args) >= 5 else (48, 1600, 16384, 4, 2)))
opt = args[5] if len(args) > 5 else "sgd"
strat = sp.StrategyConfig(sp.STANDARD) if k == 0 else sp.StrategyConfig(sp.SUPERPIPELINE, k, kp)  # k=0: Standard
ex = sp.Executor(L, d, strat, numerics=sp.BF16, trace=True)
W = np.empty((d, d), np.float32)
b = np.empty((d,), np.float32)
for i in range(L):
    _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data)
    ex.register_layer(i, W, b)
if opt == "adamw":
    ex.set_optimizer(sp.OPT_ADAMW, 0.9, 0.999, 1e-8, 0.01)
x = torch.from_numpy(sp.make_input(7, 0, rows, d)).cuda()
t = torch.from_numpy(sp.make_input(7, 1, rows, d)).cuda()
for _ in range(4):
    ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
st = ex.stats()
tr = ex.trace()


def union(iv):
    iv = sorted(iv)
    busy, gaps, cur = 0.0, [], None
    for a, b in iv:
        if cur is None:
            cur = [a, b]
        elif a > cur[1]:
            busy += cur[1] - cur[0]
            gaps.append((cur[1], a))
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    if cur:
        busy += cur[1] - cur[0]
    return busy, gaps


out = {"makespan_ms": st["makespan_ms"], "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"]}
for kind in ("H2D", "D2H", "Compute", "Update"):
    ev = [e for e in tr if e["kind"] == kind]
    if not ev:
        continue
    busy, gaps = union([(e["t_start"], e["t_end"]) for e in ev])
    big = sorted(gaps, key=lambda g: g[0] - g[1])[:8]
    out[kind] = {"n": len(ev), "first": min(e["t_start"] for e in ev), "last": max(e["t_end"] for e in ev),
                 "busy_ms": busy, "idle_gaps_ms": sum(b - a for a, b in gaps),
                 "largest_gaps": [(round(a, 3), round(b - a, 3)) for a, b in big]}
fwd_end = max(e["t_end"] for e in tr if e["kind"] == "Compute" and not e["backward"])
out["forward_end_ms"] = fwd_end
bwd_h2d = [e for e in tr if e["kind"] == "H2D" and e["backward"]]
if bwd_h2d:
    out["first_backward_h2d_start"] = min(e["t_start"] for e in bwd_h2d)
lb = (d * d + d) * 4
for kind in ("H2D", "D2H"):
    ev = [e for e in tr if e["kind"] == kind]
    dur = [e["t_end"] - e["t_start"] for e in ev]
    if dur:
        out[kind]["median_op_ms"] = float(np.median(dur))
        out[kind]["max_op_ms"] = float(np.max(dur))
for e in tr[:0]:
    pass
print(json.dumps(out, indent=1))
# ops around the forward/backward turn-around
turn = sorted([e for e in tr if abs(e["t_start"] - fwd_end) < 1.0], key=lambda e: e["t_start"])
for e in turn:
    print(f"  {e['kind']:8s} L={e['layer']:3d} bwd={int(e['backward'])} [{e['t_start']:8.3f} {e['t_end']:8.3f}]")
tail = sorted(tr, key=lambda e: e["t_end"])[-8:]
print("tail:")
for e in tail:
    print(f"  {e['kind']:8s} L={e['layer']:3d} bwd={int(e['backward'])} [{e['t_start']:8.3f} {e['t_end']:8.3f}]")
head = sorted(tr, key=lambda e: e["t_start"])[:10]
print("head:")
for e in head:
    print(f"  {e['kind']:8s} L={e['layer']:3d} bwd={int(e['backward'])} [{e['t_start']:8.3f} {e['t_end']:8.3f}]")
if os.environ.get("SEGMENT"):
    lo, hi = (float(v) for v in os.environ["SEGMENT"].split(","))
    print("segment:")
    for e in sorted(tr, key=lambda e: e["t_start"]):
        if lo <= e["t_start"] <= hi and (e["kind"] != "Stall" or os.environ.get("STALLS")):
            print(f"  {e['kind']:8s} L={e['layer']:3d} bwd={int(e['backward'])} [{e['t_start']:8.3f} {e['t_end']:8.3f}] "
                  f"dur={e['t_end'] - e['t_start']:.3f}")
