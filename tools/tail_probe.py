"""End-of-step anatomy of the training step: when the last compute, the last update and the
last writeback D2H finish, and the D2H queue depth at the end (trace=1, CUDA events)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_08791_b200 as sp  # noqa: E402
from paper_2410_08791_b200 import _capi  # noqa: E402
from paper_2410_08791_b200.trace_io import plan_ops  # noqa: E402

L, d, rows = 48, 1600, 16384
ex = sp.Executor(L, d, sp.StrategyConfig(sp.SUPERPIPELINE, 4, 2), numerics=sp.BF16, trace=True)
W = np.empty((d, d), np.float32)
b = np.empty((d,), np.float32)
for i in range(L):
    _capi.LIB.sp_build_layer(7, i, d, 0, 0, W.ctypes.data, b.ctypes.data)
    ex.register_layer(i, W, b)
x = torch.from_numpy(sp.make_input(7, 0, rows, d)).cuda()
t = torch.from_numpy(sp.make_input(7, 1, rows, d)).cuda()
for _ in range(4):
    ex.train_step_ptr(x.data_ptr(), t.data_ptr(), rows, 0.01, device=True)
tr = ex.trace()
_, ops = plan_ops(ex.last_plan())
comp = [e for e in tr if e["kind"] == "Compute"]
d2h = [e for e in tr if e["kind"] == "D2H"]
h2d = [e for e in tr if e["kind"] == "H2D"]
end = max(e["t_end"] for e in tr)
print(f"makespan {end:.3f} ms; last compute end {max(e['t_end'] for e in comp):.3f}; "
      f"last H2D end {max(e['t_end'] for e in h2d):.3f}; last D2H end {max(e['t_end'] for e in d2h):.3f}")
bwd_d2h = sorted(d2h, key=lambda e: e["t_start"])[-8:]
for e in bwd_d2h:
    print(f"  D2H layer {e['layer']:2d} [{e['t_start']:.3f}, {e['t_end']:.3f}]")
bwd_c = sorted([e for e in comp if e["backward"]], key=lambda e: e["t_start"])[-8:]
for e in bwd_c:
    print(f"  bwd compute layer {e['layer']:2d} [{e['t_start']:.3f}, {e['t_end']:.3f}]")
fwd_h2d = sorted([e for e in h2d if not e["backward"]], key=lambda e: e["t_start"])[:3]
for e in fwd_h2d:
    print(f"  fwd H2D first layers {e['first_layer']} [{e['t_start']:.3f}, {e['t_end']:.3f}]")
# every op of the last ~12 layers' backward, with its dependencies and measured interval
rows = {e["op_index"]: e for e in tr if e.get("op_index", -1) >= 0}
print("op  kind     layer  start    end      deps")
tail_start = min(e["t_start"] for e in bwd_c) - 0.6
for i, op in enumerate(ops):
    e = rows.get(i)
    if e is None or e["t_start"] < tail_start:
        continue
    print(f"{i:4d} {op['kind']:8s} {op.get('layer', op.get('layers', [-1])[0] if op.get('layers') else -1):5} "
          f"{e['t_start']:8.3f} {e['t_end']:8.3f}  {op.get('deps')}")
